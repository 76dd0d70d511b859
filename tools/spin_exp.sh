#!/bin/bash
SHAPES="1024,3,64 200,4,100 64,5,32" DBGS="0 128" timeout 900 bash tools/i8d_exp.sh 2>&1
