#!/bin/bash
SHAPES="200,4,100 1024,3,64" DBGS="0 256 258 2 34" timeout 900 bash tools/i8d_exp.sh 2>&1
