#!/bin/bash
# C3 digit TTM: N-tile width cap (Rp 32 -> ping-pong TMEM accumulators) x cluster size (A multicast)
for cfg in "" "CPD_I8_RPMAX=32" "CPD_I8_RPMAX=32 CPD_I8_CLUSTER=4" "CPD_I8_RPMAX=48"; do
  env $cfg SHAPES="200,4,100" DBGS="0" timeout 600 bash tools/i8d_exp.sh 2>&1 | sed "s/^/[$cfg] /"
done
for cfg in "" "CPD_I8_RPMAX=32 CPD_I8_CLUSTER=4"; do
  env $cfg SHAPES="2048,3,200" DBGS="0" timeout 600 bash tools/i8d_exp.sh 2>&1 | sed "s/^/[$cfg] /"
done
