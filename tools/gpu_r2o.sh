#!/bin/bash
O=gpurun_out/${1:-r02o}; mkdir -p $O
for ig in 2; do
  TS_OZAKI_VARIANT=9 TS_OZAKI_INT_GROUPS=$ig timeout 300 python tools/ozaki_stageA.py > $O/trace2_ig$ig.log 2>&1
done
grep -v "oz-trace chunk" $O/trace2_ig*.log | tail -12
