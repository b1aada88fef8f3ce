#!/bin/bash
O=gpurun_out/seg; mkdir -p $O
timeout 300 python tools/ndg_probe.py --config 1 --sums 64 --reps 2 > $O/ndg1.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ll_seg1.csv \
  python tools/ndg_probe.py --config 1 --sums 64 --reps 0 > $O/ll_seg1.log 2>&1
cat $O/ndg1.json
