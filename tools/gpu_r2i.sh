#!/bin/bash
# Round-2 (i): int8 MMA issue-rate probe, fp64 latency probe, ncu --set full of the TS Ozaki kernel.
O=gpurun_out/${1:-r02i}; mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/i8_mma_rate.cu -o /tmp/i8_mma_rate && timeout 120 /tmp/i8_mma_rate > $O/i8_mma_rate.json 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lat_probe.cu -o /tmp/lat_probe && timeout 120 /tmp/lat_probe > $O/lat_probe.json 2>&1
timeout 300 python tools/ozaki_stageA.py > $O/stageA.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ozaki_gemm -s 2 -c 1 -o $O/ncu_ozaki_ts python tools/ozaki_stageA.py > $O/ncu_ozaki.log 2>&1
timeout 300 python tools/probe_trd.py > $O/probe_trd.json 2>&1
cat $O/i8_mma_rate.json $O/lat_probe.json; tail -2 $O/stageA.log $O/ncu_ozaki.log; tail -20 $O/probe_trd.json
