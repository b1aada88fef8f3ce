#!/bin/bash
# Config 3 (accurate path) launch list and stage split.
O=gpurun_out/r24
mkdir -p $O
CMD="python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-error"
timeout 300 $CMD > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3.csv $CMD > $O/ncu.log 2>&1
TS_DEBUG_SWEEPS=1 timeout 300 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-error > $O/sw.json 2> $O/sw.err
echo done
