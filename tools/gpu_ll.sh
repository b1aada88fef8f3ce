#!/bin/bash
# ncu launch lists (per-kernel durations) of one config-5 and one config-1 call + the eigensolver probe.
O=gpurun_out/ll; mkdir -p $O
timeout 600 python tools/probe_trd.py > $O/probe_trd.json 2>&1
for c in 5 1; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ll_cfg$c.csv \
  python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-error > $O/ll_cfg$c.log 2>&1
done
ls -la $O
