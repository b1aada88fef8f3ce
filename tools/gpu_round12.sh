#!/bin/bash
# Launch lists (kernel durations) for the latency-bound configs 1 and 4, and the
# Jacobi sweep counts per ST-HOSVD mode.
O=gpurun_out/r12
mkdir -p $O
for c in 1 4 5; do
  CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-error"
  if timeout 300 $CMD > $O/plain_cfg$c.log 2>&1; then
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg$c.csv $CMD > $O/ncu_list_cfg$c.log 2>&1
  fi
  TS_DEBUG_SWEEPS=1 timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-error > $O/sweeps_cfg$c.json 2> $O/sweeps_cfg$c.err
done
echo done
