#!/bin/bash
mkdir -p gpurun_out
python bench.py --steps 50 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench rc=$?" >> gpurun_out/bench_cfg5.err
for c in 1 2 3 4; do
  python bench.py --config $c --steps 50 --no-cpu-baseline --stages > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r5.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo done
