#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-e2e --stages --steps 20"
$B > gpurun_out/r3_default.json 2> gpurun_out/r3_default.err
for c in 1 2 3 4 5; do
  TS_GEMM_CFG_TN=$c TS_GEMM_CFG_NN=$c TS_GEMM_CFG_NT=$c $B > gpurun_out/r3_cfg$c.json 2> gpurun_out/r3_cfg$c.err
done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r3.csv $CMD > gpurun_out/ncu_list.log 2>&1
for f in gpurun_out/r3_*.err; do echo $f; tail -1 $f; done
echo done
