#!/bin/bash
mkdir -p gpurun_out
./tools/dmma_issue > gpurun_out/dmma_issue.jsonl 2>&1
timeout 1200 python -m pytest tests/ -q -m gpu --timeout 600 -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
B="python bench.py --no-cpu-baseline --no-e2e --stages --steps 20"
$B > gpurun_out/r4_default.json 2> gpurun_out/r4_default.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r4.csv $CMD > gpurun_out/ncu_list.log 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -1 gpurun_out/r4_default.err
echo done
