#!/bin/bash
# GPU call: parity tests, then bench cfg5 + per-config stages.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python bench.py --no-cpu-baseline --stages > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench rc=$?" >> gpurun_out/bench_cfg5.err
for c in 1 2 3 4; do
  python bench.py --config $c --steps 50 --no-cpu-baseline --no-e2e --stages > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
done
echo done
