#!/bin/bash
# Re-validation of HEAD after session restore: GPU tests, smoke, bench cfg5 + cfg1-4.
O=gpurun_out/r8
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "rc=$?" >> $O/bench_cfg5.err
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline --stages > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e --stages > $O/bench_cfg5_stages.json 2> $O/bench_cfg5_stages.err
echo done
