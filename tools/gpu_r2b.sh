#!/bin/bash
# Round-2 session-2 check: GPU tests, smoke, benches on the current code.
O=gpurun_out/r2b; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
for c in 5 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --stages > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 300 python bench.py --config 5 --steps 20 --warmup 5 --no-cpu-baseline --eps 1e-6 --no-cap --stages > $O/bench_cfg5_eps.json 2> $O/bench_cfg5_eps.err
timeout 300 python tools/ndg_probe.py --config 1 --sums 64 > $O/ndg_cfg1.json 2>&1
timeout 300 python tools/ndg_probe.py --config 4 --sums 32 > $O/ndg_cfg4.json 2>&1
tail -3 $O/gpu_tests.log
