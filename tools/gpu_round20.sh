#!/bin/bash
# Full GPU suite + smoke + bench lines for configs 1-5 with CUDA-graph replay.
O=gpurun_out/r35
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 600 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
echo done
