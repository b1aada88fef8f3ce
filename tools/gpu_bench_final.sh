#!/bin/bash
# Bench lines on the final code (after the stacked-upload e2e path).
O=gpurun_out/final5
mkdir -p $O
timeout 600 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 600 python bench.py --config 5 --strategy kron --steps 30 --no-cpu-baseline --e2e-steps 2 > $O/bench_kron_cfg5.json 2> $O/bench_kron_cfg5.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
echo done
