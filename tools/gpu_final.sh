#!/bin/bash
# End-of-round evidence: full GPU suite, smoke, bench lines (configs 1-5, Kron,
# Lazy), reference arm, config-5 launch list (kernel shares).
O=gpurun_out/final3
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 600 python bench.py --config 5 --strategy kron --steps 30 --no-cpu-baseline --e2e-steps 2 > $O/bench_kron_cfg5.json 2> $O/bench_kron_cfg5.err
timeout 600 python bench.py --config 1 --strategy lazy --steps 50 --no-cpu-baseline > $O/bench_lazy_cfg1.json 2> $O/bench_lazy_cfg1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-error"
timeout 300 $CMD > $O/plain.log 2>&1 && TS_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg5.csv $CMD > $O/ncu_list.log 2>&1
echo done
