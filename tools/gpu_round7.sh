#!/bin/bash
# Evidence run for profiles/ (round 1, v3): tests, smoke, both bench arms, all
# configs, cfg5 launch list and full ncu captures of the stage-A GEMM, the
# Jacobi values kernel and chol_inv.
O=gpurun_out/r7
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "rc=$?" >> $O/bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline --stages > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e --stages > $O/bench_cfg5_stages.json 2> $O/bench_cfg5_stages.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
if timeout 300 $CMD > $O/plain.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tma_kernel -s 0 -c 1 -o $O/prof_gemm_tma_stageA $CMD > $O/ncu_gemm.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:jacobi_values -s 3 -c 1 -o $O/prof_jacobi_values $CMD > $O/ncu_jacobi.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:chol_inv -s 2 -c 1 -o $O/prof_chol_inv $CMD > $O/ncu_chol.log 2>&1
fi
echo done
