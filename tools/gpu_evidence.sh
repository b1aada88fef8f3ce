#!/bin/bash
# End-of-milestone evidence on the current code: bench lines (all configs, the
# default cfg5 line with e2e + CPU baselines), the reference arm, the NDG
# pattern, a cfg5 / cfg1 ncu launch list and full ncu captures of the dominant
# kernel (stage C) and the stage-G eigensolver.  Usage: tools/gpu_evidence.sh <outdir>
O=gpurun_out/${1:-ev}; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline --stages > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 600 python bench.py --config 5 --eps 1e-6 --no-cap --steps 30 --no-cpu-baseline --no-e2e > $O/bench_cfg5_eps.json 2> $O/bench_cfg5_eps.err
TS_OZAKI=0 timeout 600 python bench.py --config 5 --steps 30 --no-cpu-baseline --no-e2e > $O/bench_cfg5_dmma.json 2> $O/bench_cfg5_dmma.err
timeout 600 python bench.py --config 6 --steps 10 --no-e2e > $O/bench_fig2.json 2> $O/bench_fig2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 300 python tools/ndg_probe.py --config 1 --sums 64 > $O/ndg_cfg1.json 2>&1
timeout 300 python tools/ndg_probe.py --config 4 --sums 32 > $O/ndg_cfg4.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ll_cfg5.csv \
  python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-error > $O/ll_cfg5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ll_cfg1.csv \
  python bench.py --config 1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-error > $O/ll_cfg1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ozaki_gemm -s 4 -c 1 -o $O/ncu_ozaki_stageC \
  python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-error > $O/ncu_ozaki.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:trd_eig -s 3 -c 1 -o $O/ncu_trd \
  python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-error > $O/ncu_trd.log 2>&1
ls -la $O
