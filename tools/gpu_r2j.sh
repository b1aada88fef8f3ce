#!/bin/bash
# Round-2 (j): magic-number fp64 -> digit conversion (no F2I), high-priority side stream.
O=gpurun_out/${1:-r02j}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > $O/ozaki_tests.log 2>&1; echo rc=$? >> $O/ozaki_tests.log
timeout 300 python tools/ozaki_stageA.py > $O/stageA.log 2>&1
for v in 1 2 3; do
  TS_OZAKI_VARIANT=$v timeout 300 python tools/ozaki_stageA.py > $O/stageA_variant$v.log 2>&1
done
TS_OZAKI_TS=0 timeout 300 python tools/ozaki_stageA.py > $O/stageA_ss.log 2>&1
timeout 600 python bench.py --config 5 --steps 30 --no-cpu-baseline --no-e2e --stages > $O/bench_cfg5.json 2> $O/bench_cfg5.err
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline --no-e2e --stages > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ozaki_gemm -s 2 -c 1 -o $O/ncu_ozaki_ts python tools/ozaki_stageA.py > $O/ncu_ozaki.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > $O/parity_tests.log 2>&1; echo rc=$? >> $O/parity_tests.log
for f in $O/*.log; do echo "$f: $(tail -n 1 $f)"; done
