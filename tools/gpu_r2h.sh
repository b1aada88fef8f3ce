#!/bin/bash
# Round-2 (h): Ozaki engine with the F digits staged in TMEM (TS MMAs) vs shared
# memory (SS), wave-aware K splits; accuracy tests, stage-A-sized timing, cfg5 A/B.
O=gpurun_out/${1:-r02h}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > $O/ozaki_tests.log 2>&1; echo rc=$? >> $O/ozaki_tests.log
for ts in 1 0; do for sp in 0 3 4 6; do
  TS_OZAKI_TS=$ts TS_OZAKI_SPLITS=$sp timeout 300 python tools/ozaki_stageA.py > $O/stageA_ts${ts}_sp$sp.log 2>&1
done; done
for v in 1 2 3; do
  TS_OZAKI_VARIANT=$v timeout 300 python tools/ozaki_stageA.py > $O/stageA_ts1_variant$v.log 2>&1
done
for ts in 1 0; do
  TS_OZAKI_TS=$ts timeout 600 python bench.py --config 5 --steps 30 --no-cpu-baseline --no-e2e --stages > $O/bench_cfg5_ts$ts.json 2> $O/bench_cfg5_ts$ts.err
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ozaki.py -x -q > $O/parity_tests.log 2>&1; echo rc=$? >> $O/parity_tests.log
tail -n 3 $O/*.log
