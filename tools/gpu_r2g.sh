#!/bin/bash
# Round-2 (g): Ozaki engine with A in TMEM (vs the smem-A engine), F2 on the
# int8 engine, accuracy tests, stage-A-sized timing, cfg5 bench A/B, latency probe.
O=gpurun_out/${1:-r02g}; mkdir -p $O
python -c "from paper_2603_13532_b200 import build as b; b.build()" > $O/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lat_probe.cu -o /tmp/lat_probe && /tmp/lat_probe > $O/lat_probe.json 2>&1
timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > $O/ozaki_tests.log 2>&1; echo rc=$? >> $O/ozaki_tests.log
for ta in 1 0; do
  TS_OZAKI_TMEM_A=$ta timeout 300 python tools/ozaki_stageA.py > $O/stageA_ta$ta.log 2>&1
  TS_OZAKI_TMEM_A=$ta timeout 600 python bench.py --config 5 --steps 30 --no-cpu-baseline --no-e2e --stages > $O/bench_cfg5_ta$ta.json 2> $O/bench_cfg5_ta$ta.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg5 or reference_semantics or baseline" > $O/parity_tests.log 2>&1; echo rc=$? >> $O/parity_tests.log
timeout 300 python tools/probe_trd.py > $O/probe_trd.json 2>&1
ls -la $O
