#!/bin/bash
# Round-2 (n): hybrid conversion (integer groups under the MMAs, FP64 groups after them), bucketed F1 exponents.
O=gpurun_out/${1:-r02n}; mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/i8_mma_rate.cu -o /tmp/i8_mma_rate && timeout 120 /tmp/i8_mma_rate > $O/i8_mma_rate.json 2>&1
timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > $O/ozaki_tests.log 2>&1; echo rc=$? >> $O/ozaki_tests.log
for ig in 0 1 2 3 4; do
  TS_OZAKI_INT_GROUPS=$ig timeout 300 python tools/ozaki_stageA.py > $O/stageA_ig$ig.log 2>&1
done
for ig in 0 3; do
  TS_OZAKI_INT_GROUPS=$ig timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > $O/ozaki_tests_ig$ig.log 2>&1
done
timeout 600 python bench.py --config 5 --steps 30 --no-cpu-baseline --no-e2e --stages > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg5 or baseline or reference_semantics" > $O/parity_tests.log 2>&1; echo rc=$? >> $O/parity_tests.log
for f in $O/*.log; do echo "$f: $(tail -n 1 $f)"; done
python -c "
import json
d=json.loads(open('$O/bench_cfg5.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stages_ms'], d['roofline'].get('int8_engine_stages'))"
