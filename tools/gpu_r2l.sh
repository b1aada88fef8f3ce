#!/bin/bash
# Round-2 (l): FP64 / integer vs tensor-MMA contention probe; fused small-operand preparation.
O=gpurun_out/${1:-r02l}; mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/i8_mma_rate.cu -o /tmp/i8_mma_rate && timeout 120 /tmp/i8_mma_rate > $O/i8_mma_rate.json 2>&1
grep contend $O/i8_mma_rate.json
timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > $O/ozaki_tests.log 2>&1; echo rc=$? >> $O/ozaki_tests.log
timeout 600 python bench.py --config 5 --steps 30 --no-cpu-baseline --no-e2e --stages > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ll_cfg5.csv \
  python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-error > $O/ll_cfg5.log 2>&1
for f in $O/*.log; do echo "$f: $(tail -n 1 $f)"; done
python -c "
import json
d=json.loads(open('$O/bench_cfg5.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stages_ms'], d['roofline'].get('int8_engine_stages'))"
