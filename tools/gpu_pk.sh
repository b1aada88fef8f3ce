#!/bin/bash
O=gpurun_out/${1:-pk}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_graphs.py tests/test_gpu_segmented.py tests/test_gpu_kron.py -x -q > $O/tests_a.log 2>&1; echo rc=$? >> $O/tests_a.log
for c in 1 2 3 4 5; do
  timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline --no-e2e --stages > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
tail -n 2 $O/tests_a.log $O/parity.log
for c in 1 2 3 4 5; do python -c "
import json
d=json.loads(open('$O/bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, round(d['ms_per_step'],4), {k:round(v,3) for k,v in d['stages_ms'].items() if v>0.02})"; done
