#!/bin/bash
# Round-2 (p): vectorised split-partial stores in the Ozaki epilogue; full GPU suite.
O=gpurun_out/${1:-r02p}; mkdir -p $O
TS_OZAKI_VARIANT=9 timeout 300 python tools/ozaki_stageA.py 2>&1 | grep -v "oz-trace chunk" | tail -5 > $O/trace2.log
timeout 300 python tools/ozaki_stageA.py > $O/stageA.log 2>&1
timeout 600 python bench.py --config 5 --steps 30 --no-cpu-baseline --no-e2e --stages > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 2400 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
cat $O/trace2.log; for f in $O/stageA.log $O/gpu_tests.log; do echo "$f: $(tail -n 2 $f)"; done
python -c "
import json
d=json.loads(open('$O/bench_cfg5.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stages_ms'], d['roofline'].get('int8_engine_stages'))"
