#!/bin/bash
# One compute-sanitizer tool per call: racecheck | memcheck | synccheck
TOOL=${1:-racecheck}
O=gpurun_out/san_$TOOL; mkdir -p $O
TS_GRAPHS=0 timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_run.py > $O/out.log 2>&1; echo "rc=$?" >> $O/out.log
tail -20 $O/out.log
