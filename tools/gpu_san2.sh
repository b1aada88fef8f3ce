#!/bin/bash
# compute-sanitizer racecheck then synccheck on the sanitize workload (one tool each, bounded).
for TOOL in racecheck synccheck; do
O=gpurun_out/san_$TOOL; mkdir -p $O
TS_GRAPHS=0 timeout 1200 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_run.py > $O/out.log 2>&1; echo "rc=$?" >> $O/out.log
tail -8 $O/out.log
done
