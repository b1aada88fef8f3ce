#!/bin/bash
# ncu captures of the config-3 accurate-path kernels (TSQR factor, one-sided Jacobi SVD).
O=gpurun_out/r25
mkdir -p $O
CMD="python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-error"
timeout 300 $CMD > $O/plain.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tsqr_factor -s 4 -c 1 -o $O/prof_tsqr_factor $CMD > $O/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi_svd -s 2 -c 1 -o $O/prof_jacobi_svd $CMD > $O/ncu2.log 2>&1
echo done
