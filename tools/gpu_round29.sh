#!/bin/bash
# ncu --set full captures of the config-5 stage-B (krp3), stage-F1 (ttm3) and
# stage-A GEMM kernels, and the config-4 split-J stage-B kernel.
O=gpurun_out/r29
mkdir -p $O
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-error"
timeout 300 $CMD > $O/plain.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:krp3_dmma -s 3 -c 1 -o $O/prof_krp3 $CMD > $O/n1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ttm3_kernel -s 3 -c 1 -o $O/prof_ttm3 $CMD > $O/n2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tma_kernel -s 0 -c 1 -o $O/prof_gemm_stageA $CMD > $O/n3.log 2>&1
CMD4="python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-error"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:krp_dmma_kernel -s 3 -c 1 -o $O/prof_krp_splitj_cfg4 $CMD4 > $O/n4.log 2>&1
echo done
