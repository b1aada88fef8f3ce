#!/bin/bash
O=gpurun_out/r2a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1; nproc > $O/nproc.txt
timeout 600 python bench.py --steps 20 --stages --no-cpu-baseline --e2e-steps 2 > $O/cfg5.json 2> $O/cfg5.err
timeout 600 python bench.py --steps 20 --stages --no-cpu-baseline --no-e2e --eps 1e-6 --no-cap > $O/cfg5_eps.json 2> $O/cfg5_eps.err
timeout 600 python bench.py --config 1 --steps 50 --stages --no-cpu-baseline --no-e2e > $O/cfg1.json 2> $O/cfg1.err
timeout 600 python bench.py --config 4 --steps 20 --stages --no-cpu-baseline --no-e2e --eps 1e-6 --no-cap > $O/cfg4_eps.json 2> $O/cfg4_eps.err
echo done
