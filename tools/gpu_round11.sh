#!/bin/bash
# Bench lines for the KRP hot path (with the device error check) and the widened
# rows: Kron sketch (configs 1, 2, 5) and Lazy rounding (config 1, the only
# config whose stacked ranks fit the device QR).
O=gpurun_out/r11
mkdir -p $O
timeout 600 python bench.py --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "rc=$?" >> $O/bench_cfg5.err
for c in 1 2 5; do
  timeout 600 python bench.py --config $c --strategy kron --steps 30 --no-cpu-baseline --e2e-steps 2 > $O/bench_kron_cfg$c.json 2> $O/bench_kron_cfg$c.err
done
timeout 600 python bench.py --config 1 --strategy lazy --steps 50 --no-cpu-baseline > $O/bench_lazy_cfg1.json 2> $O/bench_lazy_cfg1.err
timeout 600 python bench.py --config 1 --steps 50 --no-cpu-baseline > $O/bench_krp_cfg1.json 2> $O/bench_krp_cfg1.err
echo done
