"""Throughput of independent small sums: sequential ts_krp_sum vs ts_krp_sum_many
(SURVEY.md §8(f) row 2).  Prints one JSON line per (config, lanes)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_13532_b200 import tucksum as T
from paper_2603_13532_b200.workloads import make_workload

eng = T.Engine(0)
for cfg, nsums in ((1, 32), (2, 16), (4, 16)):
    wl = make_workload(cfg)
    batches = [eng.upload(wl.summands) for _ in range(nsums)]
    seeds = [T.RngSeed(wl.seed.seed, wl.seed.stream + i) for i in range(nsums)]
    ws = [wl.weights] * nsums
    for s in seeds:  # Ω generation outside the timing
        eng.prepare_omega(wl.dims, max(wl.widths), s)
    def seq():
        for b, w, s in zip(batches, ws, seeds):
            eng.krp_sum(b, w, wl.widths, s, wl.eps, wl.cap).free()
    def many(lanes):
        for r in eng.krp_sum_many(batches, ws, wl.widths, seeds, wl.eps, wl.cap, lanes=lanes):
            r.free()
    seq(); many(8)
    t0 = time.perf_counter(); seq(); t1 = time.perf_counter()
    row = {"probe": "krp_sum_many", "config": wl.name, "sums": nsums, "sequential_ms_per_sum": 1e3 * (t1 - t0) / nsums}
    for lanes in (2, 4, 8, 16):
        many(lanes)
        t0 = time.perf_counter(); many(lanes); t1 = time.perf_counter()
        row[f"lanes{lanes}_ms_per_sum"] = 1e3 * (t1 - t0) / nsums
    print(json.dumps(row))
    for b in batches:
        b.free()
