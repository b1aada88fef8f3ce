"""NDG pattern (reference src/ndg.cpp:401-462): S
independent sums of a BASELINE config's shape with a shared plan, fresh data per
step (no graph replay).  Sums/s of (a) S sequential ts_krp_sum calls, (b)
ts_krp_sum_many (lanes), (c) one ts_krp_sum_segmented call; device time with
CUDA events on the engine stream, inputs resident."""
import argparse
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2603_13532_b200 import tucksum as T  # noqa: E402
from paper_2603_13532_b200.workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--sums", type=int, default=64)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--once", action="store_true")
a = ap.parse_args()
wls = [make_workload(a.config, node=i + 1) for i in range(a.sums)]
widths, cap = wls[0].widths, wls[0].cap
eng = T.Engine(0)
eng.set_graphs(False)
stream = torch.cuda.ExternalStream(eng.stream)
xs, ws, seg = [], [], [0]
for w in wls:
    xs += w.summands
    ws += list(w.weights)
    seg.append(len(xs))
big = eng.upload(xs)
singles = [eng.upload(w.summands) for w in wls]
seeds = [w.seed for w in wls]
for w in wls:
    eng.prepare_omega(w.dims, max(widths), w.seed)


def timed(fn):
    ts = []
    for i in range(a.reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        out = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        for r in out:
            r.free()
        if i >= 2:
            ts.append((e0.elapsed_time(e1), 1000 * wall))
    return float(np.median([t[0] for t in ts])), float(np.median([t[1] for t in ts]))


seq = timed(lambda: [eng.krp_sum(b, w.weights, widths, w.seed, 0.0, cap) for b, w in zip(singles, wls)])
many = timed(lambda: eng.krp_sum_many(singles, [w.weights for w in wls], widths, seeds, 0.0, cap, lanes=8))
segd = timed(lambda: eng.krp_sum_segmented(big, seg, ws, widths, seeds, 0.0, cap))
seg_paths = eng.last_paths()
if a.once:  # one extra segmented call (ncu target)
    for r in eng.krp_sum_segmented(big, seg, ws, widths, seeds, 0.0, cap):
        r.free()
line = {"pattern": "NDG: independent sums with a shared plan (src/ndg.cpp:401-462)", "config": a.config,
        "sums": a.sums, "summands_per_sum": wls[0].K, "eps": 0.0, "cap": cap, "widths": widths,
        "sequential_ms": seq[0], "sequential_wall_ms": seq[1], "many_lanes_ms": many[0], "many_lanes_wall_ms": many[1],
        "segmented_ms": segd[0], "segmented_wall_ms": segd[1],
        "sums_per_s": {"sequential": a.sums / (seq[1] / 1000), "many_lanes": a.sums / (many[1] / 1000),
                       "segmented": a.sums / (segd[1] / 1000)},
        "speedup_segmented_vs_sequential": seq[1] / segd[1], "segmented_last_paths": list(seg_paths)}
print(json.dumps(line), flush=True)
eng.close()
