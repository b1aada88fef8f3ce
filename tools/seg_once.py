"""Segmented sums only (ncu target): S sums of a BASELINE config, 2 warm-up calls + 1."""
import argparse
import sys

sys.path.insert(0, ".")
from paper_2603_13532_b200 import tucksum as T  # noqa: E402
from paper_2603_13532_b200.workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--sums", type=int, default=32)
a = ap.parse_args()
wls = [make_workload(a.config, node=i + 1) for i in range(a.sums)]
widths, cap = wls[0].widths, wls[0].cap
eng = T.Engine(0)
eng.set_graphs(False)
xs, ws, seg = [], [], [0]
for w in wls:
    xs += w.summands
    ws += list(w.weights)
    seg.append(len(xs))
big = eng.upload(xs)
for _ in range(3):
    for r in eng.krp_sum_segmented(big, seg, ws, widths, [w.seed for w in wls], 0.0, cap):
        r.free()
eng.close()
print("ok")
