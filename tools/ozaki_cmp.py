"""Config 5 (reference-exact mode): device intermediates with the Ozaki stages A/E
vs the DMMA ones (TS_OZAKI toggled between two processes via argv)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13532_b200 import tucksum as T  # noqa: E402
from paper_2603_13532_b200.workloads import make_workload  # noqa: E402

wl = make_workload(5)
eng = T.Engine(0)
eng.set_debug(True)
batch = eng.upload(wl.summands)
res = eng.krp_sum(batch, wl.weights, wl.widths, wl.seed, 1e-6, None)
inter = res.intermediates()
out = res.to_tucker()
np.savez(sys.argv[1], y0=inter["y"][0], y1=inter["y"][1], y2=inter["y"][2], h=inter["h"], ranks=np.array(out.ranks),
         core=out.dense_core(), f0=out.factors[0])
print("saved", sys.argv[1], out.ranks, flush=True)
