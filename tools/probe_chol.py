"""Phase clocks of chol_inv_kernel.

Build an instrumented library with TS_NVCC_EXTRA=-DTS_CHOL_PROBE, point
TUCKSUM_LIB at it, and run: prints the clocks of CTA 0 of the last launch
(Cholesky → inverse → store)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_13532_b200 import tucksum as T
from paper_2603_13532_b200 import workloads as W

eng = T.Engine(0)
wl = W.make_workload(int(os.environ.get("PROBE_CFG", "5")), K=16)
batch = eng.upload(wl.summands)
for _ in range(3):
    res = eng.krp_sum(batch, wl.weights, wl.widths, wl.seed, wl.eps, wl.cap)
t = (C.c_longlong * 8)()
T.lib().tsi_read_chol_probe(t)
print(json.dumps({"cholesky_clk": t[1] - t[0], "inverse_clk": t[2] - t[1], "store_clk": t[4] - t[2],
                  "n": wl.widths[0]}))
