"""Ozaki GEMM on config 5's own operands (F_0 and Ω_0) vs numpy."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13532_b200 import tucksum as T  # noqa: E402
from paper_2603_13532_b200.workloads import make_workload  # noqa: E402

wl = make_workload(5)
eng = T.Engine(0)
F0 = np.asfortranarray(wl.slabs[0])
om = T.gaussian_matrix(8192, 64, wl.seed.substream(0))
out, ms = eng.ozaki_gemm(F0, om)
ref = F0.T @ om
print("F0 shape", F0.shape, "rel fro", np.linalg.norm(out - ref) / np.linalg.norm(ref), "ms", ms, flush=True)
bad = np.argwhere(np.abs(out - ref) > 1e-8 * np.abs(ref).max())
print("bad entries", len(bad), bad[:10].tolist(), flush=True)
for m in (0, 1, 127, 128, 4096, 8191):
    print(m, np.abs(out[m] - ref[m]).max(), np.abs(ref[m]).max())
