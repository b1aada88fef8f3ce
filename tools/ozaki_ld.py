"""Ozaki GEMM timing vs the leading dimension of F (power-of-two strides vs padded)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13532_b200 import tucksum as T  # noqa: E402

eng = T.Engine(0)
rng = np.random.default_rng(0)
for k in (8192, 8200, 8256):
    f = np.asfortranarray(rng.standard_normal((k, 8192)) / 90.0)
    b = np.asfortranarray(rng.standard_normal((k, 64)))
    ts = [eng.ozaki_gemm(f, b)[1] for _ in range(3)]
    print("k", k, "ms %.4f" % min(ts), "GB/s %.0f" % (k * 8192 * 8 / min(ts) / 1e6), flush=True)
eng.close()
