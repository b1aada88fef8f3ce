"""Ozaki engine timing: stage A/E orientation (Fᵀ B) vs stage C orientation (A Btᵀ), 8192 × 8192 × 64."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13532_b200 import tucksum as T  # noqa: E402

eng = T.Engine(0)
rng = np.random.default_rng(0)
f = np.asfortranarray(rng.standard_normal((8192, 8192)) / 90.0)
b = np.asfortranarray(rng.standard_normal((8192, 64)))
bt = np.asfortranarray(b.T)
print("tn ms", ["%.4f" % eng.ozaki_gemm(f, b)[1] for _ in range(3)], flush=True)
print("nt ms", ["%.4f" % eng.ozaki_gemm_nt(f, bt)[1] for _ in range(3)], flush=True)
