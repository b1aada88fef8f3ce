"""One large Ozaki GEMM (ncu target): k = m = 8192, n = 64."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13532_b200 import tucksum as T  # noqa: E402

eng = T.Engine(0)
rng = np.random.default_rng(0)
f = np.asfortranarray(rng.standard_normal((8192, 8192)) / 90.0)
b = np.asfortranarray(rng.standard_normal((8192, 64)))
for _ in range(2):
    out, ms = eng.ozaki_gemm(f, b)
print("ms", ms)
eng.close()
