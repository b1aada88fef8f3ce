"""Stage-A-sized Ozaki GEMM (3 modes' worth of columns in one launch: k = 8192,
m = 3·8192, n = 64) vs the DMMA stage-A time (0.77 ms incl. split-K reduce)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13532_b200 import tucksum as T  # noqa: E402

eng = T.Engine(0)
rng = np.random.default_rng(0)
f = np.asfortranarray(rng.standard_normal((8192, 3 * 8192)) / 90.0)
b = np.asfortranarray(rng.standard_normal((8192, 64)))
ts = [eng.ozaki_gemm(f, b)[1] for _ in range(4)]
print("stage-A-sized ozaki ms", ["%.4f" % t for t in ts], "GB/s %.0f" % (f.nbytes / min(ts) / 1e6), flush=True)
eng.close()
