"""One call of the stage-G tridiagonalisation eigensolver at n = 64 (ncu target)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13532_b200 import tucksum as T  # noqa: E402

rng = np.random.default_rng(1)
m = rng.standard_normal((64, 4096))
eng = T.Engine(0)
for _ in range(2):
    vals, vecs, rej, ms = eng.sym_eig_tri(m @ m.T)
print("ms", ms, "rejected", rej)
eng.close()
