"""Debug/timing probe of the generic-width eigensolver (ts_sym_eig, n > 96 → wide.cu)."""
import os
import sys

import numpy as np

os.environ.setdefault("TS_DEBUG_BOSJ", "1")
sys.path.insert(0, ".")
import oracle as O  # noqa: E402
from paper_2603_13532_b200 import tucksum as T  # noqa: E402

eng = T.Engine(0)
for n in [26, 64, 96, 97, 128, 200]:
    a = O.gaussian_matrix(2 * n, n, (171, n))
    c = a.T @ a
    vals, vecs, sweeps, ms = eng.sym_eig(c)
    ov, _ = O.sym_eig(c)
    print(n, "sweeps", sweeps, "ms %.3f" % ms, "val err %.2e" % (np.max(np.abs(vals - ov)) / ov[0]),
          "orth %.2e" % np.linalg.norm(vecs.T @ vecs - np.eye(n)),
          "resid %.2e" % (np.linalg.norm(vecs @ np.diag(vals) @ vecs.T - c) / np.linalg.norm(c)), flush=True)
eng.close()
