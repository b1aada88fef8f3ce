"""The eigensolver test matrices (tests/test_gpu_parity.py::test_sym_eig_tri_matches_oracle), one line each."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
from paper_2603_13532_b200 import tucksum as T  # noqa: E402

cases = []
for n, seed in [(1, 0), (2, 1), (3, 2), (6, 3), (26, 4), (40, 5), (50, 6), (64, 7)]:
    a = O.gaussian_matrix(2 * n, n, (18, seed))
    cases.append(a.T @ a)
rng = np.random.default_rng(3)
for n, decay in [(64, 0.2), (64, 0.5), (26, 1.0)]:
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    cases.append((q * 10.0 ** (-decay * np.arange(n))) @ q.T)
b = O.gaussian_matrix(64, 10, (19, 1))
cases.append(b @ b.T)
q, _ = np.linalg.qr(rng.standard_normal((48, 48)))
lam = np.repeat([3.0, 2.0, 1.0, 0.5], 12)
cases.append((q * lam) @ q.T)
eng = T.Engine(0)
for ci, c in enumerate(cases):
    n = c.shape[0]
    vals, vecs, rej, ms = eng.sym_eig_tri(c)
    ov, _ = O.sym_eig(c)
    scale = max(abs(ov[0]), 1e-300)
    print(ci, n, "rej", rej, "valerr %.2e (tol %.1e)" % (np.max(np.abs(vals - ov)) / scale, 1e-13 * max(1, n / 8)),
          "orth %.2e" % np.linalg.norm(vecs.T @ vecs - np.eye(n)),
          "rec %.2e" % (np.linalg.norm(vecs @ np.diag(vals) @ vecs.T - c) / np.linalg.norm(c)), "ms %.3f" % ms, flush=True)
eng.close()
