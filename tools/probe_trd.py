"""A/B of the stage-G eigensolvers on the GPU: Jacobi (ts_sym_eig) vs the
tridiagonalisation solver (ts_sym_eig_tri → eig_trd.cu): time, eigenvalue error
vs the oracle, orthogonality, residual, rejection flag."""
import ctypes as C
import json
import os
import sys

os.environ.setdefault("TS_EIG_PROFILE", "1")

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
from paper_2603_13532_b200 import tucksum as T  # noqa: E402

eng = T.Engine(0)
rng = np.random.default_rng(5)
out = []
cases = []
for n in (26, 40, 48, 64):
    a = O.gaussian_matrix(2 * n, n, (21, n))
    cases.append((f"gram{n}", a.T @ a))
q = 64
idx = np.indices((q, q, q)).sum(0)
for name, sc in [("h_pow2_8", 2.0 ** (-idx / 8)), ("h_flat", np.ones((q, q, q))), ("h_pow10_12", 10.0 ** (-idx / 12))]:
    h = rng.standard_normal((q, q, q)) * sc
    m = h.reshape(q, -1)
    cases.append((name, m @ m.T))
for name, c in cases:
    n = c.shape[0]
    ov, _ = O.sym_eig(c)
    row = {"case": name, "n": n}
    for solver in ("jacobi", "trd"):
        ts = []
        for _ in range(5):
            if solver == "jacobi":
                vals, vecs, sw, ms = eng.sym_eig(c)
                rej = False
            else:
                vals, vecs, rej, ms = eng.sym_eig_tri(c)
                prof = (C.c_longlong * 22)()
                T.lib().ts_debug_eig_profile(prof)
                row["trd_phase_cycles"] = list(prof)[10:16]
                row["trd_sub"] = {"load": prof[9], "loop_start": prof[17], "loop_end": prof[16], "refl_group": prof[19], "matvec_w15": prof[20], "update_w15": prof[21]}
            ts.append(ms)
        row[solver] = {"ms": float(np.median(ts)), "rejected": bool(rej),
                       "eig_err_rel": float(np.max(np.abs(vals - ov)) / ov[0]),
                       "orth": float(np.linalg.norm(vecs.T @ vecs - np.eye(n))),
                       "resid_rel": float(np.linalg.norm(c @ vecs - vecs * vals) / ov[0])}
    out.append(row)
    print(json.dumps(row), flush=True)
eng.close()
