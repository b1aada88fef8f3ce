"""Times the tridiagonalization eigensolver (ts_sym_eig_tri) against the Jacobi
kernel (ts_sym_eig) on Gram matrices of the configs' sizes; reports errors vs
numpy and whether the acceptance check rejected."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2603_13532_b200 import tucksum as T

eng = T.Engine(0)
for n, decay in [(26, 0.05), (40, 0.1), (50, 0.05), (64, 0.0), (64, 0.01), (64, 0.2)]:
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, 4 * n)) * (10.0 ** (-decay * np.arange(n)))[:, None]
    c = x @ x.T
    ref = np.linalg.eigvalsh(c)[::-1]
    out = {"n": n, "decay": decay}
    for name, fn in (("tri", eng.sym_eig_tri), ("jacobi", eng.sym_eig)):
        ts = []
        for _ in range(5):
            vals, vecs, extra, ms = fn(c)
            ts.append(ms)
        out[name] = {"us": 1e3 * min(ts), "max_eig_err_rel": float(np.max(np.abs(vals - ref)) / ref[0]),
                     "orth": float(np.linalg.norm(vecs.T @ vecs - np.eye(n))),
                     "resid_rel": float(np.linalg.norm(vecs @ np.diag(vals) @ vecs.T - c) / np.linalg.norm(c)),
                     ("rejected" if name == "tri" else "sweeps"): extra}
    if os.environ.get("TS_EIG_PROFILE"):
        import ctypes as C
        prof = (C.c_longlong * 17)()
        T.lib().ts_debug_eig_profile(prof)
        out["tri_phase_cycles"] = {"tridiag": prof[10], "bisect": prof[11], "invit": prof[12], "cluster": prof[13],
                                   "backtr": prof[14], "check_out": prof[15]}
    print(json.dumps(out))
