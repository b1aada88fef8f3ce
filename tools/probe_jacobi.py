"""Times the device symmetric Jacobi eigensolver on Gram matrices with decaying spectra."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2603_13532_b200 import tucksum as T
eng = T.Engine(0)
for n, decay in [(64, 0.0), (64, 0.05), (64, 0.2), (50, 0.2), (26, 0.1), (96, 0.1)]:
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 10.0 ** (-decay * np.arange(n))
    c = (q * lam) @ q.T
    for _ in range(2):
        vals, vecs, sw, ms = eng.sym_eig(c)
    err = np.max(np.abs(np.sort(vals)[::-1] - np.sort(lam)[::-1]))
    import ctypes as C
    prof = (C.c_longlong * 4)()
    T.lib().ts_debug_eig_profile(prof)
    print(json.dumps({"n": n, "decay": decay, "sweeps": sw, "ms": ms, "max_eig_err": err,
                      "cycles_rot_bar_pass_bar": [int(x) for x in prof],
                      "rounds": sw * (n + (n & 1) - 1)}))
