"""Times the device symmetric Jacobi eigensolver on Gram matrices with decaying spectra.

Run with TS_EIG_PROFILE=1 for the values kernel's per-phase clock totals."""
import ctypes as C
import json
import os
import sys

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
    prof = (C.c_longlong * 8)()
    T.lib().ts_debug_eig_profile(prof)
    rounds = max(1, prof[4])
    print(json.dumps({"n": n, "decay": decay, "sweeps": sw, "ms": ms, "max_eig_err": err,
                      "rounds": sw * (n + (n & 1) - 1),
                      "us_per_round": 1e3 * ms / max(1, sw * (n + (n & 1) - 1)),
                      "loop_cycles_per_round": prof[0] / rounds,
                      "pivot_chain": prof[1] / rounds, "worker0_chain": prof[2] / rounds,
                      "sweep_tail_per_round": prof[3] / rounds}))
