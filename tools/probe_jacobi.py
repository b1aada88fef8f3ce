"""Times the device symmetric Jacobi eigensolver on Gram matrices with decaying spectra.

Run with TS_EIG_PROFILE=<mode> for the values kernel's loop clocks per round;
mode bits 4 / 8 skip the worker updates / the rotation formation (timing ablations)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2603_13532_b200 import tucksum as T

eng = T.Engine(0)
cases = [(64, 0.0), (64, 0.05), (64, 0.2), (50, 0.2), (26, 0.1), (96, 0.1)]
if os.environ.get("PROBE_NS"):
    cases = [(int(x), 0.1) for x in os.environ["PROBE_NS"].split(",")]
for n, decay in cases:
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 10.0 ** (-decay * np.arange(n))
    c = (q * lam) @ q.T
    for _ in range(2):
        vals, vecs, sw, ms = eng.sym_eig(c)
    err = np.max(np.abs(np.sort(vals)[::-1] - np.sort(lam)[::-1]))
    prof = (C.c_longlong * 17)()
    T.lib().ts_debug_eig_profile(prof)
    rounds = max(1, prof[4])
    print(json.dumps({"n": n, "decay": decay, "sweeps": sw, "ms": ms, "max_eig_err": err,
                      "rounds": sw * (n + (n & 1) - 1),
                      "us_per_round": 1e3 * ms / max(1, sw * (n + (n & 1) - 1)),
                      "loop_cycles_per_round": prof[0] / rounds,
                      "sweep_tail_cycles": prof[3] / max(1, sw),
                      "round_index_clocks": [prof[8 + i] for i in range(9)]}))
