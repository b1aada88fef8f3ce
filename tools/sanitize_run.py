"""Workload for compute-sanitizer: one config-1 KRP sum (TMA/mbarrier GEMMs,
krp3, ttm3, CholeskyQR2 on the side stream, the tridiagonalisation eigensolver),
one config-3 sum (Householder TSQR fallback, accurate ST-HOSVD path: TSQR +
one-sided Jacobi SVD), the Jacobi eigensolver, the Kron sketch and Lazy
rounding on small inputs — each checked against the oracle."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
from paper_2603_13532_b200 import tucksum as T  # noqa: E402
from paper_2603_13532_b200.workloads import make_workload  # noqa: E402

eng = T.Engine(0)
eng.set_graphs(False)
for cfg, K in ((1, None), (3, 6)):
    wl = make_workload(cfg, K=K)
    b = eng.upload(wl.summands)
    for _ in range(2):  # second call: speculative path (first may be synchronous)
        r = eng.krp_sum(b, wl.weights, wl.widths, wl.seed, wl.eps, wl.cap)
        out = r.to_tucker()
        r.free()
    ref, _ = O.krp_sum(wl.summands, wl.weights, wl.widths, (wl.seed.seed, wl.seed.stream), wl.eps, cap=wl.cap)
    assert out.ranks == ref.ranks and O.rel_error_to_sum(out, [ref], [1.0]) <= 1e-10
    kw = T.kron_sketch_dims(wl.widths, wl.dims)
    eng.krp_sum(b, wl.weights, kw, wl.seed, wl.eps, wl.cap, T.Strategy.Kron).free()
    b.free()
wl = make_workload(1)
b = eng.upload(wl.summands)
eng.lazy_sum(b, wl.weights, 0.0, wl.cap).free()
b.free()
c = O.gaussian_matrix(80, 40, (3, 4))
eng.sym_eig(c.T @ c)
eng.sym_eig_tri(c.T @ c)
eng.close()
print("sanitize workload ok")
