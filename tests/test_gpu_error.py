"""Device norms, inner products and the error to the exact sum (SURVEY.md §8(f)
row 4; reference tucker_norm / tucker_inner / tucker_rel_error,
src/tucker.cpp:132-181,298-303) against dense oracles, the CPU oracle and the
reference's assertions (proj/tests/test_tucker_core.cpp:113-134,253-258)."""
import numpy as np
import pytest

import oracle as O
from helpers import random_tucker
from paper_2603_13532_b200 import tucksum as T
from paper_2603_13532_b200.workloads import make_workload

pytestmark = pytest.mark.gpu


def test_norm_and_inner_match_dense(engine):
    """test_tucker_core.cpp:113-134."""
    x = random_tucker([6, 5, 4], [3, 2, 3], (22, 0))
    dx = O.reconstruct(x)
    assert abs(T.tucker_norm(x, engine) - np.linalg.norm(dx)) <= 1e-12 * np.linalg.norm(dx)
    q = [O.qr_econ(f)[0] for f in x.factors]
    ortho = T.TuckerTensor(x.dense_core(), q)
    assert abs(T.tucker_norm(ortho, engine) - np.linalg.norm(x.dense_core())) <= 1e-12 * np.linalg.norm(x.dense_core())
    y = random_tucker([6, 5, 4], [2, 2, 2], (23, 1))
    dy = O.reconstruct(y)
    want = float(np.sum(dx * dy))
    assert abs(T.tucker_inner(x, y, engine) - want) <= 1e-12 * abs(want)
    assert abs(T.tucker_inner(x, x, engine) - np.sum(dx * dx)) <= 1e-12 * np.sum(dx * dx)
    z = random_tucker([6, 5, 5], [2, 2, 2], (23, 2))
    with pytest.raises(ValueError):
        T.tucker_inner(x, z, engine)


def test_exact_cancellation_survives_orthogonalized_norm(engine):
    """test_tucker_core.cpp:253-258."""
    x = random_tucker([7, 6, 5], [3, 3, 3], (33, 0))
    assert T.tucker_norm(T.tucker_axby(1.0, x, -1.0, x), engine) <= 1e-14 * T.tucker_norm(x, engine)
    assert T.tucker_rel_error(x, x, engine) <= 1e-14


def test_weighted_inner_over_batches_matches_oracle(engine):
    """Σ_ab w_a w_b <X_a, X_b> over device batches (block cores included) = ‖formal_sum‖²."""
    a = [random_tucker([20, 18, 16], [3, 4, 2], (700, i)) for i in range(5)]
    xs = a[:3] + [T.tucker_axby(0.5, a[3], -2.0, a[4])]
    ws = [1.0, -0.5, 0.7, 1.3]
    ys = [random_tucker([20, 18, 16], [2, 2, 3], (701, i)) for i in range(3)]
    wy = [0.3, 1.0, -1.0]
    bx, by = engine.upload(xs), engine.upload(ys)
    try:
        ss = engine.inner(bx, ws, bx, ws)
        xy = engine.inner(bx, ws, by, wy)
        nrm = engine.tucker_norm(bx, ws)
    finally:
        bx.free()
        by.free()
    sx, sy = T.formal_sum(xs, ws), T.formal_sum(ys, wy)
    want_ss = O.tucker_norm(sx) ** 2
    assert abs(ss - want_ss) <= 1e-12 * want_ss
    assert abs(nrm - np.sqrt(want_ss)) <= 1e-12 * np.sqrt(want_ss)
    want_xy = O.tucker_inner(sx, sy)
    assert abs(xy - want_xy) <= 1e-11 * np.sqrt(want_ss) * O.tucker_norm(sy)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_device_error_to_sum_matches_oracle(engine, cfg):
    """ts_rel_error_to_sum equals the oracle's error to the exact sum (3 significant digits)."""
    wl = make_workload(cfg)
    batch = engine.upload(wl.summands)
    try:
        res = engine.krp_sum(batch, wl.weights, wl.widths, wl.seed, wl.eps, wl.cap)
        e_dev = engine.rel_error_to_sum(res, batch, wl.weights)
        out = res.to_tucker()
        res.free()
    finally:
        batch.free()
    e_ref = O.rel_error_gram(out, wl.summands, wl.weights, O.num_threads()) if cfg == 4 else \
        O.rel_error_to_sum(out, wl.summands, wl.weights)
    assert abs(e_dev - e_ref) <= 5e-4 * e_ref, (e_dev, e_ref)
