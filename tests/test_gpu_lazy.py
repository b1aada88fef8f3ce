"""Lazy rounding and the Eager fold on the sm_100a path (
reference tucker_rounding src/tucker.cpp:285-296, lazy_sum / eager_sum
src/sketch.cpp:48-64): parity with the CPU oracle and the reference's own
assertions (proj/tests/test_tucker_core.cpp, test_sketch_sum.cpp)."""
import numpy as np
import pytest

import oracle as O
from helpers import cancellation_instance, dense_rel_error, dense_weighted_sum, random_tucker
from paper_2603_13532_b200 import tucksum as T

pytestmark = pytest.mark.gpu

PARITY = 1e-10


@pytest.mark.parametrize("dims,ranks,K,cap", [
    ([64, 64, 64], [8, 8, 8], 4, None),
    ([512, 512, 512], [20, 20, 20], 4, [30, 30, 30]),
    ([16, 12, 10, 9], [2, 3, 2, 2], 3, None),
    ([30, 25], [4, 3], 5, None),
    ([9, 40, 40], [3, 5, 5], 6, None),   # mode 0: stacked rank 18 > 9 rows
])
def test_lazy_parity_with_oracle(engine, dims, ranks, K, cap):
    xs = [random_tucker(dims, ranks, (680 + len(dims), i)) for i in range(K)]
    ws = list(np.random.default_rng(K).uniform(-1.5, 1.5, size=K))
    for eps in (1e-9, 0.0):
        ref = O.lazy_sum(xs, ws, eps, cap)
        batch = engine.upload(xs)
        try:
            res = engine.lazy_sum(batch, ws, eps, cap)
            out = res.to_tucker()
            res.free()
        finally:
            batch.free()
        assert out.ranks == ref.ranks
        assert O.rel_error_to_sum(out, [ref], [1.0]) <= PARITY
        e_gpu, e_ref = O.rel_error_to_sum(out, xs, ws), O.rel_error_to_sum(ref, xs, ws)
        assert abs(e_gpu - e_ref) <= 5e-4 * max(e_ref, 1e-300) or abs(e_gpu - e_ref) <= 1e-13


def test_rounding_honors_budget(engine):
    """test_tucker_core.cpp:208-220."""
    x = random_tucker([8, 7, 6], [5, 4, 5], (29, 0))
    dense = O.reconstruct(x)
    for tau in (1e-1, 1e-4, 1e-8):
        r = T.tucker_rounding(x, tau, engine)
        assert np.linalg.norm(O.reconstruct(r) - dense) <= tau * np.linalg.norm(dense) + 1e-13 * np.linalg.norm(dense)
        for u in r.factors:
            assert np.linalg.norm(u.T @ u - np.eye(u.shape[1])) <= 1e-12


def test_rounding_recovers_copies_floor_and_zero(engine):
    """test_tucker_core.cpp:222-251."""
    x = random_tucker([9, 8, 7], [3, 2, 4], (30, 0))
    r = T.tucker_rounding(T.formal_sum([x] * 4, [0.25] * 4), 1e-10, engine)
    assert r.ranks == x.ranks
    assert O.rel_error_to_sum(r, [x], [1.0]) <= 1e-9
    u0 = O.gaussian_matrix(6, 2, (31, 0))
    f = [np.concatenate([u0, u0[:, :1]], axis=1), O.gaussian_matrix(5, 2, (31, 1)), O.gaussian_matrix(4, 2, (31, 2))]
    y = T.TuckerTensor(O.gaussian_matrix(12, 1, (31, 3))[:, 0].reshape((3, 2, 2), order="F"), f)
    r = T.tucker_rounding(y, 0.0, engine)
    assert r.ranks == [2, 2, 2]
    assert O.rel_error_to_sum(r, [y], [1.0]) <= 1e-12
    zero = T.TuckerTensor(np.zeros((2, 2)), [O.gaussian_matrix(4, 2, (32, 0)), O.gaussian_matrix(3, 2, (32, 1))])
    r = T.tucker_rounding(zero, 1e-6, engine)
    assert r.ranks == [1, 1]
    assert O.tucker_norm(r) == 0.0


def test_random_sums_lazy_and_eager(engine):
    """test_sketch_sum.cpp:266-299 (Lazy ≤ 1e-6, Eager ≤ 4·5·1e-6)."""
    rng = np.random.Generator(np.random.MT19937(907))
    for trial in range(20):
        xs, ws = [], []
        for i in range(5):
            ranks = [int(v) for v in rng.integers(1, 4, size=3)]
            xs.append(random_tucker([14, 11, 9], ranks, (1000 + trial, i)))
            ws.append((1.0 if rng.integers(0, 2) == 0 else -1.0) * rng.uniform(0.5, 2.0))
        ref = dense_weighted_sum(xs, ws)
        req = T.SumRequest(xs, ws, 1e-6, 5, T.Strategy.Lazy, T.RngSeed(42, trial))
        lazy = T.round_sum(req, engine=engine)
        assert dense_rel_error(lazy, ref) <= 1e-6
        oref = O.lazy_sum(xs, ws, 1e-6)
        assert lazy.ranks == oref.ranks and O.rel_error_to_sum(lazy, [oref], [1.0]) <= PARITY
        req.strategy = T.Strategy.Eager
        assert dense_rel_error(T.round_sum(req, engine=engine), ref) <= 4 * 5 * 1e-6


def test_dispatcher_lazy_and_eager(engine):
    """test_sketch_sum.cpp:470-512."""
    xs = [random_tucker([10, 9, 8], [2, 3, 2], (81, i)) for i in range(3)]
    ws = [1.0, -0.5, 2.0]
    req = T.SumRequest(xs, ws, 1e-8, 3, T.Strategy.Lazy, T.RngSeed(81, 9))
    a = T.round_sum(req, engine=engine)
    b = T.tucker_rounding(T.formal_sum(xs, ws), 1e-8, engine)
    assert a.ranks == b.ranks
    assert all(np.array_equal(x, y) for x, y in zip(a.factors, b.factors))
    assert np.array_equal(a.dense_core(), b.dense_core())
    req.strategy = T.Strategy.Eager
    stats = T.SumStats()
    eager = T.round_sum(req, None, stats, engine=engine)
    assert eager.dims == xs[0].dims
    assert len(stats.eager_rank_trace) == 2
    solo = T.round_sum(T.SumRequest([xs[0]], [-2.5], 1e-8, 3, T.Strategy.Eager, T.RngSeed(81, 10)), engine=engine)
    assert solo.ranks == xs[0].ranks
    assert np.array_equal(solo.factors[0], xs[0].factors[0])
    assert np.array_equal(solo.blocks[0].data, -2.5 * xs[0].blocks[0].data)


def test_eager_cancellation_loses_quiet_components(engine):
    """test_sketch_sum.cpp:560-598: the eager fold truncates the quiet target
    components away (error ≥ 0.05) and its intermediate ranks swell."""
    xs, ws, target = cancellation_instance(40, 10, (107, 0))
    ref = O.reconstruct(target)
    stats = T.SumStats()
    eager = T.round_sum(T.SumRequest(xs, ws, 1e-6, 2, T.Strategy.Eager, T.RngSeed(107, 1)), None, stats,
                        engine=engine)
    assert dense_rel_error(eager, ref) >= 0.05
    krp = T.round_sum(T.SumRequest(xs, ws, 1e-6, 2, T.Strategy.Krp, T.RngSeed(107, 1)), engine=engine)
    assert max(max(r) for r in stats.eager_rank_trace) > 2 * max(krp.ranks)


def test_lazy_rejects_bad_tolerance(engine):
    """Stacked ranks beyond 96 are supported (tests/test_gpu_wide.py); a negative
    tolerance is still the reference's invalid_argument."""
    xs = [random_tucker([20, 20, 20], [3, 3, 3], (90, i)) for i in range(3)]
    batch = engine.upload(xs)
    try:
        with pytest.raises(ValueError):
            engine.lazy_sum(batch, [1.0] * 3, -1.0)
    finally:
        batch.free()