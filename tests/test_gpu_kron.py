"""Parity of the Kronecker-sketch variant (reference
kron_sum → sketched_sum(krp=false), src/sketch.cpp:66-181,364-366) on the
sm_100a path, through the C ABI, against the CPU oracle and the reference's own
Kron test assertions (proj/tests/test_sketch_sum.cpp).

Same bar as the KRP path: factors × core within 1e-10 relative Frobenius error
of the oracle on identical inputs and Ω, same output ranks, and the same
approximation error to the exact sum to 3 significant digits.
"""
import numpy as np
import pytest

import oracle as O
from helpers import (cancellation_instance, dense_rel_error, dense_weighted_sum, random_tucker, shared_subspace,
                     sub)
from paper_2603_13532_b200 import tucksum as T

pytestmark = pytest.mark.gpu

PARITY = 1e-10


def gpu_kron(engine, xs, ws, widths, seed, eps, cap=None, debug=False):
    engine.set_debug(debug)
    batch = engine.upload(xs)
    try:
        res = engine.kron_sum(batch, ws, widths, T.RngSeed(*seed), eps, cap)
        out = res.to_tucker()
        inter = res.intermediates() if debug else None
        res.free()
    finally:
        batch.free()
        engine.set_debug(False)
    return out, inter


def check_kron(engine, xs, ws, widths, seed, eps, cap=None):
    ref, info = O.kron_sum(xs, ws, widths, seed=seed, eps=eps, cap=cap, threads=8, intermediates=True)
    out, inter = gpu_kron(engine, xs, ws, widths, seed, eps, cap, debug=True)
    for n in range(len(widths)):
        assert np.array_equal(inter["omega"][n], info["omega"][n])  # same Ω (bitwise)
        assert inter["y"][n].shape == info["y"][n].shape
        assert np.linalg.norm(inter["y"][n] - info["y"][n]) <= 1e-12 * np.linalg.norm(info["y"][n])
    assert out.ranks == ref.ranks
    assert O.rel_error_to_sum(out, [ref], [1.0]) <= PARITY
    e_gpu, e_ref = O.rel_error_to_sum(out, xs, ws), O.rel_error_to_sum(ref, xs, ws)
    assert abs(e_gpu - e_ref) <= 5e-4 * max(e_ref, 1e-300) or abs(e_gpu - e_ref) <= 1e-13
    return out, ref


@pytest.mark.parametrize("dims,ranks,K,widths,cap", [
    ([64, 64, 64], [8, 8, 8], 4, [5, 5, 6], [16, 16, 16]),          # config-1 shape, Kron widths
    ([512, 512, 512], [20, 20, 20], 16, [7, 7, 7], [30, 30, 30]),   # config-2 shape
    ([20, 17, 15], [3, 4, 2], 4, [3, 3, 4], None),
    ([16, 12, 10, 9], [2, 3, 2, 2], 3, [2, 2, 3, 2], None),         # order 4
    ([30, 25], [4, 3], 5, [6, 7], None),                             # order 2
    ([9, 40, 40], [3, 5, 5], 6, [4, 4, 4], None),                    # wide Y_0 (16 columns > 9 rows)
])
def test_kron_parity_with_oracle(engine, dims, ranks, K, widths, cap):
    xs = [random_tucker(dims, ranks, (660 + len(dims), i)) for i in range(K)]
    ws = list(np.random.default_rng(K).uniform(-1.5, 1.5, size=K))
    for eps in (1e-9, 0.0):
        check_kron(engine, xs, ws, widths, (660, 5), eps, cap)


def test_kron_block_core_summands(engine):
    """Formal-sum summands (super-diagonal block cores, tucker_axby) as extra atoms."""
    a = [random_tucker([18, 14, 11], [3, 2, 4], (670, i)) for i in range(4)]
    xs = [T.tucker_axby(0.5, a[0], -1.0, a[1]), T.tucker_axby(2.0, a[2], 1.0, a[3]), a[0]]
    check_kron(engine, xs, [1.0, -0.7, 0.3], [3, 4, 3], (670, 9), 1e-10)


def test_kron_opposite_summands_annihilate(engine):
    """test_sketch_sum.cpp:186-198 (Kron branch)."""
    x = random_tucker([12, 10, 8], [3, 4, 2], (21, 3))
    out = T.kron_sum(T.SumRequest([x, x], [1.0, -1.0], 1e-6, 5, T.Strategy.Kron, T.RngSeed(21, 4)), engine=engine)
    assert O.tucker_norm(out) <= 1e-12 * O.tucker_norm(x)


def test_kron_single_summand_passes_through(engine):
    """test_sketch_sum.cpp:200-219 (Kron branch)."""
    x = random_tucker([15, 12, 18], [4, 3, 5], (31, 0))
    out = T.kron_sum(T.SumRequest([x], [1.0], 1e-10, 2, T.Strategy.Kron, T.RngSeed(31, 1)), engine=engine)
    assert O.rel_error_to_sum(out, [x], [1.0]) <= 1e-10
    assert dense_rel_error(out, O.reconstruct(x)) <= 1e-10


def test_kron_shared_subspace_recovers_latent_ranks(engine):
    """test_sketch_sum.cpp:221-264 (Kron branch) + the Kron plan vs the oracle's."""
    seed = (51, 0)
    xs = shared_subspace(60, 4, 10, 20, seed)
    ws = [1.0] * 20
    req = T.SumRequest(xs, ws, 1e-6, 2, T.Strategy.Kron, T.RngSeed(*sub(seed, 77)))
    stats = T.SumStats()
    out = T.round_sum(req, None, stats, engine=engine)
    assert out.ranks == [10] * 4
    assert dense_rel_error(out, dense_weighted_sum(xs, ws)) <= 1e-10
    eff, tg, wd = O.effective_subrank(xs, ws, 1e-6, 2, strategy="kron")
    assert stats.plan.strategy == T.Strategy.Kron
    assert stats.plan.effective_ranks == eff and stats.plan.targets == tg and stats.plan.mode_sketch_dims == wd


def test_kron_random_sums_match_dense_and_cpu_oracle(engine):
    """test_sketch_sum.cpp:266-299 (Kron branch, 20 trials) + parity with the oracle, plans included."""
    rng = np.random.Generator(np.random.MT19937(907))
    dims = [14, 11, 9]
    for trial in range(20):
        xs, ws = [], []
        for i in range(5):
            ranks = [int(x) for x in rng.integers(1, 4, size=3)]
            xs.append(random_tucker(dims, ranks, (1000 + trial, i)))
            ws.append((1.0 if rng.integers(0, 2) == 0 else -1.0) * rng.uniform(0.5, 2.0))
        ref = dense_weighted_sum(xs, ws)
        out = T.round_sum(T.SumRequest(xs, ws, 1e-6, 5, T.Strategy.Kron, T.RngSeed(42, trial)), engine=engine)
        assert dense_rel_error(out, ref) <= 1e-6
        oref, _ = O.kron_sum(xs, ws, None, seed=(42, trial), eps=1e-6, oversampling=5)
        assert out.ranks == oref.ranks
        assert O.rel_error_to_sum(out, [oref], [1.0]) <= PARITY


def test_kron_shared_subspaces_across_seeds(engine):
    """test_sketch_sum.cpp:301-347 (Kron branch)."""
    rng = np.random.Generator(np.random.MT19937(1310))
    dims = [18, 15, 12]
    for trial in range(20):
        seed = (2000 + trial, 0)
        xs = shared_subspace(dims, 3, 4, 8, seed, rank=2, core_salt=True)
        ws = list(rng.uniform(0.5, 1.5, size=8))
        out = T.kron_sum(T.SumRequest(xs, ws, 1e-8, 2, T.Strategy.Kron, T.RngSeed(*sub(seed, 9000))), engine=engine)
        assert out.ranks == [4, 4, 4]
        assert dense_rel_error(out, dense_weighted_sum(xs, ws)) <= 1e-8


def test_kron_paired_cancellation(engine):
    """test_sketch_sum.cpp:560-598 (Kron branch, ≤ 1e-9)."""
    xs, ws, target = cancellation_instance(40, 10, (107, 0))
    out = T.kron_sum(T.SumRequest(xs, ws, 1e-6, 2, T.Strategy.Kron, T.RngSeed(107, 1)), engine=engine)
    assert dense_rel_error(out, O.reconstruct(target)) <= 1e-9


def test_kron_dispatcher_bitwise(engine):
    """test_sketch_sum.cpp:470-489: round_sum(Kron) is kron_sum, bitwise."""
    xs = [random_tucker([10, 9, 8], [2, 3, 2], (81, i)) for i in range(3)]
    req = T.SumRequest(xs, [1.0, -0.5, 2.0], 1e-8, 3, T.Strategy.Kron, T.RngSeed(81, 9))
    a, b = T.round_sum(req, engine=engine), T.kron_sum(req, engine=engine)
    assert a.ranks == b.ranks
    assert all(np.array_equal(x, y) for x, y in zip(a.factors, b.factors))
    assert np.array_equal(a.dense_core(), b.dense_core())


def test_kron_rejects_bad_widths(engine):
    """Wide complements (C_n > 96) are supported (tests/test_gpu_wide.py); a zero width is invalid."""
    x = random_tucker([200, 200, 200], [3, 3, 3], (90, 0))
    batch = engine.upload([x])
    try:
        with pytest.raises(ValueError):
            engine.kron_sum(batch, [1.0], [3, 0, 3], T.RngSeed(1, 1), 1e-8)
    finally:
        batch.free()


def test_kron_cfg5_full_size_parity(engine):
    """BASELINE config 5 at full size through the Kron sketch (K = 256, n = 8192,
    widths = kron_sketch_dims(64-targets) = (8, 8, 8), cap 48): device vs CPU
    oracle on identical inputs and Ω — 1e-10 on factors × core, same ranks, and
    the same error to the exact sum to 3 significant digits (device error kernel
    vs the oracle's Gram-based error)."""
    from paper_2603_13532_b200.workloads import make_workload

    wl = make_workload(5)
    widths = T.kron_sketch_dims(wl.widths, wl.dims)
    assert widths == [8, 8, 8]
    seed = (wl.seed.seed, wl.seed.stream)
    threads = O.num_threads()
    ref, _ = O.kron_sum(wl.summands, wl.weights, widths, seed=seed, eps=wl.eps, cap=wl.cap, threads=threads)
    batch = engine.upload(wl.summands)
    try:
        res = engine.kron_sum(batch, wl.weights, widths, wl.seed, wl.eps, wl.cap)
        e_dev = engine.rel_error_to_sum(res, batch, wl.weights)
        out = res.to_tucker()
        res.free()
    finally:
        batch.free()
    assert out.ranks == ref.ranks == [48, 48, 48]
    assert O.rel_error_to_sum(out, [ref], [1.0]) <= PARITY
    e_ref = O.rel_error_gram(ref, wl.summands, wl.weights, threads)
    assert abs(e_dev - e_ref) <= 5e-4 * e_ref
