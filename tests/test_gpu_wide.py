"""Generic widths on the sm_100a path (wide.cu): sketch widths, Kron complement
widths, Lazy stacked ranks and plan stacks beyond the one-CTA kernels' 96
columns.  The reference has no width limit (Eigen HouseholderQR / BDCSVD /
SelfAdjointEigenSolver at any size, src/kernels.cpp:50-86); these tests hold
the wide paths to the same parity bar as the rest: factors × core within 1e-10
of the CPU oracle on identical inputs and Ω, same ranks, same error to the
exact sum to 3 significant digits.  The plan-stage case is the paper's
synthetic-lowrank setting (reference bench defaults, src/bench.cpp:186-196,
include/tucksum/bench.hpp:42-48: 4 modes, latent rank 10, up to 100 rank-1
summands, so Σ_k r_n^(k) = 100 > 96)."""
import numpy as np
import pytest

import oracle as O
from helpers import random_tucker, shared_subspace
from paper_2603_13532_b200 import tucksum as T

pytestmark = pytest.mark.gpu

PARITY = 1e-10


def _err_same(out, ref, xs, ws):
    e_gpu, e_ref = O.rel_error_to_sum(out, xs, ws), O.rel_error_to_sum(ref, xs, ws)
    assert abs(e_gpu - e_ref) <= 5e-4 * max(e_ref, 1e-300) or abs(e_gpu - e_ref) <= 1e-13


@pytest.mark.parametrize("n", [97, 128, 200])
def test_sym_eig_wide_matches_oracle(engine, n):
    """Block one-sided Jacobi of a PSD Gram (n > 96): eigenvalues, orthogonality, residual."""
    a = O.gaussian_matrix(2 * n, n, (171, n))
    c = a.T @ a
    vals, vecs, sweeps, ms = engine.sym_eig(c)
    ov, _ = O.sym_eig(c)
    assert np.max(np.abs(vals - ov)) <= 1e-12 * ov[0]
    assert np.linalg.norm(vecs.T @ vecs - np.eye(n)) <= 1e-12
    assert np.linalg.norm(vecs @ np.diag(vals) @ vecs.T - c) <= 1e-12 * np.linalg.norm(c)
    assert 1 <= sweeps <= 40


def test_sym_eig_wide_graded_and_rank_deficient(engine):
    """Graded spectrum (10 decades) and an exactly rank-deficient Gram."""
    n = 120
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, (172, 0)))
    lam = 10.0 ** (-10.0 * np.arange(n) / (n - 1))
    c = (q * lam) @ q.T
    vals, vecs, _, _ = engine.sym_eig(c)
    assert np.max(np.abs(vals - lam)) <= 1e-13
    assert np.linalg.norm(vecs.T @ vecs - np.eye(n)) <= 1e-12
    b = O.gaussian_matrix(n, 30, (172, 1))
    c = b @ b.T  # rank 30
    vals, vecs, _, _ = engine.sym_eig(c)
    ov, _ = O.sym_eig(c)
    assert np.max(np.abs(vals - ov)) <= 1e-12 * ov[0]
    assert np.all(np.abs(vals[30:]) <= 1e-12 * ov[0])
    assert np.linalg.norm(vecs.T @ vecs - np.eye(n)) <= 1e-12


@pytest.mark.parametrize("s,eps,cap", [(100, 1e-9, None), (128, 1e-8, None), (128, 0.0, [60, 60, 60])])
def test_krp_wide_sketch_parity(engine, s, eps, cap):
    """KRP sketch width s > 96: stage D by BCGS2 + TSQR panels, stage G by the
    block one-sided Jacobi (fast Gram path and the accurate path on h_(k)ᵀ)."""
    dims, ranks, K = [300, 260, 220], [24, 20, 16], 8
    xs = [random_tucker(dims, ranks, (930, i)) for i in range(K)]
    ws = list(np.random.default_rng(930).uniform(-1.5, 1.5, size=K))
    seed = (930, 5)
    ref, _ = O.krp_sum(xs, ws, [s] * 3, seed, eps, cap=cap, threads=8)
    batch = engine.upload(xs)
    try:
        res = engine.krp_sum(batch, ws, [s] * 3, T.RngSeed(*seed), eps, cap)
        out = res.to_tucker()
        res.free()
    finally:
        batch.free()
    assert out.ranks == ref.ranks
    assert O.rel_error_to_sum(out, [ref], [1.0]) <= PARITY
    _err_same(out, ref, xs, ws)


def test_krp_wide_sketch_wider_than_rows(engine):
    """s > n_j for one mode (wide Y: any orthonormal basis of R^n is exact)."""
    dims, ranks, K = [90, 240, 200], [12, 14, 10], 6
    xs = [random_tucker(dims, ranks, (931, i)) for i in range(K)]
    ws = [1.0, -0.5, 0.75, 2.0, -1.25, 0.4]
    seed = (931, 2)
    ref, _ = O.krp_sum(xs, ws, [110] * 3, seed, 1e-9, threads=8)
    batch = engine.upload(xs)
    try:
        res = engine.krp_sum(batch, ws, [110] * 3, T.RngSeed(*seed), 1e-9)
        out = res.to_tucker()
        res.free()
    finally:
        batch.free()
    assert out.ranks == ref.ranks
    assert O.rel_error_to_sum(out, [ref], [1.0]) <= PARITY
    _err_same(out, ref, xs, ws)


def test_kron_wide_complement_parity(engine):
    """Kron widths (10, 10, 10): every C_n = 100 > 96."""
    dims = [200, 180, 160]
    xs = [random_tucker(dims, [3, 3, 3], (932, i)) for i in range(4)]
    ws = [1.0, -0.5, 2.0, 0.25]
    widths = [10, 10, 10]
    seed = (932, 1)
    ref, _ = O.kron_sum(xs, ws, widths, seed=seed, eps=1e-9)
    batch = engine.upload(xs)
    try:
        res = engine.kron_sum(batch, ws, widths, T.RngSeed(*seed), 1e-9)
        out = res.to_tucker()
        res.free()
    finally:
        batch.free()
    assert out.ranks == ref.ranks
    assert O.rel_error_to_sum(out, [ref], [1.0]) <= PARITY
    _err_same(out, ref, xs, ws)


@pytest.mark.parametrize("eps,cap", [(1e-8, None), (0.0, [40, 40, 40])])
def test_lazy_wide_stack_parity(engine, eps, cap):
    """Lazy rounding with stacked rank 100 > 96 per mode (tall stacks)."""
    xs = [random_tucker([200, 200, 200], [10, 10, 10], (90, i)) for i in range(10)]
    ws = list(np.random.default_rng(90).uniform(-1.0, 1.0, size=10))
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
    _err_same(out, ref, xs, ws)


def test_paper_fig2_setting_plan_and_lazy(engine):
    """The paper's synthetic-lowrank sweep point d = 100 (reference defaults:
    mode_dim 60, 4 modes, latent rank 10, 100 rank-1 summands, eps 1e-6,
    oversampling 2): the device plan equals the oracle's (stack 60 × 100 per
    mode), Lazy (wide stack: q = 60) matches the oracle, and the KRP sum with the
    device plan recovers the latent ranks."""
    xs = shared_subspace(60, 4, 10, 100, (2603, 7))
    ws = [1.0] * 100
    eff, tg, wd = O.effective_subrank_krp(xs, ws, 1e-6, 2)
    plan = T.effective_subrank(xs, ws, 1e-6, 2, T.Strategy.Krp, engine=engine)
    assert plan.effective_ranks == eff == [10] * 4
    assert plan.targets == tg and plan.mode_sketch_dims == wd
    ref = O.lazy_sum(xs, ws, 1e-6)
    batch = engine.upload(xs)
    try:
        res = engine.lazy_sum(batch, ws, 1e-6)
        out = res.to_tucker()
        res.free()
    finally:
        batch.free()
    assert out.ranks == ref.ranks == [10] * 4
    assert O.rel_error_to_sum(out, [ref], [1.0]) <= PARITY
    krp = T.krp_sum(T.SumRequest(xs, ws, 1e-6, 2, T.Strategy.Krp, T.RngSeed(2603, 8)), engine=engine)
    assert krp.ranks == [10] * 4
    assert O.rel_error_to_sum(krp, [ref], [1.0]) <= 1e-8


def test_plan_tall_stack_n4000(engine):
    """Plan stage at mode size 4000 with 100 rank-1 summands (stack 4000 × 100)."""
    xs = shared_subspace(4000, 4, 10, 100, (2603, 9))
    ws = list(np.random.default_rng(9).uniform(0.5, 1.5, size=100))
    for eps, p in ((1e-6, 2), (1e-10, 0)):
        eff, tg, wd = O.effective_subrank_krp(xs, ws, eps, p)
        plan = T.effective_subrank(xs, ws, eps, p, T.Strategy.Krp, engine=engine)
        assert plan.effective_ranks == eff and plan.targets == tg and plan.mode_sketch_dims == wd


def test_plan_stack_beyond_128(engine):
    """Plan stage with 150 stacked columns per mode (block one-sided Jacobi on the stack)."""
    xs = shared_subspace(300, 3, 12, 150, (2603, 11))
    ws = list(np.random.default_rng(11).uniform(0.5, 1.5, size=150))
    eff, tg, wd = O.effective_subrank_krp(xs, ws, 1e-6, 2)
    plan = T.effective_subrank(xs, ws, 1e-6, 2, T.Strategy.Krp, engine=engine)
    assert plan.effective_ranks == eff == [12] * 3
    assert plan.targets == tg and plan.mode_sketch_dims == wd
