"""Pins the CPU oracle against the reference's own known-answer tests and assertions.

Each test cites the reference test it restates (paths relative to
/root/reference/proj).  The reference cannot be built here (no Eigen), so these
KATs / identities / tolerance assertions plus the numpy re-derivation below are
what pin the oracle.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
from helpers import (cancellation_instance, dense_rel_error, dense_weighted_sum, orthonormal_cols, random_tucker,
                     shared_subspace, sub)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def counting_tensor(shape):
    n = int(np.prod(shape))
    return np.arange(1, n + 1, dtype=float).reshape(shape, order="F")


def random_tensor(shape, seed):
    n = int(np.prod(shape))
    return O.gaussian_matrix(n, 1, seed)[:, 0].reshape(shape, order="F")


def unfold_index_map(t, mode):
    """test_tensor_kernels.cpp:18-44 — entry (i_k, j), j = Σ_{m≠k} i_m Π_{l<m,l≠k} n_l."""
    shape = t.shape
    cols = int(np.prod([s for m, s in enumerate(shape) if m != mode]))
    out = np.zeros((shape[mode], cols))
    for idx in np.ndindex(*shape):
        j, stride = 0, 1
        for m in range(len(shape)):
            if m == mode:
                continue
            j += idx[m] * stride
            stride *= shape[m]
        out[idx[mode], j] = t[idx]
    return out


# ------------------------------------------------------------ layout KATs
def test_mode2_unfolding_frozen_layout():
    """test_tensor_kernels.cpp:93-101."""
    t = counting_tensor((2, 2, 2))
    expected = np.array([[1, 2, 5, 6], [3, 4, 7, 8]], dtype=float)
    assert np.array_equal(O.unfold(t, 1), expected)
    assert np.array_equal(unfold_index_map(t, 1), expected)


def test_matrix_unfoldings():
    """test_tensor_kernels.cpp:103-114."""
    t = np.array([[1.0, 2.0], [3.0, 4.0]], order="F")
    assert np.array_equal(O.unfold(t, 0), [[1, 2], [3, 4]])
    assert np.array_equal(O.unfold(t, 1), [[1, 3], [2, 4]])


def test_unfold_index_map_and_fold_inverse():
    """test_tensor_kernels.cpp:116-128."""
    shapes = [(3, 4, 5), (2, 3, 4, 2), (5, 2), (4,), (2, 2, 2, 2, 3)]
    for salt, shape in enumerate(shapes):
        t = random_tensor(shape, (42, salt))
        for mode in range(len(shape)):
            u = O.unfold(t, mode)
            assert np.array_equal(u, unfold_index_map(t, mode))
            assert np.array_equal(O.fold(u, mode, shape), t)


def test_ttm_contraction_oracle():
    """test_tensor_kernels.cpp:130-139 (≤ 1e-13 relative)."""
    t = random_tensor((3, 4, 2, 3), (7, 0))
    for mode in range(4):
        a = O.gaussian_matrix(5, t.shape[mode], (7, 10 + mode))
        got = O.ttm(t, a, mode)
        want = np.moveaxis(np.tensordot(a, t, axes=([1], [mode])), 0, mode)
        assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


def test_kron_frozen_example():
    """test_tensor_kernels.cpp:150-160."""
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[0.0, 1.0], [1.0, 0.0]])
    expected = np.array([[0, 1, 0, 2], [1, 0, 2, 0], [0, 3, 0, 4], [3, 0, 4, 0]], dtype=float)
    assert np.array_equal(O.kron(a, b), expected)


def test_khatri_rao_frozen_and_column_rule():
    """test_tensor_kernels.cpp:175-193."""
    kr = O.khatri_rao(np.array([[2.0]]), np.array([[3.0], [4.0]]))
    assert kr.shape == (2, 1) and kr[0, 0] == 6 and kr[1, 0] == 8
    c = O.gaussian_matrix(3, 4, (2, 1))
    d = O.gaussian_matrix(2, 4, (2, 2))
    full = O.khatri_rao(c, d)
    for col in range(4):
        assert np.array_equal(full[:, col], O.kron(c[:, [col]], d[:, [col]])[:, 0])
    with pytest.raises(ValueError):
        O.khatri_rao(c, O.gaussian_matrix(2, 3, (2, 3)))


def test_mixed_product_identities():
    """test_tensor_kernels.cpp:195-209 (≤ 1e-13)."""
    a = O.gaussian_matrix(3, 4, (3, 1))
    b = O.gaussian_matrix(2, 5, (3, 2))
    c2 = O.gaussian_matrix(4, 6, (3, 5))
    d2 = O.gaussian_matrix(5, 6, (3, 6))
    lhs = O.kron(a, b) @ O.khatri_rao(c2, d2)
    rhs = O.khatri_rao(a @ c2, b @ d2)
    assert np.linalg.norm(lhs - rhs) <= 1e-13 * np.linalg.norm(rhs)


def test_qr_econ_properties():
    """test_tensor_kernels.cpp:211-225."""
    for m, n in [(7, 4), (4, 7), (6, 6)]:
        a = O.gaussian_matrix(m, n, (4, m * 10 + n))
        q, r = O.qr_econ(a)
        k = min(m, n)
        assert q.shape == (m, k) and r.shape == (k, n)
        assert np.linalg.norm(q.T @ q - np.eye(k)) <= 1e-12
        assert np.linalg.norm(q @ r - a) <= 1e-12 * np.linalg.norm(a)
        assert np.all(np.diag(r) >= 0)
        assert np.all(np.tril(r, -1) == 0)


def test_svd_econ_properties():
    """test_tensor_kernels.cpp:227-235."""
    a = O.gaussian_matrix(8, 5, (5, 0))
    u, s, v = O.svd_econ(a)
    assert len(s) == 5 and np.all(np.diff(s) <= 0)
    assert np.linalg.norm(u @ np.diag(s) @ v.T - a) <= 1e-11 * np.linalg.norm(a)
    assert np.linalg.norm(u.T @ u - np.eye(5)) <= 1e-12
    assert np.linalg.norm(v.T @ v - np.eye(5)) <= 1e-12
    np.testing.assert_allclose(s, np.linalg.svd(a, compute_uv=False), rtol=1e-13)


def test_sym_eig_matches_squared_singular_values():
    """test_tensor_kernels.cpp:237-248."""
    a = O.gaussian_matrix(9, 6, (6, 0))
    vals, vecs = O.sym_eig(a.T @ a)
    s = O.svd_econ(a)[1]
    assert np.max(np.abs(vals - s * s)) <= 1e-10 * s[0] ** 2
    assert np.linalg.norm(vecs.T @ vecs - np.eye(6)) <= 1e-12
    with pytest.raises(ValueError):
        O.sym_eig(np.zeros((2, 3)))


def test_gaussian_matrix_determinism_streams_moments():
    """test_tensor_kernels.cpp:250-268."""
    a = O.gaussian_matrix(20, 20, (11, 3))
    assert np.array_equal(a, O.gaussian_matrix(20, 20, (11, 3)))
    assert not np.array_equal(a, O.gaussian_matrix(20, 20, (11, 4)))
    assert not np.array_equal(a, O.gaussian_matrix(20, 20, (12, 3)))
    big = O.gaussian_matrix(1000, 1000, (11, 5))
    assert abs(big.mean()) < 0.01
    assert abs(big.var(ddof=1) - 1.0) < 0.02
    s = O.substream(11, 3, 9)
    assert s[0] == 11 and s[1] != 3


def test_gaussian_golden_vectors():
    """Frozen libstdc++ draws (tests/golden/gaussian.json, made by tests/golden/make_golden.py)."""
    with open(os.path.join(GOLDEN, "gaussian.json")) as f:
        gold = json.load(f)
    for case in gold["cases"]:
        got = O.gaussian_matrix(case["rows"], case["cols"], (case["seed"], case["stream"]))
        assert got.ravel(order="F").tolist() == case["values"]
    for case in gold["substream"]:
        assert list(O.substream(case["seed"], case["stream"], case["salt"])) == [case["out_seed"], case["out_stream"]]


def test_mttkrp_identity():
    """test_tucker_core.cpp:173-188: unfold(G ×_j M_jᵀ..., n) vs G_(n)·(⊙ M_j) (≤ 1e-11)."""
    g = random_tensor((3, 4, 5), (13, 0))
    ms = [O.gaussian_matrix(g.shape[j], 6, (13, 1 + j)) for j in range(3)]
    for n in range(3):
        k = None
        for j in (2, 1, 0):
            if j == n:
                continue
            k = ms[j] if k is None else O.khatri_rao(k, ms[j])
        lhs = O.unfold(g, n) @ k
        rhs = np.einsum("abc,ax,bx,cx->" + "abc"[n] + "x", g, *[m if j != n else np.ones_like(m) for j, m in enumerate(ms)])
        assert np.linalg.norm(lhs - rhs) <= 1e-11 * np.linalg.norm(rhs)


# ------------------------------------------------------------ krp_sum assertions
def test_opposite_summands_annihilate():
    """test_sketch_sum.cpp:186-198."""
    x = random_tucker([12, 10, 8], [3, 4, 2], (21, 3))
    out, _ = O.krp_sum([x, x], [1.0, -1.0], None, (21, 4), 1e-6, oversampling=5)
    assert O.tucker_norm(out) <= 1e-12 * O.tucker_norm(x)


def test_single_summand_passes_through():
    """test_sketch_sum.cpp:200-219."""
    x = random_tucker([15, 12, 18], [4, 3, 5], (31, 0))
    ref = O.reconstruct(x)
    out, _ = O.krp_sum([x], [1.0], None, (31, 1), 1e-10, oversampling=2)
    assert out.dims == x.dims
    assert O.rel_error_to_sum(out, [x], [1.0]) <= 1e-10
    assert dense_rel_error(out, ref) <= 1e-10


@pytest.mark.slow
def test_shared_subspace_recovers_latent_ranks():
    """test_sketch_sum.cpp:221-264 (d = 20 rank-1 summands of 60⁴, latent rank 10)."""
    seed = (51, 0)
    xs = shared_subspace(60, 4, 10, 20, seed)
    ws = [1.0] * 20
    ref = dense_weighted_sum(xs, ws)
    eff, tg, wd = O.effective_subrank_krp(xs, ws, 1e-6, 2)
    assert eff == [10] * 4 and wd == [12] * 4
    out, info = O.krp_sum(xs, ws, None, sub(seed, 77), 1e-6, oversampling=2)
    assert out.ranks == [10] * 4
    assert dense_rel_error(out, ref) <= 1e-10
    assert info["widths"] == [12] * 4


def test_random_sums_match_dense_oracle():
    """test_sketch_sum.cpp:266-299 (KRP branch, 20 trials, ≤ 1e-6)."""
    rng = np.random.Generator(np.random.MT19937(907))
    dims = [14, 11, 9]
    for trial in range(20):
        xs, ws = [], []
        for i in range(5):
            ranks = [int(x) for x in rng.integers(1, 4, size=3)]
            xs.append(random_tucker(dims, ranks, (1000 + trial, i)))
            ws.append((1.0 if rng.integers(0, 2) == 0 else -1.0) * rng.uniform(0.5, 2.0))
        ref = dense_weighted_sum(xs, ws)
        out, _ = O.krp_sum(xs, ws, None, (42, trial), 1e-6, oversampling=5)
        assert dense_rel_error(out, ref) <= 1e-6


def test_shared_subspaces_across_seeds():
    """test_sketch_sum.cpp:301-347 (latent rank 4, ≤ 1e-8)."""
    rng = np.random.Generator(np.random.MT19937(1310))
    dims = [18, 15, 12]
    for trial in range(20):
        seed = (2000 + trial, 0)
        xs = shared_subspace(dims, 3, 4, 8, seed, rank=2, core_salt=True)
        ws = list(rng.uniform(0.5, 1.5, size=8))
        ref = dense_weighted_sum(xs, ws)
        eff, _, _ = O.effective_subrank_krp(xs, ws, 1e-8, 2)
        assert eff == [4, 4, 4]
        out, _ = O.krp_sum(xs, ws, None, sub(seed, 9000), 1e-8, oversampling=2)
        assert out.ranks == [4, 4, 4]
        assert dense_rel_error(out, ref) <= 1e-8


def test_paired_cancellation_keeps_quiet_components():
    """test_sketch_sum.cpp:560-598 (KRP branch, ≤ 1e-9)."""
    xs, ws, target = cancellation_instance(40, 10, (107, 0))
    ref = O.reconstruct(target)
    naive = dense_weighted_sum(xs, ws)
    assert np.linalg.norm(naive - ref) / np.linalg.norm(ref) <= 1e-9
    out, _ = O.krp_sum(xs, ws, None, (107, 1), 1e-6, oversampling=2)
    assert dense_rel_error(out, ref) <= 1e-9


def test_malformed_requests_rejected():
    """test_sketch_sum.cpp:514-547 (std::invalid_argument → ValueError)."""
    a = random_tucker([8, 7, 6], [2, 2, 2], (91, 0))
    b = random_tucker([8, 7, 5], [2, 2, 2], (91, 1))
    one_d = random_tucker([9], [2], (91, 2))
    with pytest.raises(ValueError):
        O.krp_sum([a, b], [1.0, 1.0], [3, 3, 3], (0, 0), 1e-8)
    with pytest.raises(ValueError):
        O.krp_sum([a], [1.0, 2.0], [3, 3, 3], (0, 0), 1e-8)
    with pytest.raises(ValueError):
        O.krp_sum([one_d], [1.0], [3], (0, 0), 1e-8)
    with pytest.raises(ValueError):
        O.krp_sum([a], [1.0], [3, 3, 3], (0, 0), -1.0)
    with pytest.raises(ValueError):
        O.effective_subrank_krp([a], [1.0], 1e-6, [1, 1])


def test_plan_exact_effective_ranks_for_duplicates():
    """test_sketch_sum.cpp:120-140 (Krp part)."""
    x = random_tucker([9, 8, 7], [2, 2, 2], (11, 0))
    eff, tg, wd = O.effective_subrank_krp([x] * 5, [0.7] * 5, 1e-8, [0, 0, 0])
    assert eff == [2, 2, 2] and tg == [2, 2, 2] and wd == [2, 2, 2]


# ------------------------------------------------------------ independent numpy re-derivation
def numpy_krp_sum(xs, ws, omega, eps, cap=None):
    """Independent restatement with numpy/LAPACK fed the oracle's Ω (reference
    src/sketch.cpp:66-181): einsum contractions, LAPACK QR and SVD."""
    d = len(xs[0].dims)
    y = [np.zeros_like(o) for o in omega]
    for x, w in zip(xs, ws):
        m = [x.factors[j].T @ omega[j] for j in range(d)]
        for b in x.blocks:
            g = b.data
            for n in range(d):
                sl = [m[j][b.offsets[j]:b.offsets[j] + g.shape[j]] for j in range(d)]
                letters = "abcdefgh"[:d]
                ops = [g] + [sl[j] for j in range(d) if j != n]
                spec = letters + "," + ",".join(letters[j] + "z" for j in range(d) if j != n) + "->" + letters[n] + "z"
                v = np.einsum(spec, *ops)
                y[n] += w * x.factors[n][:, b.offsets[n]:b.offsets[n] + g.shape[n]] @ v
    uh = []
    for n in range(d):
        q, r = np.linalg.qr(y[n])
        sgn = np.sign(np.diag(r))
        sgn[sgn == 0] = 1
        uh.append(q * sgn)
    h = np.zeros([u.shape[1] for u in uh])
    for x, w in zip(xs, ws):
        proj = [uh[n].T @ x.factors[n] for n in range(d)]
        for b in x.blocks:
            v = b.data
            for n in range(d):
                p = proj[n][:, b.offsets[n]:b.offsets[n] + b.data.shape[n]]
                v = np.moveaxis(np.tensordot(p, v, axes=([1], [n])), 0, n)
            h = h + w * v
    theta = eps * eps * np.sum(h * h) / d
    order = sorted(range(d), key=lambda k: h.shape[k])
    g = h
    pk = [None] * d
    for k in order:
        u, s, _ = np.linalg.svd(np.moveaxis(g, k, 0).reshape(g.shape[k], -1, order="F"), full_matrices=False)
        if eps == 0:
            rank = len(s)
            while rank > 1 and s[rank - 1] <= 1e-14 * s[0]:
                rank -= 1
        else:
            tail = np.concatenate([np.cumsum((s * s)[::-1])[::-1], [0.0]])
            rank = next(r for r in range(1, len(s) + 1) if tail[r] <= theta) if np.any(tail[1:] <= theta) else len(s)
        if cap is not None:
            rank = min(rank, cap[k])
        pk[k] = u[:, :rank]
        g = np.moveaxis(np.tensordot(pk[k].T, g, axes=([1], [k])), 0, k)
    return g, [uh[n] @ pk[n] for n in range(d)]


def test_oracle_matches_numpy_rederivation():
    """The oracle's pipeline equals an independent numpy/LAPACK restatement (≤ 1e-12)."""
    from paper_2603_13532_b200.tucksum import TuckerTensor

    for trial, (dims, r, K, s, cap) in enumerate([([20, 17, 15], [3, 4, 2], 4, 9, None),
                                                  ([16, 12, 10, 9], [2, 3, 2, 2], 3, 7, [4, 4, 3, 3]),
                                                  ([30, 25], [4, 3], 5, 8, None)]):
        xs = [random_tucker(dims, r, (600 + trial, i)) for i in range(K)]
        ws = [1.0, -0.5, 2.0, 0.25, 1.5][:K]
        out, info = O.krp_sum(xs, ws, [s] * len(dims), (600 + trial, 77), 1e-9, cap=cap, intermediates=True)
        core, factors = numpy_krp_sum(xs, ws, info["omega"], 1e-9, cap)
        alt = TuckerTensor(core, factors)
        assert O.rel_error_to_sum(alt, [out], [1.0]) <= 1e-12


def test_gram_error_matches_reference_formula():
    """Gram-based error agrees with tucker_rel_error on small cases."""
    xs = [random_tucker([20, 18, 16], [3, 3, 3], (700, i)) for i in range(5)]
    ws = [1.0, 0.5, -0.7, 1.2, 0.3]
    out, _ = O.krp_sum(xs, ws, [6, 6, 6], (700, 9), 0.0, cap=[4, 4, 4])
    ref_err = O.rel_error_to_sum(out, xs, ws)
    gram_err = O.rel_error_gram(out, xs, ws)
    assert ref_err > 1e-6
    assert abs(gram_err - ref_err) <= 1e-6 * ref_err
