"""Oracle: the Kronecker-sketch variant — the reference's
own kron_sum / kron_sketch_dims assertions restated
(/root/reference/proj/tests/test_sketch_sum.cpp), plus an independent numpy
re-derivation of the Kron pipeline fed the oracle's Ω."""
import numpy as np
import pytest

import oracle as O
from helpers import cancellation_instance, dense_rel_error, dense_weighted_sum, random_tucker, shared_subspace, sub


def feasibility_width(s, skip):
    """test_sketch_sum.cpp:61-67."""
    return int(np.prod([v for j, v in enumerate(s) if j != skip]))


def test_kron_widths_follow_balancing_rule():
    """test_sketch_sum.cpp:159-184."""
    assert O.kron_sketch_dims([4, 4, 4], [20, 20, 20]) == [2, 2, 2]
    assert O.kron_sketch_dims([10, 2, 2], [30, 30, 30]) == [1, 4, 4]
    assert O.kron_sketch_dims([3, 3, 3], [9, 9, 9]) == [2, 2, 2]
    assert O.kron_sketch_dims([2, 8, 8], [2, 10, 10]) == [2, 4, 4]
    for targets, dims in [([4, 4, 4], [20, 20, 20]), ([10, 2, 2], [30, 30, 30]), ([2, 8, 8], [2, 10, 10]),
                          ([7, 7, 2], [12, 12, 12]), ([5, 9], [11, 13])]:
        s = O.kron_sketch_dims(targets, dims)
        for n in range(len(s)):
            assert 1 <= s[n] <= dims[n]
            assert feasibility_width(s, n) >= targets[n]
    with pytest.raises(ValueError):
        O.kron_sketch_dims([5, 2, 2], [6, 2, 2])
    with pytest.raises(ValueError):
        O.kron_sketch_dims([2], [4])
    with pytest.raises(ValueError):
        O.kron_sketch_dims([0, 2], [4, 4])


def test_kron_plan_exact_effective_ranks_for_duplicates():
    """test_sketch_sum.cpp:150-156."""
    x = random_tucker([9, 8, 7], [2, 2, 2], (11, 0))
    eff, tg, wd = O.effective_subrank([x] * 5, [0.7] * 5, 1e-8, [0, 0, 0], strategy="kron")
    assert eff == [2, 2, 2] and wd == [2, 2, 2]
    for n in range(3):
        assert feasibility_width(wd, n) >= tg[n]


def test_kron_opposite_summands_annihilate():
    """test_sketch_sum.cpp:186-198 (Kron branch)."""
    x = random_tucker([12, 10, 8], [3, 4, 2], (21, 3))
    out, _ = O.kron_sum([x, x], [1.0, -1.0], None, seed=(21, 4), eps=1e-6, oversampling=5)
    assert O.tucker_norm(out) <= 1e-12 * O.tucker_norm(x)


def test_kron_single_summand_passes_through():
    """test_sketch_sum.cpp:200-219 (Kron branch)."""
    x = random_tucker([15, 12, 18], [4, 3, 5], (31, 0))
    ref = O.reconstruct(x)
    out, _ = O.kron_sum([x], [1.0], None, seed=(31, 1), eps=1e-10, oversampling=2)
    assert O.rel_error_to_sum(out, [x], [1.0]) <= 1e-10
    assert dense_rel_error(out, ref) <= 1e-10


@pytest.mark.slow
def test_kron_shared_subspace_recovers_latent_ranks():
    """test_sketch_sum.cpp:221-264 (Kron branch)."""
    seed = (51, 0)
    xs = shared_subspace(60, 4, 10, 20, seed)
    ws = [1.0] * 20
    ref = dense_weighted_sum(xs, ws)
    out, _ = O.kron_sum(xs, ws, None, seed=sub(seed, 77), eps=1e-6, oversampling=2)
    assert out.ranks == [10] * 4
    assert dense_rel_error(out, ref) <= 1e-10


def test_kron_random_sums_match_dense_oracle():
    """test_sketch_sum.cpp:266-299 (Kron branch, 20 trials, ≤ 1e-6)."""
    rng = np.random.Generator(np.random.MT19937(907))
    dims = [14, 11, 9]
    for trial in range(20):
        xs, ws = [], []
        for i in range(5):
            ranks = [int(x) for x in rng.integers(1, 4, size=3)]
            xs.append(random_tucker(dims, ranks, (1000 + trial, i)))
            ws.append((1.0 if rng.integers(0, 2) == 0 else -1.0) * rng.uniform(0.5, 2.0))
        ref = dense_weighted_sum(xs, ws)
        out, _ = O.kron_sum(xs, ws, None, seed=(42, trial), eps=1e-6, oversampling=5)
        assert dense_rel_error(out, ref) <= 1e-6


def test_kron_shared_subspaces_across_seeds():
    """test_sketch_sum.cpp:301-347 (Kron branch, latent rank 4, ≤ 1e-8)."""
    rng = np.random.Generator(np.random.MT19937(1310))
    dims = [18, 15, 12]
    for trial in range(20):
        seed = (2000 + trial, 0)
        xs = shared_subspace(dims, 3, 4, 8, seed, rank=2, core_salt=True)
        ws = list(rng.uniform(0.5, 1.5, size=8))
        ref = dense_weighted_sum(xs, ws)
        out, _ = O.kron_sum(xs, ws, None, seed=sub(seed, 9000), eps=1e-8, oversampling=2)
        assert out.ranks == [4, 4, 4]
        assert dense_rel_error(out, ref) <= 1e-8


def test_kron_weight_rescaling_keeps_plan():
    """test_sketch_sum.cpp:349-367 (both strategies)."""
    xs = [random_tucker([13, 9, 11], [2, 3, 2], (61, i)) for i in range(4)]
    ws = [1.0 + 0.25 * i for i in range(4)]
    for strat in ("krp", "kron"):
        base = O.effective_subrank(xs, ws, 1e-6, 2, strategy=strat)
        for scale in (1e3, 1e-6):
            other = O.effective_subrank(xs, [w * scale for w in ws], 1e-6, 2, strategy=strat)
            assert other[0] == base[0] and other[2] == base[2]


def test_plans_feasible_on_skewed_instances():
    """test_sketch_sum.cpp:369-403 (30 skewed random instances, both strategies)."""
    rng = np.random.Generator(np.random.MT19937(4242))
    for it in range(30):
        order = 2 + it % 3
        dims = [int(2 + rng.integers(0, 23)) for _ in range(order)]
        count = int(1 + rng.integers(0, 5))
        xs, ws = [], []
        for i in range(count):
            ranks = [int(1 + rng.integers(0, min(dims[k], 4))) for k in range(order)]
            xs.append(random_tucker(dims, ranks, (7000 + it, i)))
            ws.append(float(int(rng.integers(0, 5)) - 2))
        eps = 1e-4 if it % 2 == 0 else 1e-8
        p = (it % 3) * 2
        _, tg, wd = O.effective_subrank(xs, ws, eps, p, strategy="kron")
        for n in range(order):
            assert tg[n] >= 1 and 1 <= wd[n] <= dims[n]
            assert feasibility_width(wd, n) >= tg[n]
        _, tg, wd = O.effective_subrank(xs, ws, eps, p, strategy="krp")
        assert wd == [max(tg)] * order


def test_kron_paired_cancellation_keeps_quiet_components():
    """test_sketch_sum.cpp:560-598 (Kron branch, ≤ 1e-9)."""
    xs, ws, target = cancellation_instance(40, 10, (107, 0))
    ref = O.reconstruct(target)
    out, _ = O.kron_sum(xs, ws, None, seed=(107, 1), eps=1e-6, oversampling=2)
    assert dense_rel_error(out, ref) <= 1e-9


def test_kron_malformed_requests_rejected():
    """test_sketch_sum.cpp:514-547 (kron_sum of a first-order summand)."""
    one_d = random_tucker([9], [2], (91, 2))
    with pytest.raises(ValueError):
        O.kron_sum([one_d], [1.0], [3], seed=(0, 0), eps=1e-8)


def numpy_kron_sum(xs, ws, omega, eps, cap=None):
    """Independent numpy/LAPACK restatement of the Kron pipeline (reference
    src/sketch.cpp:66-181, krp = false) fed the oracle's Ω."""
    d = len(xs[0].dims)
    cols = [int(np.prod([omega[j].shape[1] for j in range(d) if j != n])) for n in range(d)]
    y = [np.zeros((omega[n].shape[0], cols[n])) for n in range(d)]
    for x, w in zip(xs, ws):
        m = [omega[j].T @ x.factors[j] for j in range(d)]
        for b in x.blocks:
            for n in range(d):
                v = b.data
                for j in range(d):
                    if j == n:
                        continue
                    mj = m[j][:, b.offsets[j]:b.offsets[j] + b.data.shape[j]]
                    v = np.moveaxis(np.tensordot(mj, v, axes=([1], [j])), 0, j)
                un = np.moveaxis(v, n, 0).reshape(v.shape[n], -1, order="F")
                y[n] += w * x.factors[n][:, b.offsets[n]:b.offsets[n] + b.data.shape[n]] @ un
    return y


def test_kron_oracle_matches_numpy_rederivation():
    """The oracle's Kron sketches Y_n equal the numpy restatement (≤ 1e-12), and
    the oracle's output reproduces the exact sum where the sketch covers it."""
    for trial, (dims, r, K, widths) in enumerate([([20, 17, 15], [3, 4, 2], 4, [3, 3, 4]),
                                                   ([16, 12, 10, 9], [2, 3, 2, 2], 3, [2, 2, 3, 2]),
                                                   ([30, 25], [4, 3], 5, [6, 7])]):
        xs = [random_tucker(dims, r, (650 + trial, i)) for i in range(K)]
        ws = [1.0, -0.5, 2.0, 0.25, 1.5][:K]
        out, info = O.kron_sum(xs, ws, widths, seed=(650 + trial, 77), eps=1e-9, intermediates=True)
        for n, om in enumerate(info["omega"]):
            assert om.shape == (dims[n], widths[n])
        y = numpy_kron_sum(xs, ws, info["omega"], 1e-9)
        for n in range(len(dims)):
            assert info["y"][n].shape == y[n].shape
            assert np.linalg.norm(info["y"][n] - y[n]) <= 1e-12 * np.linalg.norm(y[n])
