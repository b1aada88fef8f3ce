"""Parity of the sm_100a CUDA path (through the C ABI) with the CPU oracle.

Tolerances (BASELINE.json north_star): the returned factors × core within 1e-10
relative Frobenius error of the oracle's on identical inputs and identical Ω,
and the same approximation error to the exact sum to 3 significant digits.
Factors are never compared directly (SVD sign / rank-deficient QR freedom,
SURVEY.md §8(c)); reconstructions are compared through the reference's
orthogonalized-difference norm (tucker_rel_error, src/tucker.cpp:298-303).
"""
import numpy as np
import pytest

import oracle as O
from helpers import (cancellation_instance, dense_rel_error, dense_weighted_sum, random_tucker, shared_subspace,
                     sub)
from paper_2603_13532_b200 import tucksum as T
from paper_2603_13532_b200.workloads import make_workload

pytestmark = pytest.mark.gpu

PARITY = 1e-10  # relative Frobenius error of factors × core vs the oracle


def gpu_sum(engine, xs, ws, widths, seed, eps, cap=None, debug=False):
    engine.set_debug(debug)
    batch = engine.upload(xs)
    try:
        res = engine.krp_sum(batch, ws, widths, T.RngSeed(*seed), eps, cap)
        out = res.to_tucker()
        inter = res.intermediates() if debug else None
        res.free()
    finally:
        batch.free()
        engine.set_debug(False)
    return out, inter


def rel_diff(a, b):
    return O.rel_error_to_sum(a, [b], [1.0])


def check_pair(engine, xs, ws, widths, seed, eps, cap=None, err_digits=True, gram=False):
    ref, _ = O.krp_sum(xs, ws, widths, seed, eps, cap=cap, threads=8)
    out, _ = gpu_sum(engine, xs, ws, widths, seed, eps, cap)
    assert out.ranks == ref.ranks
    assert rel_diff(out, ref) <= PARITY
    if err_digits:
        if gram:
            e_gpu, e_ref = O.rel_error_gram(out, xs, ws, 8), O.rel_error_gram(ref, xs, ws, 8)
        else:
            e_gpu, e_ref = O.rel_error_to_sum(out, xs, ws), O.rel_error_to_sum(ref, xs, ws)
        assert abs(e_gpu - e_ref) <= 5e-4 * max(e_ref, 1e-300) or abs(e_gpu - e_ref) <= 1e-13
    return out, ref


# ------------------------------------------------------------ BASELINE configs
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_baseline_config_parity(engine, cfg):
    wl = make_workload(cfg)
    check_pair(engine, wl.summands, wl.weights, wl.widths, (wl.seed.seed, wl.seed.stream), wl.eps, wl.cap)


def test_baseline_cfg4_parity(engine):
    wl = make_workload(4)
    check_pair(engine, wl.summands, wl.weights, wl.widths, (wl.seed.seed, wl.seed.stream), wl.eps, wl.cap, gram=True)


def test_baseline_cfg5_reduced_parity(engine):
    """Config 5 shapes (n = 8192, r = 32, s = 64, cap 48) at K = 16 summands."""
    wl = make_workload(5, K=16)
    check_pair(engine, wl.summands, wl.weights, wl.widths, (wl.seed.seed, wl.seed.stream), wl.eps, wl.cap, gram=True)


def test_numerical_paths_are_exercised(engine):
    """CholeskyQR2 must hand exactly rank-deficient sketches (config 3, modes 2-3:
    rank 10 < s = 50) to Householder TSQR, and ST-HOSVD must take the accurate
    SVD path whenever the Gram decision is not provably exact."""
    wl = make_workload(3)
    seed = (wl.seed.seed, wl.seed.stream)
    check_pair(engine, wl.summands, wl.weights, wl.widths, seed, wl.eps, wl.cap)
    qr_fb, _ = engine.last_paths()
    assert qr_fb >= 2
    wl1 = make_workload(1)
    s1 = (wl1.seed.seed, wl1.seed.stream)
    check_pair(engine, wl1.summands, wl1.weights, wl1.widths, s1, wl1.eps, wl1.cap)
    assert engine.last_paths() == (0, 0)  # well-conditioned: CholQR2 and Gram fast paths
    # Config 3's parameter modes have exact rank 10 < q = 50: with eps = 1e-10 the
    # tail threshold sits below the Gram's rounding noise → accurate SVD path.
    check_pair(engine, wl.summands, wl.weights, wl.widths, seed, 1e-10, None)
    assert engine.last_paths()[1] >= 1


def test_speculative_tail_matches_synchronous_path():
    """The speculative tail (stage D/G acceptance checks on the device, one sync
    per call) gives bitwise the synchronous path's result when accepted, and a
    rejected speculation is recomputed on the synchronous path."""
    wl1, wl3 = make_workload(1), make_workload(3)
    s1, s3 = (wl1.seed.seed, wl1.seed.stream), (wl3.seed.seed, wl3.seed.stream)
    eng = T.Engine(0)
    try:
        spec1, _ = gpu_sum(eng, wl1.summands, wl1.weights, wl1.widths, s1, wl1.eps, wl1.cap)  # accepted
        out3, _ = gpu_sum(eng, wl3.summands, wl3.weights, wl3.widths, s3, wl3.eps, wl3.cap)  # rejected → rerun
        ref3, _ = O.krp_sum(wl3.summands, wl3.weights, wl3.widths, s3, wl3.eps, cap=wl3.cap, threads=8)
        assert out3.ranks == ref3.ranks and rel_diff(out3, ref3) <= PARITY
        sync1, _ = gpu_sum(eng, wl1.summands, wl1.weights, wl1.widths, s1, wl1.eps, wl1.cap)  # synchronous path
        assert sync1.ranks == spec1.ranks
        assert np.array_equal(sync1.dense_core(), spec1.dense_core())
        for a, b in zip(sync1.factors, spec1.factors):
            assert np.array_equal(a, b)
    finally:
        eng.close()


def test_nccl_path_single_rank_matches():
    """The multi-GPU code path — NCCL resolved at run time, a communicator, the
    two in-place all-reduces on the library stream — run with one rank gives
    bitwise the single-GPU result (only one GPU is available to this build)."""
    wl = make_workload(5, K=16)
    seed = (wl.seed.seed, wl.seed.stream)
    ref, _ = gpu_sum(T.Engine(0), wl.summands, wl.weights, wl.widths, seed, wl.eps, wl.cap)
    eng = T.Engine(0)
    try:
        assert eng.comm_info() == (1, 0)
        eng.init_nccl(T.Engine.nccl_unique_id(), 1, 0)
        assert eng.comm_info() == (1, 0)  # ncclCommCount / ncclCommUserRank
        out, _ = gpu_sum(eng, wl.summands, wl.weights, wl.widths, seed, wl.eps, wl.cap)
    finally:
        eng.close()
    assert out.ranks == ref.ranks
    assert np.array_equal(out.dense_core(), ref.dense_core())
    for a, b in zip(out.factors, ref.factors):
        assert np.array_equal(a, b)


def test_krp_sum_many_matches_sequential_calls():
    """Independent sums run side by side (ts_krp_sum_many) give bitwise the
    results of sequential krp_sum calls, for mixed shapes and seeds."""
    eng = T.Engine(0)
    try:
        wls = [make_workload(1), make_workload(2), make_workload(1, K=3), make_workload(4)]
        # same order required only per call: run the order-3 ones together
        wl3 = [w for w in wls if len(w.dims) == 3]
        batches = [eng.upload(w.summands) for w in wl3]
        seeds = [T.RngSeed(w.seed.seed, w.seed.stream + i) for i, w in enumerate(wl3)]
        widths = [30, 30, 30]
        cap = [16, 16, 16]
        many = eng.krp_sum_many(batches, [w.weights for w in wl3], widths, seeds, 0.0, cap, lanes=4)
        for b, w, sd, r in zip(batches, wl3, seeds, many):
            one = eng.krp_sum(b, w.weights, widths, sd, 0.0, cap)
            x, y = r.to_tucker(), one.to_tucker()
            assert x.ranks == y.ranks
            assert np.array_equal(x.dense_core(), y.dense_core())
            for a, c in zip(x.factors, y.factors):
                assert np.array_equal(a, c)
            r.free()
            one.free()
        for b in batches:
            b.free()
    finally:
        eng.close()


def test_krp_sum_many_matches_oracle_per_sum():
    """Every sum of a ts_krp_sum_many call (mixed shapes, seeds, both truncation
    modes) against the CPU oracle on its own inputs and Ω (1e-10, same ranks)."""
    eng = T.Engine(0)
    try:
        cases = [make_workload(1), make_workload(2), make_workload(1, K=3), make_workload(2, K=5, n_override=[300, 200, 100])]
        for eps, cap in [(0.0, [16, 16, 16]), (1e-6, None)]:
            batches = [eng.upload(w.summands) for w in cases]
            seeds = [T.RngSeed(w.seed.seed, w.seed.stream + 7 * i) for i, w in enumerate(cases)]
            widths = [30, 30, 30]
            many = eng.krp_sum_many(batches, [w.weights for w in cases], widths, seeds, eps, cap, lanes=3)
            for w, sd, r in zip(cases, seeds, many):
                out = r.to_tucker()
                r.free()
                ref, _ = O.krp_sum(w.summands, w.weights, widths, (sd.seed, sd.stream), eps, cap=cap, threads=8)
                assert out.ranks == ref.ranks
                assert rel_diff(out, ref) <= PARITY
            for b in batches:
                b.free()
    finally:
        eng.close()


def test_cpp_host_caller():
    """A C++ program drives the C ABI end to end (upload, two krp_sum calls,
    malformed requests, ranks, orthonormality, determinism, exact-sum norm)."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "tests", "cpp", "capi_host")
    if not os.path.exists(exe):
        subprocess.run([os.path.join(root, "tests", "cpp", "build.sh")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "capi_host ok" in r.stdout


@pytest.mark.parametrize("cfg", [1, 2])
def test_reference_semantics_eps(engine, cfg):
    """Pure reference semantics (eps > 0, no rank cap) on the same inputs."""
    wl = make_workload(cfg)
    check_pair(engine, wl.summands, wl.weights, wl.widths, (wl.seed.seed, wl.seed.stream), 1e-6, None)


@pytest.mark.parametrize("eps", [1e-6, 1e-10])
def test_reference_semantics_cfg4(engine, eps):
    """The path the drop-in adapter runs (eps > 0, max_rank = NULL; reference
    src/sketch.cpp:171, src/tucker.cpp:244-276) at BASELINE config 4 (d = 4)."""
    wl = make_workload(4)
    check_pair(engine, wl.summands, wl.weights, wl.widths, (wl.seed.seed, wl.seed.stream), eps, None, gram=True)


@pytest.mark.parametrize("eps", [1e-6, 1e-10])
def test_reference_semantics_cfg5_full_size(engine, eps):
    """Reference-exact mode at full config 5 (K = 256, n = 8192, s = 64, no cap):
    1e-10 on factors × core, same ranks, error to the exact sum to 3 digits."""
    wl = make_workload(5)
    out, ref = check_pair(engine, wl.summands, wl.weights, wl.widths, (wl.seed.seed, wl.seed.stream), eps, None,
                          gram=True)
    assert out.ranks == ref.ranks and max(out.ranks) <= 64


def test_stage_intermediates_cfg1(engine):
    """Ω bitwise; Y, Û, h against the oracle's intermediates."""
    wl = make_workload(1)
    seed = (wl.seed.seed, wl.seed.stream)
    ref, info = O.krp_sum(wl.summands, wl.weights, wl.widths, seed, 0.0, cap=wl.cap, intermediates=True)
    _, inter = gpu_sum(engine, wl.summands, wl.weights, wl.widths, seed, 0.0, wl.cap, debug=True)
    for n in range(3):
        assert np.array_equal(inter["omega"][n], info["omega"][n])
        y, yr = inter["y"][n], info["y"][n]
        assert np.linalg.norm(y - yr) <= 1e-13 * np.linalg.norm(yr)
        u, ur = inter["uhat"][n], info["uhat"][n]
        assert np.linalg.norm(u - ur) <= 1e-11
    assert np.linalg.norm(inter["h"] - info["h"]) <= 1e-11 * np.linalg.norm(info["h"])


# ------------------------------------------------------------ reference test assertions through the C ABI
def test_opposite_summands_annihilate(engine):
    """test_sketch_sum.cpp:186-198."""
    x = random_tucker([12, 10, 8], [3, 4, 2], (21, 3))
    req = T.SumRequest([x, x], [1.0, -1.0], 1e-6, 5, T.Strategy.Krp, T.RngSeed(21, 4))
    out = T.krp_sum(req, engine=engine)
    assert O.tucker_norm(out) <= 1e-12 * O.tucker_norm(x)


def test_single_summand_passes_through(engine):
    """test_sketch_sum.cpp:200-219."""
    x = random_tucker([15, 12, 18], [4, 3, 5], (31, 0))
    ref = O.reconstruct(x)
    req = T.SumRequest([x], [1.0], 1e-10, 2, T.Strategy.Krp, T.RngSeed(31, 1))
    out = T.krp_sum(req, engine=engine)
    assert out.dims == x.dims
    assert O.rel_error_to_sum(out, [x], [1.0]) <= 1e-10
    assert dense_rel_error(out, ref) <= 1e-10


def test_shared_subspace_recovers_latent_ranks(engine):
    """test_sketch_sum.cpp:221-264."""
    seed = (51, 0)
    xs = shared_subspace(60, 4, 10, 20, seed)
    ws = [1.0] * 20
    ref = dense_weighted_sum(xs, ws)
    req = T.SumRequest(xs, ws, 1e-6, 2, T.Strategy.Krp, T.RngSeed(*sub(seed, 77)))
    stats = T.SumStats()
    out = T.krp_sum(req, None, stats, engine=engine)
    assert out.ranks == [10] * 4
    assert dense_rel_error(out, ref) <= 1e-10
    assert stats.has_plan
    assert stats.plan.effective_ranks == [10] * 4
    assert stats.plan.mode_sketch_dims == [12] * 4


def test_random_sums_match_dense_oracle_and_cpu_oracle(engine):
    """test_sketch_sum.cpp:266-299 (KRP) + parity with the CPU oracle, plans included."""
    rng = np.random.Generator(np.random.MT19937(907))
    dims = [14, 11, 9]
    for trial in range(20):
        xs, ws = [], []
        for i in range(5):
            ranks = [int(x) for x in rng.integers(1, 4, size=3)]
            xs.append(random_tucker(dims, ranks, (1000 + trial, i)))
            ws.append((1.0 if rng.integers(0, 2) == 0 else -1.0) * rng.uniform(0.5, 2.0))
        ref = dense_weighted_sum(xs, ws)
        req = T.SumRequest(xs, ws, 1e-6, 5, T.Strategy.Krp, T.RngSeed(42, trial))
        stats = T.SumStats()
        out = T.round_sum(req, None, stats, engine=engine)
        assert dense_rel_error(out, ref) <= 1e-6
        eff, tg, wd = O.effective_subrank_krp(xs, ws, 1e-6, 5)
        assert stats.plan.effective_ranks == eff and stats.plan.mode_sketch_dims == wd
        oref, _ = O.krp_sum(xs, ws, wd, (42, trial), 1e-6)
        assert out.ranks == oref.ranks
        assert rel_diff(out, oref) <= PARITY


def test_shared_subspaces_across_seeds(engine):
    """test_sketch_sum.cpp:301-347."""
    rng = np.random.Generator(np.random.MT19937(1310))
    dims = [18, 15, 12]
    for trial in range(20):
        seed = (2000 + trial, 0)
        xs = shared_subspace(dims, 3, 4, 8, seed, rank=2, core_salt=True)
        ws = list(rng.uniform(0.5, 1.5, size=8))
        ref = dense_weighted_sum(xs, ws)
        req = T.SumRequest(xs, ws, 1e-8, 2, T.Strategy.Krp, T.RngSeed(*sub(seed, 9000)))
        stats = T.SumStats()
        out = T.krp_sum(req, None, stats, engine=engine)
        assert out.ranks == [4, 4, 4]
        assert dense_rel_error(out, ref) <= 1e-8
        assert stats.plan.effective_ranks == [4, 4, 4]


def test_paired_cancellation_keeps_quiet_components(engine):
    """test_sketch_sum.cpp:560-598 (block cores: every summand is a 2-block formal sum)."""
    xs, ws, target = cancellation_instance(40, 10, (107, 0))
    ref = O.reconstruct(target)
    req = T.SumRequest(xs, ws, 1e-6, 2, T.Strategy.Krp, T.RngSeed(107, 1))
    out = T.round_sum(req, engine=engine)
    assert dense_rel_error(out, ref) <= 1e-9
    eff, tg, wd = O.effective_subrank_krp(xs, ws, 1e-6, 2)
    oref, _ = O.krp_sum(xs, ws, wd, (107, 1), 1e-6)
    # The summands cancel by a factor ~1e7 (±1e6-amplitude noise around a unit
    # target), so any two summation orders differ by ~eps·1e7 ≈ 1e-9 relative;
    # the parity bound here is the reference's own bound for this instance
    # (test_sketch_sum.cpp:591), not the 1e-10 of the well-conditioned configs.
    assert rel_diff(out, oref) <= 1e-9


def test_malformed_requests_rejected(engine):
    """test_sketch_sum.cpp:514-547."""
    a = random_tucker([8, 7, 6], [2, 2, 2], (91, 0))
    b = random_tucker([8, 7, 5], [2, 2, 2], (91, 1))
    one_d = random_tucker([9], [2], (91, 2))
    with pytest.raises(ValueError):
        T.krp_sum(T.SumRequest([a, b], [1.0, 1.0], strategy=T.Strategy.Krp), engine=engine)
    with pytest.raises(ValueError):
        T.round_sum(T.SumRequest([], []), engine=engine)
    with pytest.raises(ValueError):
        T.round_sum(T.SumRequest([a], [1.0, 2.0], strategy=T.Strategy.Krp), engine=engine)
    with pytest.raises(ValueError):
        T.round_sum(T.SumRequest([a, None], [1.0, 1.0], strategy=T.Strategy.Krp), engine=engine)
    with pytest.raises(ValueError):
        T.krp_sum(T.SumRequest([one_d], [1.0], strategy=T.Strategy.Krp), engine=engine)
    with pytest.raises(ValueError):
        T.krp_sum(T.SumRequest([a], [1.0], eps=-1.0, strategy=T.Strategy.Krp), engine=engine)
    with pytest.raises(ValueError):
        T.effective_subrank([a], [1.0], 1e-6, [1, 1], T.Strategy.Krp, engine=engine)
    with pytest.raises(ValueError):
        T.effective_subrank([a], [1.0], 1e-6, -1, T.Strategy.Krp, engine=engine)
    # C-ABI level: mismatched batch / weights / widths.
    batch = engine.upload([a])
    with pytest.raises(ValueError):
        engine.krp_sum(batch, [1.0, 2.0], [3, 3, 3], T.RngSeed(1, 1), 1e-8)
    with pytest.raises(ValueError):
        engine.krp_sum(batch, [1.0], [3, 0, 3], T.RngSeed(1, 1), 1e-8)
    with pytest.raises(ValueError):
        engine.krp_sum(batch, [1.0], [3, 3], T.RngSeed(1, 1), 1e-8)
    batch.free()


def test_dispatcher_bitwise_equals_entry_point(engine):
    """test_sketch_sum.cpp:473-491 (Krp) and same-seed bitwise determinism
    (test_ndg_transport.cpp:618-626)."""
    xs = [random_tucker([10, 9, 8], [2, 3, 2], (81, i)) for i in range(3)]
    req = T.SumRequest(xs, [1.0, -0.5, 2.0], 1e-8, 3, T.Strategy.Krp, T.RngSeed(81, 9))
    a = T.round_sum(req, engine=engine)
    b = T.krp_sum(req, engine=engine)
    assert a.ranks == b.ranks
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)
    assert np.array_equal(a.dense_core(), b.dense_core())


def test_plan_matches_oracle_plan(engine):
    """Device effective_subrank == oracle effective_subrank on skewed random instances
    (test_sketch_sum.cpp:372-404 style)."""
    rng = np.random.Generator(np.random.MT19937(4242))
    for it in range(30):
        order = 2 + it % 3
        dims = [2 + int(rng.integers(0, 23)) for _ in range(order)]
        count = 1 + int(rng.integers(0, 5))
        xs, ws = [], []
        for i in range(count):
            ranks = [1 + int(rng.integers(0, min(dims[k], 4))) for k in range(order)]
            xs.append(random_tucker(dims, ranks, (7000 + it, i)))
            ws.append(float(int(rng.integers(0, 5)) - 2.0))
        if all(w == 0 for w in ws):
            ws[0] = 1.0
        eps = 1e-4 if it % 2 == 0 else 1e-8
        p = (it % 3) * 2
        eff, tg, wd = O.effective_subrank_krp(xs, ws, eps, p)
        plan = T.effective_subrank(xs, ws, eps, p, T.Strategy.Krp, engine=engine)
        assert plan.effective_ranks == eff and plan.targets == tg and plan.mode_sketch_dims == wd


def test_general_orders_and_block_cores(engine):
    """d = 2 and d = 5, mixed ranks, block-core summands, n < s."""
    cases = [([30, 25], [4, 3], 5, 9), ([7, 6, 5, 4, 6], [2, 2, 1, 2, 2], 3, 8), ([9, 40, 11], [3, 5, 2], 4, 12)]
    for t, (dims, r, K, s) in enumerate(cases):
        xs = [random_tucker(dims, r, (800 + t, i)) for i in range(K)]
        xs.append(T.tucker_axby(0.5, xs[0], -1.5, xs[1]))
        ws = [1.0, -0.75, 0.5, 2.0, 1.25, 0.3][:len(xs)]
        check_pair(engine, xs, ws, [s] * len(dims), (800 + t, 5), 1e-9, None)


# ------------------------------------------------------------ full-size config 5 properties
def test_cfg5_full_properties(engine):
    """K = 256 at n = 8192: linearity in the weights, bitwise determinism, orthonormal factors."""
    wl = make_workload(5)
    seed = wl.seed
    batch = engine.upload(wl.summands)
    try:
        r1 = engine.krp_sum(batch, wl.weights, wl.widths, seed, 0.0, wl.cap).to_tucker()
        r2 = engine.krp_sum(batch, wl.weights, wl.widths, seed, 0.0, wl.cap).to_tucker()
        r3 = engine.krp_sum(batch, 2.0 * wl.weights, wl.widths, seed, 0.0, wl.cap).to_tucker()
    finally:
        batch.free()
    assert r1.ranks == [48, 48, 48]
    # Stages A, C and E of a sum this large run on the int8 tensor-core engine
    # (ozaki.cu); the parity tests below therefore cover it at full size (stage F2
    # joins them with TS_OZAKI_F2=1: bit 3).
    assert engine.last_int8_stages() & 0b0111 == 0b0111
    for a, b in zip(r1.factors, r2.factors):
        assert np.array_equal(a, b)
    assert np.array_equal(r1.dense_core(), r2.dense_core())
    for f in r1.factors:
        assert np.linalg.norm(f.T @ f - np.eye(f.shape[1])) <= 1e-12
    # 2·sum → 2·result (sketch, QR and truncation are scale-equivariant).
    assert O.rel_error_to_sum(r3, [r1], [2.0]) <= 1e-12


def test_cfg5_full_size_parity(engine):
    """BASELINE config 5 at full size (K = 256, n = 8192, s = 64, cap 48): the
    device result against the CPU oracle on identical inputs and Ω — 1e-10
    relative Frobenius on factors × core, same ranks, and the same error to the
    exact sum to 3 significant digits (Gram-based, both on the oracle)."""
    wl = make_workload(5)
    seed = (wl.seed.seed, wl.seed.stream)
    threads = O.num_threads()
    ref, _ = O.krp_sum(wl.summands, wl.weights, wl.widths, seed, wl.eps, cap=wl.cap, threads=threads)
    out, _ = gpu_sum(engine, wl.summands, wl.weights, wl.widths, seed, wl.eps, wl.cap)
    assert out.ranks == ref.ranks == [48, 48, 48]
    assert rel_diff(out, ref) <= PARITY
    e_gpu = O.rel_error_gram(out, wl.summands, wl.weights, threads)
    e_ref = O.rel_error_gram(ref, wl.summands, wl.weights, threads)
    assert abs(e_gpu - e_ref) <= 5e-4 * e_ref
    # The device error kernel (ts_rel_error_to_sum) agrees.
    batch = engine.upload(wl.summands)
    try:
        res = engine.krp_sum(batch, wl.weights, wl.widths, wl.seed, wl.eps, wl.cap)
        e_dev = engine.rel_error_to_sum(res, batch, wl.weights)
        res.free()
    finally:
        batch.free()
    assert abs(e_dev - e_ref) <= 5e-4 * e_ref


def test_sym_eig_matches_oracle(engine):
    """Device Jacobi eigensolver vs the oracle's sym_eig (test_tensor_kernels.cpp:237-248 style)."""
    for n, seed in [(6, 1), (26, 2), (50, 3), (64, 4), (96, 5)]:
        a = O.gaussian_matrix(2 * n, n, (17, seed))
        c = a.T @ a
        vals, vecs, sweeps, ms = engine.sym_eig(c)
        ov, _ = O.sym_eig(c)
        assert np.max(np.abs(vals - ov)) <= 1e-12 * ov[0]
        assert np.linalg.norm(vecs.T @ vecs - np.eye(n)) <= 1e-12
        assert np.linalg.norm(vecs @ np.diag(vals) @ vecs.T - c) <= 1e-12 * np.linalg.norm(c)
        assert 1 <= sweeps <= 20, sweeps


def test_sym_eig_tri_matches_oracle(engine):
    """The stage-G default eigensolver for n <= 64 (eig_trd.cu: register-resident
    tridiagonalisation, multisection, inverse iteration, Löwdin) vs the oracle's
    sym_eig: Gram matrices, decaying spectra, exact clusters (rank-deficient
    Grams) and tiny sizes.  A rejected result (flag) is recomputed by Jacobi in
    the pipeline; the well-separated Grams must be accepted."""
    cases = []
    for n, seed in [(1, 0), (2, 1), (3, 2), (6, 3), (26, 4), (40, 5), (50, 6), (64, 7)]:
        a = O.gaussian_matrix(2 * n, n, (18, seed))
        cases.append(a.T @ a)
    rng = np.random.default_rng(3)
    for n, decay in [(64, 0.2), (64, 0.5), (26, 1.0)]:
        q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        cases.append((q * 10.0 ** (-decay * np.arange(n))) @ q.T)
    b = O.gaussian_matrix(64, 10, (19, 1))
    cases.append(b @ b.T)  # rank 10: a cluster of 54 zero eigenvalues
    q, _ = np.linalg.qr(rng.standard_normal((48, 48)))
    lam = np.repeat([3.0, 2.0, 1.0, 0.5], 12)
    cases.append((q * lam) @ q.T)  # four 12-fold eigenvalues
    accepted_required = list(range(8))  # the Gram matrices of Gaussian factors
    for ci, c in enumerate(cases):
        n = c.shape[0]
        vals, vecs, rejected, ms = engine.sym_eig_tri(c)
        if ci in accepted_required:
            assert not rejected, (ci, n)
        ov, _ = O.sym_eig(c)
        scale = max(abs(ov[0]), 1e-300)
        assert np.max(np.abs(vals - ov)) <= 1e-13 * scale * max(1, n / 8), (n, np.max(np.abs(vals - ov)))
        if not rejected:
            assert np.linalg.norm(vecs.T @ vecs - np.eye(n)) <= 1e-12
            assert np.linalg.norm(vecs @ np.diag(vals) @ vecs.T - c) <= 1e-12 * np.linalg.norm(c)
    print("tri-eig rejections:", sum(engine.sym_eig_tri(c)[2] for c in cases), "of", len(cases))


def test_accurate_path_hint_is_bitwise_neutral():
    """Config 3 needs the accurate ST-HOSVD path for its parameter modes; after
    the first call a context goes there directly (a performance hint).  Repeated
    calls and a fresh context give bitwise the same result."""
    wl = make_workload(3)
    outs = []
    for fresh in (True, False):
        eng = T.Engine(0)
        try:
            batch = eng.upload(wl.summands)
            runs = 1 if fresh else 3
            for _ in range(runs):
                res = eng.krp_sum(batch, wl.weights, wl.widths, wl.seed, wl.eps, wl.cap)
                outs.append(res.to_tucker())
                res.free()
            assert eng.last_paths()[1] >= 1  # accurate path used
            batch.free()
        finally:
            eng.close()
    for o in outs[1:]:
        assert o.ranks == outs[0].ranks
        assert all(np.array_equal(a, b) for a, b in zip(o.factors, outs[0].factors))
        assert np.array_equal(o.dense_core(), outs[0].dense_core())


def test_plans_for_every_strategy_match_oracle(engine):
    """effective_subrank on the device for Krp / Kron / Lazy / Eager (reference
    src/sketch.cpp:340-346): ranks and targets equal the oracle's; widths follow
    each strategy's rule."""
    xs = [random_tucker([13, 9, 11], [2, 3, 2], (61, i)) for i in range(4)]
    ws = [1.0 + 0.25 * i for i in range(4)]
    eff, tg, wd_krp = O.effective_subrank(xs, ws, 1e-6, 2, strategy="krp")
    _, _, wd_kron = O.effective_subrank(xs, ws, 1e-6, 2, strategy="kron")
    for strat, want in ((T.Strategy.Krp, wd_krp), (T.Strategy.Kron, wd_kron), (T.Strategy.Lazy, tg),
                        (T.Strategy.Eager, tg)):
        plan = T.effective_subrank(xs, ws, 1e-6, 2, strat, engine=engine)
        assert plan.strategy == strat
        assert plan.effective_ranks == eff and plan.targets == tg and plan.mode_sketch_dims == want


@pytest.mark.parametrize("cfg", [1, 4])
def test_stacked_upload_equals_per_summand_upload(engine, cfg):
    """ts_batch_upload_stacked (the workload's host slabs as they are) gives
    bitwise the same sum as ts_batch_upload of the per-summand views."""
    wl = make_workload(cfg)
    d = len(wl.dims)
    outs = []
    for stacked in (False, True):
        batch = engine.upload_stacked(wl.slabs[:d], wl.slabs[d], wl.ranks) if stacked else engine.upload(wl.summands)
        try:
            res = engine.krp_sum(batch, wl.weights, wl.widths, wl.seed, wl.eps, wl.cap)
            outs.append(res.to_tucker())
            res.free()
        finally:
            batch.free()
    a, b = outs
    assert a.ranks == b.ranks
    assert all(np.array_equal(x, y) for x, y in zip(a.factors, b.factors))
    assert np.array_equal(a.dense_core(), b.dense_core())
