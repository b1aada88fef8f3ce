"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference publishes no dataset for this path; these generators follow the
recipes of BASELINE.json and SURVEY.md §8(d): orthonormal factor =
thin-Q (R_ii >= 0) of ``gaussian_matrix(n, r, seed')`` (reference
src/bench.cpp:73-75), core = ``gaussian_matrix(prod r, 1, seed'')`` reshaped
column-major (src/bench.cpp:815-825) times the configured decay.  Frozen salts:
base S = RngSeed{2603, cfg}; U_j^(k) ← S.substream(100000 + 16k + j);
G^(k) ← S.substream(900000 + k); weights ← S.substream(7); request seed ←
S.substream(5000).

All summands of one workload live in per-mode slabs (the stacked formal-sum
layout), so a batch upload is one host→device copy per mode.  Summand k depends
only on (cfg, k), so a rank of a sharded run generates (and pins) only its own
contiguous block ``k_range`` of the K summands.

The RNG backend is pluggable: by default the library's host generator
(``ts_substream`` / ``ts_gaussian_matrix``); the reference arm of ``bench.py``
passes the CPU oracle's bit-identical generator instead, so that arm never maps
``libtucksum_cuda.so`` (tests/test_capi_cpu.py checks the two agree bitwise).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Tuple

import numpy as np

from .tucksum import RngSeed, TuckerTensor


@dataclass
class Workload:
    name: str
    cfg: int
    dims: List[int]
    ranks: List[List[int]]           # per summand
    summands: List[TuckerTensor]
    weights: np.ndarray
    widths: List[int]                # plan.mode_sketch_dims (uniform s)
    cap: Optional[List[int]]         # BASELINE target rank (SURVEY.md §8(d) rank cap)
    eps: float
    seed: RngSeed                    # request seed (Ω streams)
    slabs: List[np.ndarray]          # per-mode stacked factors + core slab (host), this shard only
    reps: int = 1                    # repetitions per step (cfg4 time-stepping loop)
    K_total: int = 0                 # summands of the whole job (all shards)
    k_begin: int = 0                 # first summand index of this shard

    @property
    def K(self) -> int:
        """Summands held by this Workload (= K_total unless built for a shard)."""
        return len(self.summands)


def _thin_q(a: np.ndarray) -> np.ndarray:
    q, r = np.linalg.qr(a)
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return np.asfortranarray(q * s)


def _legendre_q(npts: int, deg: int) -> np.ndarray:
    """Thin-Q of Legendre P_0..P_{deg-1} sampled on npts uniform points of [-1, 1]
    (three-term recurrence as reference src/ndg.cpp:17-27)."""
    t = np.linspace(-1.0, 1.0, npts)
    P = np.zeros((npts, deg))
    P[:, 0] = 1.0
    if deg > 1:
        P[:, 1] = t
    for l in range(2, deg):
        P[:, l] = ((2 * l - 1) * t * P[:, l - 1] - (l - 1) * P[:, l - 2]) / l
    return _thin_q(P)


_SPECS = {
    1: dict(name="cfg1_small", dims=[64, 64, 64], K=4, r=[8, 8, 8], s=26, cap=[16, 16, 16], decay=None),
    2: dict(name="cfg2_mid_decaying", dims=[512] * 3, K=16, r=[20, 20, 20], s=40, cap=[30] * 3, decay=("pow10", 12.0)),
    3: dict(name="cfg3_krylov", dims=[4096, 64, 64], K=30, r=[30, 10, 10], s=50, cap=[40, 12, 12], decay=None),
    4: dict(name="cfg4_dg_x100", dims=[256] * 4, K=8, r=[16] * 4, s=26, cap=[16] * 4, decay=("geom", 0.7), reps=100),
    5: dict(name="cfg5_large", dims=[8192] * 3, K=256, r=[32] * 3, s=64, cap=[48] * 3, decay=("pow2", 8.0)),
}


def config_spec(cfg: int) -> dict:
    return dict(_SPECS[cfg])


Gaussian = Callable[[int, int, Tuple[int, int]], np.ndarray]
Substream = Callable[[Tuple[int, int], int], Tuple[int, int]]


def _library_rng() -> Tuple[Gaussian, Substream]:
    from . import tucksum as T

    def gauss(rows, cols, seed):
        return T.gaussian_matrix(rows, cols, T.RngSeed(*seed))

    def sub(seed, salt):
        x = T.RngSeed(*seed).substream(salt)
        return x.seed, x.stream

    return gauss, sub


def make_workload(cfg: int, K: Optional[int] = None, n_override: Optional[List[int]] = None,
                  k_range: Optional[Tuple[int, int]] = None, gaussian: Optional[Gaussian] = None,
                  substream: Optional[Substream] = None, node: int = 0) -> Workload:
    """Builds BASELINE config `cfg` (1..5).  `K` / `n_override` shrink it for parity tests;
    `k_range` = [begin, end) builds only that shard of the K summands; `gaussian` /
    `substream` replace the library's host RNG by a bit-identical one (e.g. the oracle's);
    `node` > 0 draws an independent instance (base seed S.substream(700000 + node)),
    e.g. one sum per NDG node."""
    sp = _SPECS[cfg]
    dims = list(n_override or sp["dims"])
    K = int(K or sp["K"])
    kb, ke = k_range if k_range is not None else (0, K)
    if not 0 <= kb <= ke <= K:
        raise ValueError("make_workload: bad k_range")
    if gaussian is None or substream is None:
        gaussian, substream = _library_rng()
    r = list(sp["r"])
    d = len(dims)
    S = (2603, cfg)
    if node:
        S = substream(S, 700000 + node)
    Kl = ke - kb
    R = [Kl * r[j] for j in range(d)]
    slabs = [np.zeros((dims[j], R[j]), order="F") for j in range(d)]
    core_size = int(np.prod(r))
    core_slab = np.zeros(Kl * core_size)
    idx = np.indices(r).sum(axis=0).astype(np.float64)  # i1 + i2 + ... (0-based)
    decay = sp["decay"]
    if decay is None:
        scale = None
    elif decay[0] == "pow10":
        scale = 10.0 ** (-idx / decay[1])
    elif decay[0] == "pow2":
        scale = 2.0 ** (-idx / decay[1])
    else:
        scale = decay[1] ** idx
    qleg = _legendre_q(dims[1], 10) if cfg == 3 else None
    summands = []
    for k in range(kb, ke):
        kl = k - kb
        factors = []
        for j in range(d):
            g = gaussian(dims[j], r[j], substream(S, 100000 + 16 * k + j))
            if cfg == 3 and j > 0:
                o = _thin_q(g[: r[j], : r[j]])  # random 10×10 orthogonal from the same stream
                f = qleg @ o
            else:
                f = _thin_q(g)
            slabs[j][:, kl * r[j]:(kl + 1) * r[j]] = f
            factors.append(slabs[j][:, kl * r[j]:(kl + 1) * r[j]])
        core = gaussian(core_size, 1, substream(S, 900000 + k)).reshape(r, order="F")
        if scale is not None:
            core = core * scale
        seg = core_slab[kl * core_size:(kl + 1) * core_size]
        seg[:] = core.reshape(-1, order="F")
        summands.append(TuckerTensor(seg.reshape(r, order="F"), factors))
    if cfg == 3:
        weights = gaussian(K, 1, substream(S, 7))[kb:ke, 0].copy()
    else:
        weights = np.ones(Kl)
    widths = [min(sp["s"], max(dims))] * d
    return Workload(name=sp["name"], cfg=cfg, dims=dims, ranks=[list(r) for _ in range(Kl)], summands=summands,
                    weights=weights, widths=widths, cap=list(sp["cap"]), eps=0.0, seed=RngSeed(*substream(S, 5000)),
                    slabs=slabs + [core_slab], reps=int(sp.get("reps", 1)), K_total=K, k_begin=kb)


# The paper's synthetic low-rank sweep (Fig. 2; reference
# runner src/bench.cpp:327-400 with shared_subspace_summands :101-122): N = 4
# modes, n = 4000, d rank-1 summands whose mode-k factors are Q_k·m (Q_k a fixed
# orthonormal 4000 × 10 basis, m ~ N(0, I_10)), unit cores and weights,
# eps = 1e-6, oversampling p = 2, the plan computed inside every call.
FIG2 = dict(name="fig2_synthetic_lowrank", dims=[4000] * 4, d=100, latent=10, eps=1e-6, oversampling=2)


def make_fig2_workload(d: int = 100, n: int = 4000, modes: int = 4, latent: int = 10, trial: int = 0,
                       gaussian: Optional[Gaussian] = None, substream: Optional[Substream] = None) -> Workload:
    """Reference shared_subspace_summands (src/bench.cpp:101-122): bases
    Q_k = thin-Q(gaussian(n, latent, tseed.substream(10 + k))), factor
    U_k^(i) = Q_k · gaussian(latent, 1, tseed.substream(1000 + i·modes + k)),
    core = 1; trial seed tseed = {2603, 6}.substream(trial), request seed
    tseed.substream(5000 + d) (src/bench.cpp:352)."""
    if gaussian is None or substream is None:
        gaussian, substream = _library_rng()
    tseed = substream((2603, 6), trial)
    bases = [_thin_q(gaussian(n, latent, substream(tseed, 10 + k))) for k in range(modes)]
    slabs = [np.zeros((n, d), order="F") for _ in range(modes)]
    core_slab = np.ones(d)
    summands = []
    for i in range(d):
        factors = []
        for k in range(modes):
            slabs[k][:, i:i + 1] = bases[k] @ gaussian(latent, 1, substream(tseed, 1000 + i * modes + k))
            factors.append(slabs[k][:, i:i + 1])
        summands.append(TuckerTensor(core_slab[i:i + 1].reshape([1] * modes, order="F"), factors))
    return Workload(name=FIG2["name"], cfg=6, dims=[n] * modes, ranks=[[1] * modes for _ in range(d)],
                    summands=summands, weights=np.ones(d), widths=[latent + 2] * modes, cap=None, eps=FIG2["eps"],
                    seed=RngSeed(*substream(tseed, 5000 + d)), slabs=slabs + [core_slab], K_total=d)


def f_alg(dims, ranks_per_summand, s, q=None) -> float:
    """Algorithmic FLOPs of stages A+B+C+E+F."""
    d = len(dims)
    q = q or [min(n, s) for n in dims]
    total = 0.0
    for r in ranks_per_summand:
        pr = float(np.prod(r))
        a = sum(2.0 * dims[j] * r[j] * s for j in range(d))
        b = 2.0 * d * pr * s
        c = sum(2.0 * dims[n] * r[n] * s for n in range(d))
        e = sum(2.0 * q[n] * dims[n] * r[n] for n in range(d))
        f = 0.0
        for m in range(d):
            f += 2.0 * q[m] * r[m] * float(np.prod(q[:m])) * float(np.prod(r[m + 1:]))
        total += a + b + c + e + f
    return total
