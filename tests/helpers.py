"""Shared test helpers: the reference test suites' generators, restated.

Generators follow /root/reference/proj/tests/test_sketch_sum.cpp:17-44,77-115
(random_tucker, orthonormal_cols, dense_weighted_sum, the cancellation
instance) and use the oracle's libstdc++ Gaussian stream, which the product's
``gaussian_matrix`` reproduces bit for bit.
"""
from __future__ import annotations

import numpy as np

import oracle as O
from paper_2603_13532_b200.tucksum import TuckerTensor, tucker_axby


def sub(seed, salt):
    return O.substream(seed[0], seed[1], salt)


def random_tucker(dims, ranks, seed):
    """test_sketch_sum.cpp:17-26."""
    factors = [O.gaussian_matrix(dims[k], ranks[k], sub(seed, 100 + k)) for k in range(len(dims))]
    size = int(np.prod(ranks))
    core = O.gaussian_matrix(size, 1, sub(seed, 999))[:, 0].reshape(ranks, order="F")
    return TuckerTensor(core, factors)


def orthonormal_cols(rows, cols, seed):
    """test_sketch_sum.cpp:28-30."""
    return O.qr_econ(O.gaussian_matrix(rows, cols, seed))[0]


def dense_weighted_sum(xs, ws):
    """test_sketch_sum.cpp:33-44 (independent dense reference)."""
    acc = np.zeros(tuple(xs[0].dims), order="F")
    for x, w in zip(xs, ws):
        acc += w * O.reconstruct(x)
    return acc


def dense_rel_error(approx, ref):
    return float(np.linalg.norm(O.reconstruct(approx) - ref) / np.linalg.norm(ref))


def cancellation_instance(n, pairs, seed):
    """test_sketch_sum.cpp:77-115: rank-5 target hidden in paired ±noise summands."""
    dims = [n, n, n]
    target_diag = [1.0, 0.8, 0.6, 2e-6, 1e-6]
    rt = len(target_diag)
    tf = [orthonormal_cols(n, rt, sub(seed, 10 + k)) for k in range(3)]
    tcore = np.zeros((rt, rt, rt), order="F")
    for j in range(rt):
        tcore[j, j, j] = target_diag[j]
    target = TuckerTensor(tcore, tf)
    rn = 6
    d = 2.0 * pairs
    noise = []
    for i in range(pairs):
        nf = [orthonormal_cols(n, rn, sub(seed, 100 + 7 * i + k)) for k in range(3)]
        ncore = np.zeros((rn, rn, rn), order="F")
        for j in range(rn):
            ncore[j, j, j] = 10.0 ** (6.0 - 11.0 * j / (rn - 1))
        noise.append(TuckerTensor(ncore, nf))
    summands = [tucker_axby(1.0 / d, target, 1.0, noise[i]) for i in range(pairs)]
    summands += [tucker_axby(1.0 / d, target, -1.0, noise[i]) for i in range(pairs)]
    return summands, [1.0] * len(summands), target


def shared_subspace(n, order, latent, count, seed, rank=1, core_salt=None):
    """Summands whose mode factors live in one fixed orthonormal basis
    (test_sketch_sum.cpp:221-264 with rank 1; :301-347 with rank 2)."""
    q = [orthonormal_cols(n[k] if isinstance(n, (list, tuple)) else n, latent, sub(seed, k if core_salt is None else 500 + k))
         for k in range(order)]
    xs = []
    for i in range(count):
        if core_salt is None:
            factors = [q[k] @ O.gaussian_matrix(latent, rank, sub(seed, 1000 + order * i + k)) for k in range(order)]
            core = np.ones([1] * order, order="F") if rank == 1 else None
        else:
            factors = [q[k] @ O.gaussian_matrix(latent, rank, sub(seed, 30 * i + k)) for k in range(order)]
            core = O.gaussian_matrix(rank ** order, 1, sub(seed, 30 * i + 9))[:, 0].reshape([rank] * order, order="F")
        xs.append(TuckerTensor(core, factors))
    return xs
