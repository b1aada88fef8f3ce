"""Segmented independent sums (ts_krp_sum_segmented, the
NDG pattern of reference src/ndg.cpp:401-462: one round_sum per node with a
shared plan).  Every sum of one segmented call must match the CPU oracle run on
that sum alone (1e-10 on factors × core, same ranks) and the single-sum device
call, in BASELINE mode (eps = 0 + cap) and the reference's own mode (eps, no cap)."""
import numpy as np
import pytest

import oracle as O
from paper_2603_13532_b200 import tucksum as T
from paper_2603_13532_b200.workloads import make_workload

pytestmark = pytest.mark.gpu


def nodes(cfg, S, K=None):
    return [make_workload(cfg, K=K, node=i + 1) for i in range(S)]


def seg_inputs(wls):
    xs, ws, seg = [], [], [0]
    for w in wls:
        xs += w.summands
        ws += list(w.weights)
        seg.append(len(xs))
    return xs, np.asarray(ws), seg


@pytest.mark.parametrize("cfg,S,K,eps,cap", [(1, 6, None, 0.0, True), (1, 5, None, 1e-6, False), (4, 4, None, 0.0, True),
                                             (4, 3, None, 1e-6, False), (2, 3, 5, 0.0, True), (3, 3, 6, 1e-10, False)])
def test_segmented_sums_match_oracle_per_sum(engine, cfg, S, K, eps, cap):
    wls = nodes(cfg, S, K)
    xs, ws, seg = seg_inputs(wls)
    widths = wls[0].widths
    mr = wls[0].cap if cap else None
    batch = engine.upload(xs)
    try:
        res = engine.krp_sum_segmented(batch, seg, ws, widths, [w.seed for w in wls], eps, mr)
        outs = [r.to_tucker() for r in res]
        for r in res:
            r.free()
    finally:
        batch.free()
    for w, out in zip(wls, outs):
        ref, _ = O.krp_sum(w.summands, w.weights, widths, (w.seed.seed, w.seed.stream), eps, cap=mr, threads=8)
        assert out.ranks == ref.ranks
        assert O.rel_error_to_sum(out, [ref], [1.0]) <= 1e-10
        # the same sum as a single device call
        b1 = engine.upload(w.summands)
        one = engine.krp_sum(b1, w.weights, widths, w.seed, eps, mr).to_tucker()
        b1.free()
        assert one.ranks == out.ranks
        assert O.rel_error_to_sum(out, [one], [1.0]) <= 1e-12


def test_segmented_rejects_bad_segments(engine):
    wls = nodes(1, 2)
    xs, ws, seg = seg_inputs(wls)
    batch = engine.upload(xs)
    try:
        for bad in ([0, 4, 4, 8], [1, 4, 8], [0, 4, 7]):
            with pytest.raises(ValueError):
                engine.krp_sum_segmented(batch, bad, ws, wls[0].widths, [w.seed for w in wls[:len(bad) - 1]], 0.0,
                                         wls[0].cap)
    finally:
        batch.free()
