"""CUDA-graph replay of repeated identical calls (capi.cu run_sum): replays are
bitwise equal to plain launches, every replay returns an independent result, a
changed weight vector or batch never hits a stale graph, and all three device
strategies (Krp, Kron, Lazy) replay."""
import numpy as np
import pytest

from paper_2603_13532_b200 import tucksum as T
from paper_2603_13532_b200.workloads import make_workload

pytestmark = pytest.mark.gpu


def same(a, b):
    return a.ranks == b.ranks and all(np.array_equal(x, y) for x, y in zip(a.factors, b.factors)) and \
        np.array_equal(a.dense_core(), b.dense_core())


def run(eng, batch, wl, weights, strategy, n, eps=0.0, cap="cfg"):
    outs = []
    cap = wl.cap if cap == "cfg" else cap
    for _ in range(n):
        if strategy == "lazy":
            res = eng.lazy_sum(batch, weights, eps, cap)
        else:
            widths = T.kron_sketch_dims(wl.widths, wl.dims) if strategy == "kron" else wl.widths
            st = T.Strategy.Kron if strategy == "kron" else T.Strategy.Krp
            res = eng.krp_sum(batch, weights, widths, wl.seed, eps, cap, st)
        outs.append(res)
    return outs


@pytest.mark.parametrize("cfg,K,strategy", [(1, None, "krp"), (4, None, "krp"), (2, None, "krp"), (1, None, "kron"), (2, None, "kron"),
                                            (1, None, "lazy")])
def test_graph_replay_bitwise_equal_to_plain_launches(cfg, K, strategy):
    wl = make_workload(cfg, K=K)
    plain = T.Engine(0)
    plain.set_graphs(False)
    graphed = T.Engine(0)
    try:
        bp, bg = plain.upload(wl.summands), graphed.upload(wl.summands)
        ref = [r.to_tucker() for r in run(plain, bp, wl, wl.weights, strategy, 1)]
        res = run(graphed, bg, wl, wl.weights, strategy, 5)
        # plain, plain + capture, then three replays — unless the speculative path
        # was rejected (an accurate-path fallback), which keeps the call unrecorded.
        assert graphed.graph_replays in (0, 3)
        if cfg in (1, 4):
            assert graphed.graph_replays == 3
        outs = [r.to_tucker() for r in res]
        for r in res[:2]:
            r.free()  # freeing earlier results leaves later ones intact
        assert all(same(o, ref[0]) for o in outs)
        assert same(res[4].to_tucker(), ref[0])
        for r in res[2:]:
            r.free()
        # Different weights: a different key, never a stale replay.
        w2 = np.asarray(wl.weights) * np.linspace(0.5, 1.5, len(wl.weights))
        ref2 = run(plain, bp, wl, w2, strategy, 1)[0].to_tucker()
        got2 = [r.to_tucker() for r in run(graphed, bg, wl, w2, strategy, 3)]
        assert all(same(g, ref2) for g in got2)
        # A new upload of the same data is a new batch: plain launches again, same numbers.
        bg2 = graphed.upload(wl.summands)
        before = graphed.graph_replays
        assert same(run(graphed, bg2, wl, wl.weights, strategy, 1)[0].to_tucker(), ref[0])
        assert graphed.graph_replays == before
        bp.free(), bg.free(), bg2.free()
    finally:
        plain.close()
        graphed.close()


@pytest.mark.parametrize("cfg,eps", [(1, 1e-6), (4, 1e-6), (2, 1e-10)])
def test_graph_replay_reference_semantics_eps(cfg, eps):
    """Reference-exact mode (eps > 0, no rank cap) also replays as a CUDA graph:
    the captured ranks are the probe run's, and every replay re-derives the
    reference tail rule on the device (gram_rank_check_kernel) — bitwise equal
    to plain launches."""
    wl = make_workload(cfg)
    plain = T.Engine(0)
    plain.set_graphs(False)
    graphed = T.Engine(0)
    try:
        bp, bg = plain.upload(wl.summands), graphed.upload(wl.summands)
        ref = run(plain, bp, wl, wl.weights, "krp", 1, eps, None)[0].to_tucker()
        res = run(graphed, bg, wl, wl.weights, "krp", 5, eps, None)
        if cfg in (1, 4):
            assert graphed.graph_replays == 3
        for r in res:
            assert same(r.to_tucker(), ref)
            r.free()
        # A different tolerance is a different key (other ranks), never a stale replay.
        ref2 = run(plain, bp, wl, wl.weights, "krp", 1, eps * 1e3, None)[0].to_tucker()
        got2 = [r.to_tucker() for r in run(graphed, bg, wl, wl.weights, "krp", 3, eps * 1e3, None)]
        assert all(same(g, ref2) for g in got2)
        bp.free(), bg.free()
    finally:
        plain.close()
        graphed.close()
