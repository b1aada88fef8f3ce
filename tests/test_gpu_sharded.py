"""World-size-2 run of the PRODUCT's sharded orchestration (capi.cu
sketched_sum_impl: partial Y all-reduced after stage C, replicated QR, partial h
all-reduced after stage F; reference src/sketch.cpp:103-143,155-169).

Only one GPU exists on the test box, so both ranks run on cuda:0 as separate
processes and exchange through the library's host all-reduce hook
(ts_ctx_set_host_allreduce) over gloo — the same two exchange points NCCL serves
on a multi-GPU box; no kernel ever waits on another rank's kernel.  Each rank
generates and uploads only its own shard (workloads.make_workload(k_range=…)).
Both ranks must return the same result, equal to the single-process device
result and the oracle within the parity bar, for BASELINE mode and the
reference-exact mode.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, cfg, K, eps, use_cap):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2603_13532_b200.sharding import init_host_engine, shard_range
    from paper_2603_13532_b200.workloads import make_workload

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = shard_range(K, world, rank)
    wl = make_workload(cfg, K=K, k_range=(b, e))
    eng = init_host_engine(0, rank, world)
    try:
        assert eng.comm_info() == (world, rank)
        batch = eng.upload(wl.summands)
        res = eng.krp_sum(batch, wl.weights, wl.widths, wl.seed, eps, wl.cap if use_cap else None)
        out = res.to_tucker()
        res.free()
        batch.free()
    finally:
        eng.close()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), core=out.dense_core(), ranks=np.asarray(out.ranks),
             **{f"f{j}": f for j, f in enumerate(out.factors)})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,K,eps,use_cap", [(2, 16, 0.0, True), (5, 16, 0.0, True), (1, 4, 1e-6, False),
                                               (3, 30, 1e-10, False)])
def test_two_rank_product_orchestration(tmp_path, cfg, K, eps, use_cap):
    import oracle as O
    from paper_2603_13532_b200 import tucksum as T
    from paper_2603_13532_b200.workloads import make_workload

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), cfg, K, eps, use_cap), nprocs=2, join=True)
    outs = []
    for r in range(2):
        z = np.load(tmp_path / f"rank{r}.npz")
        d = len(z["ranks"])
        outs.append(T.TuckerTensor(z["core"], [z[f"f{j}"] for j in range(d)]))
    # Replicated tail: both ranks hold bitwise the same result.
    assert outs[0].ranks == outs[1].ranks
    assert np.array_equal(outs[0].dense_core(), outs[1].dense_core())
    wl = make_workload(cfg, K=K)
    cap = wl.cap if use_cap else None
    seed = (wl.seed.seed, wl.seed.stream)
    ref, _ = O.krp_sum(wl.summands, wl.weights, wl.widths, seed, eps, cap=cap, threads=8)
    assert outs[0].ranks == ref.ranks
    assert O.rel_error_to_sum(outs[0], [ref], [1.0]) <= 1e-10
    e_sh = O.rel_error_gram(outs[0], wl.summands, wl.weights, 8)
    e_ref = O.rel_error_gram(ref, wl.summands, wl.weights, 8)
    assert abs(e_sh - e_ref) <= 5e-4 * e_ref
