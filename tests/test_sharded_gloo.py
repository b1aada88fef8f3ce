"""World-size-2 CPU test of the summand-sharded data flow.

Two gloo ranks each take their shard (paper_2603_13532_b200.sharding.shard_range),
build the partial sketches Y on it, all-reduce, QR replicated, build the partial
projected core h, all-reduce — exactly the decomposition ts_krp_sum performs with
NCCL on B200s — and must reproduce the single-process oracle's Y and h.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, strategy="krp"):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle as O
    from paper_2603_13532_b200.sharding import shard_range
    from paper_2603_13532_b200.workloads import make_workload

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = make_workload(2, K=7, n_override=[60, 50, 40])
    b, e = shard_range(wl.K, world, rank)
    xs, ws = wl.summands[b:e], wl.weights[b:e]
    seed = (wl.seed.seed, wl.seed.stream)
    if strategy == "krp":
        s = wl.widths[0]
        ys = O.partial_sketch(xs, ws, s, seed)
    else:  # Kron sketch with the reference's balanced widths
        ys = O.partial_sketch_kron(xs, ws, O.kron_sketch_dims(wl.widths, wl.dims), seed)
    flat = torch.from_numpy(np.concatenate([y.ravel(order="F") for y in ys]))
    dist.all_reduce(flat)
    ys_full, off = [], 0
    for n, y in zip(wl.dims, ys):
        c = y.shape[1]
        ys_full.append(flat[off:off + n * c].numpy().reshape((n, c), order="F"))
        off += n * c
    uh = [O.qr_econ(y)[0] for y in ys_full]
    h = O.partial_core(xs, ws, uh)
    ht = torch.from_numpy(h.ravel(order="F").copy())
    dist.all_reduce(ht)
    if rank == 0:
        np.save(os.path.join(out_dir, "y.npy"), flat.numpy())
        np.save(os.path.join(out_dir, "h.npy"), ht.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("strategy", ["krp", "kron"])
def test_two_rank_sharded_sum_matches_single_process(tmp_path, strategy):
    import oracle as O
    from paper_2603_13532_b200.workloads import make_workload

    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path), strategy), nprocs=2, join=True)
    wl = make_workload(2, K=7, n_override=[60, 50, 40])
    widths = wl.widths if strategy == "krp" else O.kron_sketch_dims(wl.widths, wl.dims)
    _, info = O.krp_sum(wl.summands, wl.weights, widths, (wl.seed.seed, wl.seed.stream), 0.0, cap=wl.cap,
                        intermediates=True, strategy=strategy)
    y = np.load(tmp_path / "y.npy")
    yref = np.concatenate([m.ravel(order="F") for m in info["y"]])
    assert np.linalg.norm(y - yref) <= 1e-13 * np.linalg.norm(yref)
    h = np.load(tmp_path / "h.npy")
    href = info["h"].ravel(order="F")
    assert np.linalg.norm(h - href) <= 1e-12 * np.linalg.norm(href)


@pytest.mark.parametrize("count,world", [(256, 8), (7, 2), (3, 4), (1, 1)])
def test_shard_range_partitions(count, world):
    from paper_2603_13532_b200.sharding import shard_range

    seen = []
    for r in range(world):
        b, e = shard_range(count, world, r)
        seen.extend(range(b, e))
        assert e - b in (count // world, count // world + 1)
    assert seen == list(range(count))
