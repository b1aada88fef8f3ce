"""Where the pipelined e2e step goes: per-step upload duration (on the upload
thread) and sum + download duration (main thread) while they overlap."""
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_13532_b200 import tucksum as T  # noqa: E402
from paper_2603_13532_b200.workloads import make_workload  # noqa: E402

wl = make_workload(5)
eng = T.Engine(0)
up = T.Engine(0)
cudart = torch.cuda.cudart()
for s in wl.slabs:
    cudart.cudaHostRegister(s.ctypes.data, s.nbytes, 0)
d_ = len(wl.dims)
rk = np.asarray([list(r) for r in wl.ranks], dtype=np.int64)
slabs, cores = wl.slabs[:d_], wl.slabs[d_]
pool = ThreadPoolExecutor(max_workers=1)


def up_step():
    t0 = time.perf_counter()
    b = up.upload_stacked(slabs, cores, rk)
    return b, time.perf_counter() - t0


pool.submit(lambda: up_step()[0].free()).result()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
t_all = time.perf_counter()
nxt = pool.submit(up_step)
rows = []
for i in range(steps):
    t0 = time.perf_counter()
    bt, tu = nxt.result()
    t1 = time.perf_counter()
    if i + 1 < steps:
        nxt = pool.submit(up_step)
    res = eng.krp_sum(bt, wl.weights, wl.widths, wl.seed, wl.eps, wl.cap)
    t2 = time.perf_counter()
    out = res.to_tucker()
    t3 = time.perf_counter()
    res.free()
    pool.submit(bt.free)
    rows.append((1e3 * (t1 - t0), 1e3 * tu, 1e3 * (t2 - t1), 1e3 * (t3 - t2)))
pool.submit(lambda: None).result()
tot = 1e3 * (time.perf_counter() - t_all) / steps
for r in rows:
    print("wait-for-upload %.2f ms (upload itself %.2f) | sum %.2f | download %.2f" % r)
print("per step %.2f ms" % tot)
