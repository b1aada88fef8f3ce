import time, sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2603_13532_b200 import tucksum as T
from paper_2603_13532_b200.workloads import make_workload
wl = make_workload(5)
eng = T.Engine(0)
cudart = torch.cuda.cudart()
for s in wl.slabs:
    cudart.cudaHostRegister(s.ctypes.data, s.nbytes, 0)
xs = wl.summands
for it in range(3):
    t0 = time.perf_counter(); views = T.TuckerViews(xs) if hasattr(T, 'TuckerViews') else None; t1 = time.perf_counter()
    bt = eng.upload(xs); torch.cuda.synchronize(); t2 = time.perf_counter()
    res = eng.krp_sum(bt, wl.weights, wl.widths, wl.seed, wl.eps, wl.cap); t3 = time.perf_counter()
    out = res.to_tucker(); t4 = time.perf_counter()
    res.free(); bt.free(); t5 = time.perf_counter()
    print(f"upload {1e3*(t2-t1):.1f} ms  sum {1e3*(t3-t2):.2f}  to_host {1e3*(t4-t3):.2f}  free {1e3*(t5-t4):.2f}")
# raw H2D of one slab
s = wl.slabs[0]
d = torch.empty(s.nbytes // 8, dtype=torch.float64, device='cuda')
src = torch.from_numpy(s.reshape(-1))
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(src, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"raw H2D {s.nbytes/1e9:.2f} GB in {1e3*(t1-t0):.1f} ms = {s.nbytes/(t1-t0)/1e9:.1f} GB/s")
