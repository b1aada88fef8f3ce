"""Host→device bandwidth from pinned memory with 1/2/4 concurrent copy streams (B200 box)."""
import json, time
import torch
n = 1_677_721_600 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = (n + ns - 1) // ns
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(json.dumps({"probe": "h2d_pinned", "streams": ns, "GB": n * 8 / 1e9, "ms": best * 1e3, "GBps": n * 8 / best / 1e9}))
