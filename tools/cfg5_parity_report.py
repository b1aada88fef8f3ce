"""Full-size config 5: device vs oracle numbers for profiles/ (same checks as
tests/test_gpu_parity.py::test_cfg5_full_size_parity, printed)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as O
from paper_2603_13532_b200 import tucksum as T
from paper_2603_13532_b200.workloads import make_workload

wl = make_workload(5)
seed = (wl.seed.seed, wl.seed.stream)
th = O.num_threads()
t0 = time.perf_counter()
ref, _ = O.krp_sum(wl.summands, wl.weights, wl.widths, seed, wl.eps, cap=wl.cap, threads=th)
t1 = time.perf_counter()
eng = T.Engine(0)
b = eng.upload(wl.summands)
res = eng.krp_sum(b, wl.weights, wl.widths, T.RngSeed(*seed), wl.eps, wl.cap)
out = res.to_tucker()
rel = O.rel_error_to_sum(out, [ref], [1.0])
e_gpu = O.rel_error_gram(out, wl.summands, wl.weights, th)
e_ref = O.rel_error_gram(ref, wl.summands, wl.weights, th)
print(json.dumps({"config": wl.name, "ranks_gpu": out.ranks, "ranks_oracle": ref.ranks,
                  "rel_frobenius_gpu_vs_oracle": rel, "err_to_exact_sum_gpu": e_gpu, "err_to_exact_sum_oracle": e_ref,
                  "err_rel_diff": abs(e_gpu - e_ref) / e_ref, "oracle_threads": th, "oracle_seconds": t1 - t0}))
