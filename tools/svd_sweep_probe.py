import ctypes as C, json, sys, os
sys.path.insert(0, os.getcwd())
from paper_2603_13532_b200 import tucksum as T
from paper_2603_13532_b200.workloads import make_workload
wl = make_workload(3)
eng = T.Engine(0)
b = eng.upload(wl.summands)
for i in range(3):
    r = eng.krp_sum(b, wl.weights, wl.widths, wl.seed, wl.eps, wl.cap); r.free()
    prof = (C.c_longlong * 32)()
    T.lib().ts_debug_eig_profile(prof)
    print("svd sweeps (last launch):", prof[16])
