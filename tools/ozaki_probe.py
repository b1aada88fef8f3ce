"""Accuracy / timing probe of the Ozaki-split FP64 GEMM (ozaki.cu) vs numpy:
error relative to |F|ᵀ|B| (the fp64 GEMM error scale) and to ‖FᵀB‖."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13532_b200 import tucksum as T  # noqa: E402

eng = T.Engine(0)
rng = np.random.default_rng(0)
cases = [(64, 128, 8), (256, 128, 64), (1000, 300, 40), (8192, 1024, 64), (8192, 8192, 64)]
for k, m, n in cases:
    f = np.asfortranarray(rng.standard_normal((k, m)) / np.sqrt(k))
    f[:, 1] *= 1e-8  # a tiny column
    b = np.asfortranarray(rng.standard_normal((k, n)))
    for rep in range(2):
        out, ms = eng.ozaki_gemm(f, b)
    if k * m * n <= 3e7:  # extended-precision reference (numpy's own fp64 GEMM error is ~K·ε)
        ref = (f.T.astype(np.longdouble) @ b.astype(np.longdouble)).astype(np.float64)
    else:
        ref = f.T @ b
    scale = np.abs(f).T @ np.abs(b)
    err = np.abs(out - ref)
    print(f"k={k} m={m} n={n}: max err/scale {np.max(err / scale):.2e}  rel fro {np.linalg.norm(out - ref) / np.linalg.norm(ref):.2e}"
          f"  ms {ms:.3f}  TFLOP/s(fp64-equiv) {2.0 * k * m * n / ms / 1e9:.1f}", flush=True)
eng.close()
# determinism / race check: the same product 20 times must be bitwise equal
eng = T.Engine(0)
f = np.asfortranarray(rng.standard_normal((8192, 4096)) / 90.0)
b = np.asfortranarray(rng.standard_normal((8192, 64)))
first, _ = eng.ozaki_gemm(f, b)
same = all(np.array_equal(first, eng.ozaki_gemm(f, b)[0]) for _ in range(20))
print("bitwise repeatable over 20 runs:", same, flush=True)
eng.close()
