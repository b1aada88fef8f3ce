"""The FP64 GEMM on the int8 tensor cores (ozaki.cu, stages A and E of large
sums): accuracy against an extended-precision reference, the digit-range edge
(column maxima just below a power of two — the case a 55-bit fixed point
overflows), zero / tiny / mixed-magnitude columns, and run-to-run bitwise
determinism."""
import numpy as np
import pytest

from paper_2603_13532_b200 import tucksum as T

pytestmark = pytest.mark.gpu


def _ref(f, b):
    return (f.T.astype(np.longdouble) @ b.astype(np.longdouble)).astype(np.float64)


def _check(engine, f, b, tol=2e-15):
    out, _ = engine.ozaki_gemm(f, b)
    ref = _ref(f, b)
    scale = np.abs(f).T @ np.abs(b)
    err = np.abs(out - ref)
    assert np.all(err <= tol * np.maximum(scale, 1e-300)), float(np.max(err / np.maximum(scale, 1e-300)))
    return out


@pytest.mark.parametrize("k,m,n", [(64, 128, 8), (300, 200, 64), (1000, 257, 33), (2048, 640, 64)])
def test_ozaki_matches_extended_precision(engine, k, m, n):
    rng = np.random.default_rng(k + m + n)
    f = np.asfortranarray(rng.standard_normal((k, m)))
    b = np.asfortranarray(rng.standard_normal((k, n)))
    _check(engine, f, b)


def test_ozaki_digit_range_edges(engine):
    """Column maxima at ±(1 − 2^-52)·2^e, exact powers of two, zero and tiny
    columns, 1e±200 magnitudes."""
    rng = np.random.default_rng(7)
    k, m, n = 512, 160, 48
    f = rng.uniform(-1.0, 1.0, size=(k, m))
    b = rng.uniform(-1.0, 1.0, size=(k, n))
    top = 1.0 - 2.0 ** -52
    for j in range(0, m, 4):
        f[j % k, j] = top * 2.0 ** (j % 7)
    for j in range(1, m, 4):
        f[j % k, j] = -top * 2.0 ** (j % 5)
    for j in range(2, m, 8):
        f[:, j] = 0.0
    f[:, 3] *= 1e-200
    f[:, 7] *= 1e200
    for j in range(0, n, 3):
        b[(2 * j) % k, j] = top
        b[(2 * j + 1) % k, j] = -top
    b[:, 5] = 0.0
    b[:, 6] *= 2.0 ** 40
    _check(engine, np.asfortranarray(f), np.asfortranarray(b))


def test_ozaki_bitwise_repeatable(engine):
    rng = np.random.default_rng(3)
    f = np.asfortranarray(rng.standard_normal((4096, 1024)) / 64.0)
    b = np.asfortranarray(rng.standard_normal((4096, 64)))
    first, _ = engine.ozaki_gemm(f, b)
    for _ in range(5):
        assert np.array_equal(first, engine.ozaki_gemm(f, b)[0])


@pytest.mark.parametrize("m,k,n", [(128, 64, 8), (300, 200, 64), (1000, 777, 26), (4096, 1024, 64)])
def test_ozaki_stage_c_orientation(engine, m, k, n):
    """Stage C's orientation (Y = F·W with W stored transposed): A M-contiguous,
    per-row exponents, column-major output."""
    rng = np.random.default_rng(m + k)
    a = np.asfortranarray(rng.standard_normal((m, k)))
    a[5 % m, :] *= 1e-9
    bt = np.asfortranarray(rng.standard_normal((n, k)))
    out, _ = engine.ozaki_gemm_nt(a, bt)
    ref = (a.astype(np.longdouble) @ bt.T.astype(np.longdouble)).astype(np.float64)
    scale = np.abs(a) @ np.abs(bt).T
    assert np.all(np.abs(out - ref) <= 2e-15 * np.maximum(scale, 1e-300))


def test_ozaki_nonfinite_inputs_give_nan(engine):
    """A NaN or Inf anywhere in an operand makes the affected outputs NaN (as an
    FP64 GEMM's would be non-finite) instead of finite garbage from the digit
    conversion; all other outputs stay exact."""
    rng = np.random.default_rng(11)
    k, m, n = 256, 160, 32
    f = np.asfortranarray(rng.standard_normal((k, m)))
    b = np.asfortranarray(rng.standard_normal((k, n)))
    f[17, 5] = np.nan
    f[100, 131] = np.inf
    b[3, 7] = -np.inf
    out, _ = engine.ozaki_gemm(f, b)
    bad_rows = np.zeros(m, dtype=bool)
    bad_rows[[5, 131]] = True
    bad_cols = np.zeros(n, dtype=bool)
    bad_cols[7] = True
    bad = bad_rows[:, None] | bad_cols[None, :]
    assert np.all(np.isnan(out[bad]))
    good = ~bad
    fz, bz = np.nan_to_num(f, nan=0.0, posinf=0.0, neginf=0.0), np.nan_to_num(b, nan=0.0, posinf=0.0, neginf=0.0)
    ref = _ref(fz, bz)
    scale = np.abs(fz).T @ np.abs(bz)
    assert np.all(np.abs(out - ref)[good] <= 2e-15 * np.maximum(scale, 1e-300)[good])
    # stage-C orientation: a non-finite entry of A poisons its row, one of Bt its column
    a = np.asfortranarray(rng.standard_normal((200, 96)))
    bt = np.asfortranarray(rng.standard_normal((24, 96)))
    a[9, 50] = np.nan
    bt[4, 2] = np.inf
    out2, _ = engine.ozaki_gemm_nt(a, bt)
    assert np.all(np.isnan(out2[9, :])) and np.all(np.isnan(out2[:, 4]))
    mask = np.ones_like(out2, dtype=bool)
    mask[9, :] = False
    mask[:, 4] = False
    assert np.all(np.isfinite(out2[mask]))
