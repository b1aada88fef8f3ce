"""CPU oracle for the KRP sketched Tucker summation — TEST INFRASTRUCTURE ONLY.

ctypes bindings for ``oracle/libtucksum_oracle.so`` (built from
``oracle/tucksum_oracle.cpp`` by ``oracle/Makefile``), an Eigen-free C++
restatement of the reference's ``krp_sum`` path (reference
``proj/src/sketch.cpp:66-181``).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this module; the product package never does.

Parity status: the reference cannot be compiled in this image (Eigen >= 3.4 is
absent), so this restatement is pinned by the reference's own
frozen KATs and test assertions (``proj/tests/test_tensor_kernels.cpp``,
``proj/tests/test_tucker_core.cpp``, ``proj/tests/test_sketch_sum.cpp``) restated
in ``tests/test_oracle.py``, by an independent numpy/LAPACK re-derivation of the
pipeline fed with the same Ω, and by Ω being produced by the same libstdc++
``<random>`` the reference uses (bit-identical draws).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtucksum_oracle.so")
_lib = None

i64 = C.c_int64
u64 = C.c_uint64
dptr = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)


class OrTuckerView(C.Structure):
    _fields_ = [
        ("order", i64),
        ("dims", i64p),
        ("ranks", i64p),
        ("factors", C.POINTER(dptr)),
        ("num_blocks", i64),
        ("block_offsets", i64p),
        ("block_shapes", i64p),
        ("block_data", C.POINTER(dptr)),
    ]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "tucksum_oracle.cpp")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        # Passive OpenMP waiting: in a process that also loaded torch (whose own
        # OpenMP runtime keeps spinning threads), active waiting made a 3 ms
        # config-1 call take ~48 ms on 8 threads.  Read by libgomp when it loads.
        os.environ.setdefault("OMP_WAIT_POLICY", "passive")
        L = C.CDLL(_LIB_PATH)
        L.or_last_error.restype = C.c_char_p
        L.or_result_order.restype = i64
        L.or_result_inter.restype = i64
        L.or_num_threads.restype = C.c_int
        L.or_krp_sum.argtypes = [C.POINTER(OrTuckerView), i64, dptr, i64p, i64, u64, u64, C.c_double, i64p,
                                 C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.or_sketched_sum.argtypes = [C.POINTER(OrTuckerView), i64, dptr, i64p, i64, u64, u64, C.c_double, i64p,
                                      C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        for name in ("or_result_order", "or_result_dims", "or_result_ranks", "or_result_widths", "or_result_factor",
                     "or_result_core", "or_result_inter", "or_result_free"):
            getattr(L, name).argtypes = None
        _lib = L
    return _lib


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _check(rc: int):
    if rc != 0:
        msg = lib().or_last_error().decode()
        if rc == 1:
            raise ValueError(msg)  # std::invalid_argument
        raise RuntimeError(msg)


def _p(a: np.ndarray):
    return a.ctypes.data_as(dptr)


def _f64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


class _Views:
    """Keeps the numpy buffers alive while a C call reads the views."""

    def __init__(self, tensors):
        self.keep = []
        self.arr = (OrTuckerView * max(1, len(tensors)))()
        for i, t in enumerate(tensors):
            self.arr[i] = self._view(t)

    def _view(self, t):
        order = len(t.dims)
        dims = np.asarray(t.dims, dtype=np.int64)
        ranks = np.asarray(t.ranks, dtype=np.int64)
        facs = [_f64(f) for f in t.factors]
        fptrs = (dptr * order)(*[_p(f) for f in facs])
        nb = len(t.blocks)
        offs = np.asarray([list(b.offsets) for b in t.blocks], dtype=np.int64).reshape(-1)
        shps = np.asarray([list(np.shape(b.data)) for b in t.blocks], dtype=np.int64).reshape(-1)
        datas = [_f64(b.data) for b in t.blocks]
        bptrs = (dptr * max(1, nb))(*[_p(d) for d in datas])
        self.keep += [dims, ranks, facs, fptrs, offs, shps, datas, bptrs]
        return OrTuckerView(order, dims.ctypes.data_as(i64p), ranks.ctypes.data_as(i64p), fptrs, nb,
                            offs.ctypes.data_as(i64p), shps.ctypes.data_as(i64p), bptrs)

    def ptr(self, i=0):
        return C.pointer(self.arr[i]) if i == 0 else C.cast(C.addressof(self.arr[i]), C.POINTER(OrTuckerView))


# ----------------------------------------------------------------- kernels
def substream(seed: int, stream: int, salt: int):
    s, t = u64(), u64()
    lib().or_substream(u64(seed), u64(stream), u64(salt), C.byref(s), C.byref(t))
    return int(s.value), int(t.value)


def gaussian_matrix(rows: int, cols: int, seed) -> np.ndarray:
    out = np.zeros((rows, cols), dtype=np.float64, order="F")
    _check(lib().or_gaussian_matrix(i64(rows), i64(cols), u64(seed[0]), u64(seed[1]), _p(out)))
    return out


def unfold(t: np.ndarray, mode: int) -> np.ndarray:
    t = _f64(t)
    shape = np.asarray(t.shape, dtype=np.int64)
    rows = t.shape[mode]
    out = np.zeros((rows, t.size // rows), order="F")
    _check(lib().or_unfold(i64(t.ndim), shape.ctypes.data_as(i64p), _p(t), i64(mode), _p(out)))
    return out


def fold(m: np.ndarray, mode: int, shape) -> np.ndarray:
    m = _f64(m)
    sh = np.asarray(shape, dtype=np.int64)
    out = np.zeros(tuple(shape), order="F")
    _check(lib().or_fold(i64(len(shape)), sh.ctypes.data_as(i64p), _p(m), i64(mode), _p(out)))
    return out


def ttm(t: np.ndarray, a: np.ndarray, mode: int) -> np.ndarray:
    t = _f64(t)
    a = _f64(a)
    shape = np.asarray(t.shape, dtype=np.int64)
    out_shape = list(t.shape)
    out_shape[mode] = a.shape[0]
    out = np.zeros(tuple(out_shape), order="F")
    _check(lib().or_ttm(i64(t.ndim), shape.ctypes.data_as(i64p), _p(t), _p(a), i64(a.shape[0]), i64(a.shape[1]),
                        i64(mode), _p(out)))
    return out


def kron(a, b) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    out = np.zeros((a.shape[0] * b.shape[0], a.shape[1] * b.shape[1]), order="F")
    _check(lib().or_kron(i64(a.shape[0]), i64(a.shape[1]), _p(a), i64(b.shape[0]), i64(b.shape[1]), _p(b), _p(out)))
    return out


def khatri_rao(a, b) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    out = np.zeros((a.shape[0] * b.shape[0], a.shape[1]), order="F")
    _check(lib().or_khatri_rao(i64(a.shape[0]), i64(a.shape[1]), _p(a), i64(b.shape[0]), i64(b.shape[1]), _p(b),
                               _p(out)))
    return out


def qr_econ(a):
    a = _f64(a)
    m, n = a.shape
    k = min(m, n)
    q = np.zeros((m, k), order="F")
    r = np.zeros((k, n), order="F")
    _check(lib().or_qr_econ(i64(m), i64(n), _p(a), _p(q), _p(r)))
    return q, r


def svd_econ(a):
    a = _f64(a)
    m, n = a.shape
    k = min(m, n)
    u = np.zeros((m, k), order="F")
    s = np.zeros(k)
    v = np.zeros((n, k), order="F")
    _check(lib().or_svd_econ(i64(m), i64(n), _p(a), _p(u), _p(s), _p(v)))
    return u, s, v


def sym_eig(a):
    a = _f64(a)
    n = a.shape[0]
    if a.shape[0] != a.shape[1]:
        raise ValueError("sym_eig: matrix must be square")
    vals = np.zeros(n)
    vecs = np.zeros((n, n), order="F")
    _check(lib().or_sym_eig(i64(n), _p(a), _p(vals), _p(vecs)))
    return vals, vecs


# ----------------------------------------------------------------- Tucker level
class OracleTucker:
    """Plain Tucker container (dense core, as krp_sum returns)."""

    def __init__(self, core, factors):
        self.core = _f64(core)
        self.factors = [_f64(f) for f in factors]
        self.dims = [f.shape[0] for f in self.factors]
        self.ranks = list(self.core.shape)

        class _B:
            pass

        b = _B()
        b.offsets = [0] * len(self.ranks)
        b.data = self.core
        self.blocks = [b]


def krp_sum(summands, weights, widths=None, seed=(0, 0), eps=1e-8, cap=None, oversampling=5, threads=1,
            intermediates=False, strategy="krp"):
    """Oracle krp_sum (strategy "krp") or kron_sum ("kron"). Returns (OracleTucker, info dict)."""
    L = lib()
    if strategy not in ("krp", "kron"):
        raise ValueError("unknown strategy")
    if len(summands) == 0 or len(summands) != len(weights):
        raise ValueError("sum request needs matching, nonempty summands and weights")  # src/sketch.cpp:18-20
    views = _Views(summands)
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    wid = None if widths is None else np.ascontiguousarray(np.asarray(widths, dtype=np.int64))
    capa = None if cap is None else np.ascontiguousarray(np.asarray(cap, dtype=np.int64))
    h = C.c_void_p()
    rc = L.or_sketched_sum(views.arr, i64(len(summands)), _p(w) if len(w) else dptr(),
                           wid.ctypes.data_as(i64p) if wid is not None else None, i64(oversampling), u64(seed[0]),
                           u64(seed[1]), C.c_double(eps), capa.ctypes.data_as(i64p) if capa is not None else None,
                           C.c_int(threads), C.c_int(1 if intermediates else 0), C.c_int(strategy == "krp"),
                           C.byref(h))
    _check(rc)
    try:
        order = L.or_result_order(h)
        dims = np.zeros(order, dtype=np.int64)
        ranks = np.zeros(order, dtype=np.int64)
        wds = np.zeros(order, dtype=np.int64)
        L.or_result_dims(h, dims.ctypes.data_as(i64p))
        L.or_result_ranks(h, ranks.ctypes.data_as(i64p))
        L.or_result_widths(h, wds.ctypes.data_as(i64p))
        factors = []
        for k in range(order):
            f = np.zeros((dims[k], ranks[k]), order="F")
            L.or_result_factor(h, i64(k), _p(f))
            factors.append(f)
        core = np.zeros(tuple(ranks), order="F")
        L.or_result_core(h, _p(core))
        info = {"widths": [int(x) for x in wds]}
        if intermediates:
            rows, cols = i64(), i64()
            for name, which in (("omega", 0), ("y", 1), ("uhat", 2)):
                mats = []
                for k in range(order):
                    L.or_result_inter(h, C.c_int(which), i64(k), None, C.byref(rows), C.byref(cols))
                    m = np.zeros((rows.value, cols.value), order="F")
                    L.or_result_inter(h, C.c_int(which), i64(k), _p(m), None, None)
                    mats.append(m)
                info[name] = mats
            qd = tuple(m.shape[1] for m in info["uhat"])
            hh = np.zeros(qd, order="F")
            L.or_result_inter(h, C.c_int(3), i64(0), _p(hh), None, None)
            info["h"] = hh
        return OracleTucker(core, factors), info
    finally:
        L.or_result_free(h)


def _result(h, order_hint=None):
    L = lib()
    try:
        order = L.or_result_order(h)
        dims = np.zeros(order, dtype=np.int64)
        ranks = np.zeros(order, dtype=np.int64)
        L.or_result_dims(h, dims.ctypes.data_as(i64p))
        L.or_result_ranks(h, ranks.ctypes.data_as(i64p))
        factors = []
        for k in range(order):
            f = np.zeros((dims[k], ranks[k]), order="F")
            L.or_result_factor(h, i64(k), _p(f))
            factors.append(f)
        core = np.zeros(tuple(ranks), order="F")
        L.or_result_core(h, _p(core))
        return OracleTucker(core, factors)
    finally:
        L.or_result_free(h)


def lazy_sum(summands, weights, eps, cap=None):
    """Oracle lazy_sum: tucker_rounding(formal_sum(summands, weights), eps) (reference
    src/sketch.cpp:48-50, src/tucker.cpp:285-296)."""
    views = _Views(summands)
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    capa = None if cap is None else np.ascontiguousarray(np.asarray(cap, dtype=np.int64))
    h = C.c_void_p()
    _check(lib().or_lazy_sum(views.arr, i64(len(summands)), _p(w) if len(w) else dptr(), C.c_double(eps),
                             capa.ctypes.data_as(i64p) if capa is not None else None, C.byref(h)))
    return _result(h)


def kron_sum(summands, weights, widths=None, **kw):
    """Oracle kron_sum (reference src/sketch.cpp:364-366)."""
    return krp_sum(summands, weights, widths, strategy="kron", **kw)


def kron_sketch_dims(targets, dims):
    """Reference kron_sketch_dims (src/sketch.cpp:222-270)."""
    t = np.ascontiguousarray(np.asarray(targets, dtype=np.int64))
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int64))
    if len(t) != len(d):
        raise ValueError("kron_sketch_dims: need order >= 2 and matching dims")
    out = np.zeros(max(1, len(t)), dtype=np.int64)
    _check(lib().or_kron_sketch_dims(i64(len(t)), t.ctypes.data_as(i64p), d.ctypes.data_as(i64p),
                                     out.ctypes.data_as(i64p)))
    return [int(x) for x in out[:len(t)]]


def effective_subrank_krp(summands, weights, eps, oversampling, strategy="krp"):
    order = len(summands[0].dims)
    ov = np.asarray(oversampling if np.ndim(oversampling) else [oversampling] * order, dtype=np.int64)
    if len(ov) != order:
        raise ValueError("oversampling vector must have one entry per mode")  # src/sketch.cpp:281-283
    eff = np.zeros(order, dtype=np.int64)
    tg = np.zeros(order, dtype=np.int64)
    wd = np.zeros(order, dtype=np.int64)
    views = _Views(summands)
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    _check(lib().or_effective_subrank(views.arr, i64(len(summands)), _p(w), C.c_double(eps),
                                      ov.ctypes.data_as(i64p), C.c_int(strategy == "krp"), eff.ctypes.data_as(i64p),
                                      tg.ctypes.data_as(i64p), wd.ctypes.data_as(i64p)))
    return [int(x) for x in eff], [int(x) for x in tg], [int(x) for x in wd]


def effective_subrank(summands, weights, eps, oversampling, strategy="krp"):
    return effective_subrank_krp(summands, weights, eps, oversampling, strategy)


def partial_sketch(summands, weights, s, seed):
    """Y_n partial sums over `summands` (one shard of the range-finder loop)."""
    views = _Views(summands)
    dims = summands[0].dims
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    out = np.zeros(sum(int(n) * s for n in dims))
    _check(lib().or_partial_sketch(views.arr, i64(len(summands)), _p(w), i64(s), u64(seed[0]), u64(seed[1]), _p(out)))
    ys, off = [], 0
    for n in dims:
        ys.append(out[off:off + n * s].reshape((n, s), order="F"))
        off += n * s
    return ys


def partial_sketch_kron(summands, weights, widths, seed):
    """Kron-sketch Y_n partial sums over `summands` (Y_n: dims[n] × Π_{j≠n} widths[j])."""
    views = _Views(summands)
    dims = summands[0].dims
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    wd = np.ascontiguousarray(np.asarray(widths, dtype=np.int64))
    cols = [int(np.prod([wd[j] for j in range(len(dims)) if j != n])) for n in range(len(dims))]
    out = np.zeros(sum(int(n) * c for n, c in zip(dims, cols)))
    _check(lib().or_partial_sketch_ex(views.arr, i64(len(summands)), _p(w), wd.ctypes.data_as(i64p), C.c_int(0),
                                      u64(seed[0]), u64(seed[1]), _p(out)))
    ys, off = [], 0
    for n, c in zip(dims, cols):
        ys.append(out[off:off + n * c].reshape((n, c), order="F"))
        off += n * c
    return ys


def partial_core(summands, weights, uhat):
    """h partial sum over `summands` projected on the given bases Û_n."""
    views = _Views(summands)
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    us = [_f64(u) for u in uhat]
    uptr = (dptr * len(us))(*[_p(u) for u in us])
    q = np.asarray([u.shape[1] for u in us], dtype=np.int64)
    out = np.zeros(tuple(int(x) for x in q), order="F")
    _check(lib().or_partial_core(views.arr, i64(len(summands)), _p(w), uptr, q.ctypes.data_as(i64p), _p(out)))
    return out


def tucker_norm(x) -> float:
    v = _Views([x])
    out = C.c_double()
    _check(lib().or_tucker_norm(v.arr, C.byref(out)))
    return out.value


def tucker_inner(x, y) -> float:
    vx, vy = _Views([x]), _Views([y])
    out = C.c_double()
    _check(lib().or_tucker_inner(vx.arr, vy.arr, C.byref(out)))
    return out.value


def rel_error_to_sum(x, summands, weights) -> float:
    """tucker_rel_error(x, formal_sum(summands, weights)) — reference src/tucker.cpp:298-303."""
    vx, vs = _Views([x]), _Views(summands)
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    out = C.c_double()
    _check(lib().or_rel_error_to_sum(vx.arr, vs.arr, i64(len(summands)), _p(w), C.byref(out)))
    return out.value


def rel_error_gram(x, summands, weights, threads=1) -> float:
    vx, vs = _Views([x]), _Views(summands)
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    out = C.c_double()
    _check(lib().or_rel_error_gram(vx.arr, vs.arr, i64(len(summands)), _p(w), C.c_int(threads), C.byref(out)))
    return out.value


def reconstruct(x) -> np.ndarray:
    v = _Views([x])
    out = np.zeros(tuple(int(d) for d in x.dims), order="F")
    _check(lib().or_reconstruct(v.arr, _p(out)))
    return out


def num_threads() -> int:
    return int(lib().or_num_threads())
