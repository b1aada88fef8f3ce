"""Host-side mirror of the reference ``tucksum`` interface for the KRP hot path.

Same names, argument meaning and error behaviour as the reference C++ API
(``/root/reference/proj/include/tucksum/{types,tucker,sketch}.hpp``), backed by
the sm_100a CUDA library through its C ABI (``include/tucksum_cuda.h``).  There
is no CPU fallback: if ``libtucksum_cuda.so`` is missing or no GPU is present the
calls raise.

Reference → here:
  RngSeed / substream          types.hpp:17-24, kernels.cpp:23-25   → RngSeed
  gaussian_matrix              kernels.cpp:88-101                   → gaussian_matrix
  CoreBlock / TuckerTensor     tucker.hpp:13-48, tucker.cpp:16-79   → CoreBlock / TuckerTensor
  formal_sum / tucker_axby     tucker.cpp:183-233                   → formal_sum / tucker_axby (structural)
  Strategy / SketchPlan /      sketch.hpp:18-58                     → same names
  SumRequest / SumStats
  effective_subrank (Krp)      sketch.cpp:272-349                   → effective_subrank
  krp_sum                      sketch.cpp:66-181,360-362            → krp_sum
  round_sum (Strategy::Krp)    sketch.cpp:368-376                   → round_sum
std::invalid_argument maps to ValueError, std::runtime_error to RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TUCKSUM_LIB points at an alternative build of the same library (A/B timing).
LIB_PATH = os.environ.get("TUCKSUM_LIB") or os.path.join(_HERE, "libtucksum_cuda.so")

i64 = C.c_int64
u64 = C.c_uint64
dptr = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)

TS_OK, TS_INVALID_ARGUMENT, TS_RUNTIME, TS_CUDA, TS_NCCL, TS_OOM, TS_UNSUPPORTED = range(7)
MAX_ORDER = 8

# Every symbol include/tucksum_cuda.h declares (checked by the CPU test suite).
EXPORTED_SYMBOLS = [
    "ts_last_error", "ts_version", "ts_ctx_create", "ts_ctx_destroy", "ts_nccl_unique_id", "ts_ctx_init_nccl",
    "ts_ctx_stream", "ts_ctx_launch_count", "ts_batch_upload", "ts_batch_free", "ts_batch_count", "ts_batch_bytes",
    "ts_substream", "ts_gaussian_matrix", "ts_omega_prepare", "ts_krp_sum", "ts_krp_sum_many", "ts_effective_subrank",
    "ts_result_order", "ts_result_dims", "ts_result_ranks", "ts_result_factor", "ts_result_core",
    "ts_result_factor_device", "ts_result_core_device", "ts_result_intermediate", "ts_result_free",
    "ts_ctx_set_debug", "ts_ctx_stage_times", "ts_ctx_set_timing", "ts_ctx_last_paths", "ts_sym_eig",
    "ts_kron_sum", "ts_kron_sketch_dims", "ts_effective_subrank_kron", "ts_lazy_sum",
    "ts_tucker_norm", "ts_tucker_inner", "ts_rel_error_to_sum", "ts_sym_eig_tri",
    "ts_ctx_set_graphs", "ts_ctx_graph_replays", "ts_batch_upload_stacked", "ts_ctx_comm_info",
    "ts_ctx_set_host_allreduce", "ts_krp_sum_segmented", "ts_debug_ozaki_gemm",
    "ts_debug_ozaki_gemm_nt", "ts_ctx_last_int8_stages",
]

HOST_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)


class TucksumCudaError(RuntimeError):
    """CUDA / NCCL / out-of-memory / unsupported-shape failures of the device path."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class TsTuckerView(C.Structure):
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


_lib_handle = None


def lib():
    """Loads libtucksum_cuda.so (raises if it was not built — no fallback)."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run paper_2603_13532_b200/build.py (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.ts_last_error.restype = C.c_char_p
        L.ts_version.restype = C.c_char_p
        L.ts_ctx_stream.restype = C.c_void_p
        L.ts_ctx_stream.argtypes = [C.c_void_p]
        L.ts_ctx_launch_count.restype = i64
        L.ts_ctx_graph_replays.restype = i64
        L.ts_ctx_graph_replays.argtypes = [C.c_void_p]
        L.ts_ctx_set_graphs.argtypes = [C.c_void_p, C.c_int]
        L.ts_ctx_launch_count.argtypes = [C.c_void_p]
        L.ts_batch_count.restype = i64
        L.ts_batch_bytes.restype = i64
        L.ts_batch_bytes.argtypes = [C.c_void_p]
        L.ts_result_order.restype = i64
        L.ts_result_order.argtypes = [C.c_void_p]
        L.ts_result_intermediate.restype = i64
        L.ts_result_factor_device.restype = C.c_void_p
        L.ts_result_core_device.restype = C.c_void_p
        L.ts_krp_sum.argtypes = [C.c_void_p, C.c_void_p, dptr, i64p, u64, u64, C.c_double, i64p,
                                 C.POINTER(C.c_void_p)]
        L.ts_kron_sum.argtypes = L.ts_krp_sum.argtypes
        L.ts_lazy_sum.argtypes = [C.c_void_p, C.c_void_p, dptr, C.c_double, i64p, C.POINTER(C.c_void_p)]
        L.ts_tucker_norm.argtypes = [C.c_void_p, C.c_void_p, dptr, dptr]
        L.ts_tucker_inner.argtypes = [C.c_void_p, C.c_void_p, dptr, C.c_void_p, dptr, dptr]
        L.ts_rel_error_to_sum.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, dptr, dptr]
        L.ts_effective_subrank.argtypes = [C.c_void_p, C.c_void_p, dptr, C.c_double, i64p, i64p, i64p, i64p]
        L.ts_effective_subrank_kron.argtypes = L.ts_effective_subrank.argtypes
        L.ts_kron_sketch_dims.argtypes = [i64, i64p, i64p, i64p]
        L.ts_batch_upload.argtypes = [C.c_void_p, C.POINTER(TsTuckerView), i64, C.POINTER(C.c_void_p)]
        L.ts_omega_prepare.argtypes = [C.c_void_p, i64, i64p, i64, u64, u64]
        L.ts_ctx_set_host_allreduce.argtypes = [C.c_void_p, HOST_ALLREDUCE_FN, C.c_void_p, C.c_int, C.c_int]
        L.ts_krp_sum_segmented.argtypes = [C.c_void_p, C.c_void_p, i64, i64p, dptr, i64p, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint64), C.c_double, i64p, C.POINTER(C.c_void_p)]
        for name in ("ts_result_factor", "ts_result_core", "ts_result_free", "ts_result_dims", "ts_result_ranks",
                     "ts_batch_free", "ts_ctx_destroy", "ts_ctx_set_debug", "ts_ctx_set_timing",
                     "ts_ctx_stage_times", "ts_result_intermediate"):
            getattr(L, name).restype = C.c_int if name not in ("ts_result_dims", "ts_result_ranks") else None
        L.ts_result_intermediate.restype = i64
        _lib_handle = L
    return _lib_handle


def _check(rc: int):
    if rc != TS_OK:
        msg = lib().ts_last_error().decode()
        if rc == TS_INVALID_ARGUMENT:
            raise ValueError(msg)
        if rc == TS_RUNTIME:
            raise RuntimeError(msg)
        raise TucksumCudaError(rc, msg)


def _f64(a) -> np.ndarray:
    if isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.f_contiguous:
        return a
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(dptr)


# ---------------------------------------------------------------------------- RNG
@dataclass(frozen=True)
class RngSeed:
    """Seed plus stream index (reference include/tucksum/types.hpp:17-24)."""

    seed: int = 0
    stream: int = 0

    def substream(self, salt: int) -> "RngSeed":
        s, t = u64(), u64()
        lib().ts_substream(u64(self.seed), u64(self.stream), u64(salt), C.byref(s), C.byref(t))
        return RngSeed(int(s.value), int(t.value))


def gaussian_matrix(rows: int, cols: int, seed: RngSeed) -> np.ndarray:
    """iid N(0,1) rows×cols, column-major fill, bit-identical to the reference stream."""
    out = np.zeros((rows, cols), dtype=np.float64, order="F")
    _check(lib().ts_gaussian_matrix(i64(rows), i64(cols), u64(seed.seed), u64(seed.stream), _p(out)))
    return out


# ---------------------------------------------------------------------------- Tucker
@dataclass
class CoreBlock:
    """Dense sub-core at per-mode offsets (reference include/tucksum/tucker.hpp:13-16)."""

    offsets: List[int]
    data: np.ndarray


class TuckerTensor:
    """Tucker tensor with a (block super-diagonal) core (reference tucker.hpp:22-48).

    ``TuckerTensor(core, factors)`` builds a dense-core tensor;
    ``TuckerTensor(ranks=..., blocks=..., factors=...)`` a block-core one.
    Factors are column-major n_k × r_k float64 arrays; cores are Fortran-ordered
    (first index fastest), matching the reference's DenseTensor buffer.
    """

    def __init__(self, core=None, factors=None, *, ranks=None, blocks=None):
        if factors is None:
            raise ValueError("TuckerTensor: one factor matrix per mode required")
        self.factors = [_f64(f) for f in factors]
        if blocks is None:
            core = _f64(core)
            self.ranks = [int(x) for x in core.shape]
            self.blocks = [CoreBlock([0] * core.ndim, core)]
        else:
            self.ranks = [int(x) for x in ranks]
            self.blocks = [CoreBlock([int(o) for o in b.offsets], _f64(b.data)) for b in blocks]
        self.dims = [int(f.shape[0]) for f in self.factors]
        self._validate()

    def _validate(self):  # reference src/tucker.cpp:16-55
        order = len(self.ranks)
        if order == 0:
            raise ValueError("TuckerTensor: order must be >= 1")
        if len(self.factors) != order:
            raise ValueError("TuckerTensor: one factor matrix per mode required")
        for k in range(order):
            if self.factors[k].ndim != 2 or self.factors[k].shape[1] != self.ranks[k]:
                raise ValueError("TuckerTensor: factor shape must be dims[k] x ranks[k]")
            if self.dims[k] < 1 or self.ranks[k] < 1:
                raise ValueError("TuckerTensor: dims and ranks must be positive")
        if not self.blocks:
            raise ValueError("TuckerTensor: core needs at least one block")
        cursor = [0] * order
        for b in self.blocks:
            if len(b.offsets) != order or b.data.ndim != order:
                raise ValueError("TuckerTensor: block order mismatch")
            for k in range(order):
                if b.offsets[k] != cursor[k]:
                    raise ValueError("TuckerTensor: blocks must tile the super-diagonal")
                cursor[k] += b.data.shape[k]
        if cursor != self.ranks:
            raise ValueError("TuckerTensor: blocks must span the full rank box")

    def order(self) -> int:
        return len(self.ranks)

    def has_dense_core(self) -> bool:
        return len(self.blocks) == 1 and list(self.blocks[0].data.shape) == self.ranks

    def dense_core(self) -> np.ndarray:
        if not self.has_dense_core():
            raise RuntimeError("TuckerTensor::dense_core: core is block-diagonal")
        return self.blocks[0].data

    def core_norm(self) -> float:
        return float(np.sqrt(sum(float(np.sum(b.data * b.data)) for b in self.blocks)))

    def max_rank(self) -> int:
        return max(self.ranks)


def formal_sum(xs: Sequence[TuckerTensor], weights: Sequence[float]) -> TuckerTensor:
    """Concatenate factors, stack scaled cores on the super-diagonal (tucker.cpp:183-226)."""
    if len(xs) == 0 or len(xs) != len(weights):
        raise ValueError("formal_sum: need matching, nonempty summands and weights")
    if any(x is None for x in xs):
        raise ValueError("formal_sum: null summand")
    dims = xs[0].dims
    if any(x.dims != dims for x in xs):
        raise ValueError("formal_sum: all summands must share dims")
    order = len(dims)
    factors = [np.concatenate([x.factors[k] for x in xs], axis=1) for k in range(order)]
    ranks = [sum(x.ranks[k] for x in xs) for k in range(order)]
    blocks, shift = [], [0] * order
    for x, w in zip(xs, weights):
        for b in x.blocks:
            blocks.append(CoreBlock([shift[k] + b.offsets[k] for k in range(order)], b.data * float(w)))
        shift = [shift[k] + x.ranks[k] for k in range(order)]
    return TuckerTensor(ranks=ranks, blocks=blocks, factors=factors)


def save_tucker(dst, x: TuckerTensor) -> None:
    """Reference binary format (src/tucker.cpp:329-352): little-endian u64 order,
    dims, ranks; each factor's column-major doubles; u64 block count; per block
    u64 offsets, u64 extents and the column-major block data.  ``dst`` is a path
    or a binary file object."""
    import struct

    def body(f):
        u64s = lambda vals: f.write(struct.pack("<%dQ" % len(vals), *[int(v) for v in vals]))
        u64s([len(x.dims)])
        u64s(x.dims)
        u64s(x.ranks)
        for fac in x.factors:
            f.write(np.asarray(fac, dtype="<f8").tobytes(order="F"))
        u64s([len(x.blocks)])
        for b in x.blocks:
            u64s(b.offsets)
            u64s(np.shape(b.data))
            f.write(np.asarray(b.data, dtype="<f8").tobytes(order="F"))

    if hasattr(dst, "write"):
        body(dst)
    else:
        with open(dst, "wb") as f:
            body(f)


def load_tucker(src) -> TuckerTensor:
    """Reads the format of save_tucker (reference src/tucker.cpp:354-383); a
    truncated stream raises RuntimeError("load_tucker: truncated stream")."""
    import struct

    def body(f):
        def read(n):
            data = f.read(n)
            if len(data) != n:
                raise RuntimeError("load_tucker: truncated stream")
            return data

        def u64s(k):
            return list(struct.unpack("<%dQ" % k, read(8 * k)))

        order = u64s(1)[0]
        if order == 0 or order > 32:
            raise RuntimeError("load_tucker: implausible order")
        dims, ranks = u64s(order), u64s(order)
        factors = [np.frombuffer(read(8 * n * r), dtype="<f8").reshape((n, r), order="F").copy()
                   for n, r in zip(dims, ranks)]
        blocks = []
        for _ in range(u64s(1)[0]):
            off, shape = u64s(order), u64s(order)
            data = np.frombuffer(read(8 * int(np.prod(shape))), dtype="<f8").reshape(shape, order="F").copy()
            blocks.append(CoreBlock(off, data))
        return TuckerTensor(ranks=ranks, blocks=blocks, factors=factors)

    if hasattr(src, "read"):
        return body(src)
    with open(src, "rb") as f:
        return body(f)


def tucker_axby(alpha: float, x: TuckerTensor, beta: float, y: TuckerTensor) -> TuckerTensor:
    return formal_sum([x, y], [alpha, beta])


# ---------------------------------------------------------------------------- sketch API
class Strategy(enum.Enum):
    Lazy = 0
    Eager = 1
    Krp = 2
    Kron = 3


def strategy_name(s: Strategy) -> str:
    return s.name.lower()


def strategy_from_name(name: str) -> Strategy:
    for s in Strategy:
        if s.name.lower() == name:
            return s
    raise ValueError("unknown strategy name: " + name)


@dataclass
class SketchPlan:
    """Per-mode sketch widths (reference include/tucksum/sketch.hpp:26-39)."""

    strategy: Strategy = Strategy.Krp
    effective_ranks: List[int] = field(default_factory=list)
    oversampling: List[int] = field(default_factory=list)
    targets: List[int] = field(default_factory=list)
    mode_sketch_dims: List[int] = field(default_factory=list)
    eps: float = 0.0
    seed: RngSeed = RngSeed()

    def report(self) -> str:  # reference src/sketch.cpp:203-220
        def fld(v, i):
            return str(v[i]) if i < len(v) else "-"

        lines = [f"summation plan ({strategy_name(self.strategy)}): eps={self.eps:g}, seed=({self.seed.seed},{self.seed.stream})"]
        for n in range(len(self.mode_sketch_dims)):
            line = (f"  mode {n + 1}: effective_rank={fld(self.effective_ranks, n)} oversample="
                    f"{fld(self.oversampling, n)} target={fld(self.targets, n)} sketch_dim={self.mode_sketch_dims[n]}")
            if self.strategy == Strategy.Kron:
                line += f" complement_width={complement_product(self.mode_sketch_dims, n)}"
            lines.append(line)
        return "\n".join(lines) + "\n"


def complement_product(v, skip: int) -> int:
    """Π_{j≠skip} v_j, saturating at 2^50 (reference src/sketch.cpp complement_product)."""
    cap = 1 << 50
    prod = 1
    for j, x in enumerate(v):
        if j == skip:
            continue
        f = max(int(x), 1)
        if prod > cap // f:
            return cap
        prod *= f
    return prod


def kron_sketch_dims(targets, dims) -> List[int]:
    """Kron widths for per-mode targets (reference src/sketch.cpp:222-270), via the C ABI."""
    t = np.ascontiguousarray(np.asarray(targets, dtype=np.int64))
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int64))
    if len(t) != len(d):
        raise ValueError("kron_sketch_dims: need order >= 2 and matching dims")
    out = np.zeros(max(1, len(t)), dtype=np.int64)
    _check(lib().ts_kron_sketch_dims(i64(len(t)), t.ctypes.data_as(i64p), d.ctypes.data_as(i64p),
                                     out.ctypes.data_as(i64p)))
    return [int(x) for x in out[:len(t)]]


@dataclass
class SumRequest:
    """sum_i weights[i] * summands[i] at tolerance eps (reference sketch.hpp:43-50).

    ``max_rank`` is this build's optional per-mode output-rank cap (SURVEY.md
    §8(d)); ``None`` reproduces the reference semantics exactly.
    """

    summands: List[TuckerTensor] = field(default_factory=list)
    weights: List[float] = field(default_factory=list)
    eps: float = 1e-8
    oversampling: int = 5
    strategy: Strategy = Strategy.Lazy
    seed: RngSeed = RngSeed()
    max_rank: Optional[List[int]] = None


@dataclass
class SumStats:
    eager_rank_trace: List[List[int]] = field(default_factory=list)
    plan: SketchPlan = field(default_factory=SketchPlan)
    has_plan: bool = False


# ---------------------------------------------------------------------------- device engine
class _Views:
    """Marshals TuckerTensors into ts_tucker_view structs (keeps buffers alive).

    Shape metadata is shared between summands of equal structure and pointer
    arrays are built from raw addresses: marshalling K = 256 summands must not
    cost more than their PCIe transfer."""

    def __init__(self, tensors: Sequence[TuckerTensor]):
        self.keep = []
        self._meta = {}
        self.arr = (TsTuckerView * max(1, len(tensors)))()
        for i, t in enumerate(tensors):
            if t is None:
                raise ValueError("sum request holds a null summand")
            self.arr[i] = self._view(t)

    def _shape_meta(self, t: TuckerTensor):
        key = (tuple(t.dims), tuple(t.ranks), tuple((tuple(b.offsets), b.data.shape) for b in t.blocks))
        meta = self._meta.get(key)
        if meta is None:
            dims = np.asarray(t.dims, dtype=np.int64)
            ranks = np.asarray(t.ranks, dtype=np.int64)
            offs = np.asarray([b.offsets for b in t.blocks], dtype=np.int64).reshape(-1)
            shps = np.asarray([list(b.data.shape) for b in t.blocks], dtype=np.int64).reshape(-1)
            meta = (dims, ranks, offs, shps, dims.ctypes.data_as(i64p), ranks.ctypes.data_as(i64p),
                    offs.ctypes.data_as(i64p), shps.ctypes.data_as(i64p))
            self._meta[key] = meta
        return meta

    def _view(self, t: TuckerTensor) -> TsTuckerView:
        order = len(t.dims)
        if order > MAX_ORDER:
            raise TucksumCudaError(TS_UNSUPPORTED, "order exceeds TS_MAX_ORDER")
        _, _, _, _, pdims, pranks, poffs, pshps = self._shape_meta(t)
        facs = [_f64(f) for f in t.factors]
        datas = [_f64(b.data) for b in t.blocks]
        fptrs = (C.c_void_p * order)(*[f.ctypes.data for f in facs])
        bptrs = (C.c_void_p * len(datas))(*[x.ctypes.data for x in datas])
        self.keep += [facs, fptrs, datas, bptrs]
        return TsTuckerView(order, pdims, pranks, C.cast(fptrs, C.POINTER(dptr)), len(datas), poffs, pshps,
                            C.cast(bptrs, C.POINTER(dptr)))


class DeviceBatch:
    """Summands resident in HBM in the stacked formal-sum layout (ts_batch)."""

    def __init__(self, engine: "Engine", handle: C.c_void_p, count: int, order: int, dims):
        self.engine, self.handle, self.count, self.order, self.dims = engine, handle, count, order, list(dims)

    @property
    def nbytes(self) -> int:
        return int(lib().ts_batch_bytes(self.handle))

    def free(self):
        if self.handle:
            if self.engine is None or self.engine.handle:  # the context (and its stream) still exists
                lib().ts_batch_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class DeviceResult:
    """A dense-core Tucker tensor in device memory (ts_result)."""

    def __init__(self, handle: C.c_void_p, engine: "Engine" = None):
        self.handle = handle
        self.engine = engine  # results must not outlive their context's stream
        L = lib()
        order = int(L.ts_result_order(handle))
        dims = np.zeros(order, dtype=np.int64)
        ranks = np.zeros(order, dtype=np.int64)
        L.ts_result_dims(handle, dims.ctypes.data_as(i64p))
        L.ts_result_ranks(handle, ranks.ctypes.data_as(i64p))
        self.order, self.dims, self.ranks = order, [int(x) for x in dims], [int(x) for x in ranks]

    def to_tucker(self) -> TuckerTensor:
        L = lib()
        factors = []
        for k in range(self.order):
            f = np.empty((self.dims[k], self.ranks[k]), order="F")
            _check(L.ts_result_factor(self.handle, i64(k), _p(f)))
            factors.append(f)
        core = np.empty(tuple(self.ranks), order="F")
        _check(L.ts_result_core(self.handle, _p(core)))
        return TuckerTensor(core, factors)

    def intermediates(self) -> dict:
        """Stage intermediates captured in debug mode: omega, y, uhat (per mode) and h."""
        L = lib()
        out = {}
        rows, cols = i64(), i64()
        for name, which in (("omega", 0), ("y", 1), ("uhat", 2)):
            mats = []
            for k in range(self.order):
                n = L.ts_result_intermediate(self.handle, C.c_int(which), i64(k), None, C.byref(rows), C.byref(cols))
                m = np.zeros((rows.value, cols.value), order="F")
                if n > 0:
                    L.ts_result_intermediate(self.handle, C.c_int(which), i64(k), _p(m), None, None)
                mats.append(m)
            out[name] = mats
        n = L.ts_result_intermediate(self.handle, C.c_int(3), i64(0), None, C.byref(rows), C.byref(cols))
        h = np.zeros(max(n, 0))
        if n > 0:
            L.ts_result_intermediate(self.handle, C.c_int(3), i64(0), _p(h), None, None)
        qd = tuple(m.shape[1] for m in out["uhat"])
        out["h"] = h.reshape(qd, order="F") if n > 0 else h
        return out

    def free(self):
        if self.handle:
            if self.engine is None or self.engine.handle:  # the context (and its stream) still exists
                lib().ts_result_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Engine:
    """One CUDA device context (stream, scratch pool, Ω cache, optional NCCL comm)."""

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        _check(lib().ts_ctx_create(C.c_int(device), C.byref(h)))
        self.handle = h

    # -- multi-GPU
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().ts_nccl_unique_id(buf))
        return buf.raw

    def init_nccl(self, unique_id: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(unique_id, 128)
        _check(lib().ts_ctx_init_nccl(self.handle, buf, C.c_int(nranks), C.c_int(rank)))

    def set_host_allreduce(self, fn, nranks: int, rank: int):
        """Sharded sums without NCCL: fn(buf: np.ndarray) must sum buf over the
        ranks in place (e.g. a gloo all-reduce); None removes the hook."""
        if fn is None:
            self._host_ar = None
            _check(lib().ts_ctx_set_host_allreduce(self.handle, None, None, C.c_int(1), C.c_int(0)))
            return

        def tramp(_user, buf, count):
            try:
                fn(np.ctypeslib.as_array(buf, shape=(int(count),)))
                return 0
            except Exception:  # noqa: BLE001 — reported to the library as a failed exchange
                return 1

        self._host_ar = HOST_ALLREDUCE_FN(tramp)  # kept alive with the engine
        _check(lib().ts_ctx_set_host_allreduce(self.handle, self._host_ar, None, C.c_int(nranks), C.c_int(rank)))

    def comm_info(self):
        """(nranks, rank) of the context's NCCL communicator (ncclCommCount / ncclCommUserRank)."""
        n, r = C.c_int(), C.c_int()
        _check(lib().ts_ctx_comm_info(self.handle, C.byref(n), C.byref(r)))
        return int(n.value), int(r.value)

    @property
    def stream(self) -> int:
        return int(lib().ts_ctx_stream(self.handle) or 0)

    @property
    def launch_count(self) -> int:
        return int(lib().ts_ctx_launch_count(self.handle))

    def sym_eig(self, a):
        """Device symmetric eigensolver (reference sym_eig): (values desc, vectors, sweeps, ms)."""
        a = _f64(a)
        n = a.shape[0]
        vals = np.zeros(n)
        vecs = np.zeros((n, n), order="F")
        sw = C.c_int()
        ms = C.c_double()
        _check(lib().ts_sym_eig(self.handle, i64(n), _p(a), _p(vals), _p(vecs), C.byref(sw), C.byref(ms)))
        return vals, vecs, int(sw.value), float(ms.value)

    def sym_eig_tri(self, a):
        """Tridiagonalization eigensolver (ts_sym_eig_tri): (values desc, vectors, rejected, ms)."""
        a = _f64(a)
        n = a.shape[0]
        vals = np.zeros(n)
        vecs = np.zeros((n, n), order="F")
        fl = C.c_int()
        ms = C.c_double()
        _check(lib().ts_sym_eig_tri(self.handle, i64(n), _p(a), _p(vals), _p(vecs), C.byref(fl), C.byref(ms)))
        return vals, vecs, bool(fl.value), float(ms.value)

    def last_int8_stages(self) -> int:
        """Bitmask of the last call's stages A (1), C (2), E (4) run on the int8 engine."""
        return int(lib().ts_ctx_last_int8_stages(self.handle))

    def ozaki_gemm(self, f, b):
        """Fᵀ·B on the int8 tensor cores (ts_debug_ozaki_gemm): (result m × n, ms)."""
        f = _f64(f)
        b = _f64(b)
        k, m = f.shape
        n = b.shape[1]
        out = np.zeros((n, m), order="F")
        ms = C.c_double()
        _check(lib().ts_debug_ozaki_gemm(self.handle, i64(k), i64(m), i64(n), _p(f), _p(b), _p(out), C.byref(ms)))
        return out.T.copy(), float(ms.value)

    def ozaki_gemm_nt(self, a, bt):
        """A·Btᵀ on the int8 tensor cores, stage-C orientation (ts_debug_ozaki_gemm_nt): (result, ms)."""
        a = _f64(a)
        bt = _f64(bt)
        m, k = a.shape
        n = bt.shape[0]
        out = np.zeros((m, n), order="F")
        ms = C.c_double()
        _check(lib().ts_debug_ozaki_gemm_nt(self.handle, i64(m), i64(k), i64(n), _p(a), _p(bt), _p(out), C.byref(ms)))
        return out, float(ms.value)

    def set_graphs(self, on: bool):
        """CUDA-graph replay of repeated identical calls (ts_ctx_set_graphs)."""
        _check(lib().ts_ctx_set_graphs(self.handle, 1 if on else 0))

    @property
    def graph_replays(self) -> int:
        return int(lib().ts_ctx_graph_replays(self.handle))

    def last_paths(self):
        """(qr_fallback_modes, svd_fallback_modes) of the last krp_sum."""
        a, b = C.c_int(), C.c_int()
        _check(lib().ts_ctx_last_paths(self.handle, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def set_debug(self, on: bool):
        _check(lib().ts_ctx_set_debug(self.handle, C.c_int(1 if on else 0)))

    def set_timing(self, on: bool):
        _check(lib().ts_ctx_set_timing(self.handle, C.c_int(1 if on else 0)))

    def stage_times(self) -> List[float]:
        buf = (C.c_double * 16)()
        n = lib().ts_ctx_stage_times(self.handle, buf, C.c_int(16))
        return [buf[i] for i in range(n)]

    # -- data
    def upload(self, summands: Sequence[TuckerTensor]) -> DeviceBatch:
        if len(summands) == 0:
            raise ValueError("sum request needs matching, nonempty summands and weights")
        views = _Views(summands)
        h = C.c_void_p()
        _check(lib().ts_batch_upload(self.handle, views.arr, i64(len(summands)), C.byref(h)))
        return DeviceBatch(self, h, len(summands), len(summands[0].dims), summands[0].dims)

    def upload_stacked(self, factor_slabs, core_slab, ranks) -> DeviceBatch:
        """Upload summands already stacked (ts_batch_upload_stacked): factor_slabs[j] is
        dims[j] × Σ_k r_j^(k) (Fortran order), core_slab the dense cores concatenated,
        ranks a K × order integer array."""
        slabs = [np.asarray(f) for f in factor_slabs]
        for f in slabs:
            if f.dtype != np.float64 or not f.flags.f_contiguous:
                raise ValueError("upload_stacked: factor slabs must be Fortran-ordered float64")
        core = np.asarray(core_slab)
        if core.dtype != np.float64 or not core.flags.c_contiguous:
            raise ValueError("upload_stacked: the core slab must be contiguous float64")
        rk = np.ascontiguousarray(np.asarray(ranks, dtype=np.int64))
        order = len(slabs)
        dims = np.ascontiguousarray([f.shape[0] for f in slabs], dtype=np.int64)
        fptrs = (dptr * order)(*[_p(f) for f in slabs])
        h = C.c_void_p()
        _check(lib().ts_batch_upload_stacked(self.handle, i64(order), dims.ctypes.data_as(i64p), i64(rk.shape[0]),
                                             rk.ctypes.data_as(i64p), fptrs, _p(core), C.byref(h)))
        return DeviceBatch(self, h, int(rk.shape[0]), order, [int(x) for x in dims])

    def upload_views(self, views: "C.Array", count: int, order: int, dims) -> DeviceBatch:
        h = C.c_void_p()
        _check(lib().ts_batch_upload(self.handle, views, i64(count), C.byref(h)))
        return DeviceBatch(self, h, count, order, dims)

    def prepare_omega(self, dims, width: int, seed: RngSeed):
        d = np.asarray(dims, dtype=np.int64)
        _check(lib().ts_omega_prepare(self.handle, i64(len(d)), d.ctypes.data_as(i64p), i64(width), u64(seed.seed),
                                      u64(seed.stream)))

    def krp_sum(self, batch: DeviceBatch, weights, widths, seed: RngSeed, eps: float,
                max_rank=None, strategy: "Strategy" = None) -> DeviceResult:
        """ts_krp_sum (or ts_kron_sum when strategy is Strategy.Kron)."""
        kron = strategy == Strategy.Kron
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        if len(w) != batch.count:
            raise ValueError("sum request needs matching, nonempty summands and weights")
        wd = np.ascontiguousarray(np.asarray(widths, dtype=np.int64))
        if len(wd) != batch.order:
            raise ValueError("plan order does not match summand order")
        cap = None if max_rank is None else np.ascontiguousarray(np.asarray(max_rank, dtype=np.int64))
        h = C.c_void_p()
        fn = lib().ts_kron_sum if kron else lib().ts_krp_sum
        _check(fn(self.handle, batch.handle, _p(w), wd.ctypes.data_as(i64p), u64(seed.seed), u64(seed.stream),
                  C.c_double(eps), cap.ctypes.data_as(i64p) if cap is not None else None, C.byref(h)))
        return DeviceResult(h, self)

    def kron_sum(self, batch: DeviceBatch, weights, widths, seed: RngSeed, eps: float, max_rank=None) -> DeviceResult:
        return self.krp_sum(batch, weights, widths, seed, eps, max_rank, Strategy.Kron)

    def tucker_norm(self, batch: DeviceBatch, weights) -> float:
        """‖Σ w_k X_k‖ by the orthogonalized-core norm (ts_tucker_norm)."""
        w = self._weights(batch, weights)
        out = C.c_double()
        _check(lib().ts_tucker_norm(self.handle, batch.handle, _p(w), C.byref(out)))
        return out.value

    def inner(self, bx: DeviceBatch, wx, by: DeviceBatch, wy) -> float:
        """Σ wx_a wy_b <X_a, Y_b> by per-block Gram contractions (ts_tucker_inner)."""
        a, b = self._weights(bx, wx), self._weights(by, wy)
        out = C.c_double()
        _check(lib().ts_tucker_inner(self.handle, bx.handle, _p(a), by.handle, _p(b), C.byref(out)))
        return out.value

    def rel_error_to_sum(self, result: "DeviceResult", batch: DeviceBatch, weights) -> float:
        """‖result − Σ w_k X_k‖ / ‖Σ w_k X_k‖ on the device (ts_rel_error_to_sum)."""
        w = self._weights(batch, weights)
        out = C.c_double()
        _check(lib().ts_rel_error_to_sum(self.handle, result.handle, batch.handle, _p(w), C.byref(out)))
        return out.value

    @staticmethod
    def _weights(batch: DeviceBatch, weights) -> np.ndarray:
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        if len(w) != batch.count:
            raise ValueError("sum request needs matching, nonempty summands and weights")
        return w

    def lazy_sum(self, batch: DeviceBatch, weights, eps: float, max_rank=None) -> DeviceResult:
        """ts_lazy_sum: tucker_rounding(formal_sum(batch, weights), eps) on the device."""
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        if len(w) != batch.count:
            raise ValueError("formal_sum: need matching, nonempty summands and weights")
        cap = None if max_rank is None else np.ascontiguousarray(np.asarray(max_rank, dtype=np.int64))
        h = C.c_void_p()
        _check(lib().ts_lazy_sum(self.handle, batch.handle, _p(w), C.c_double(eps),
                                 cap.ctypes.data_as(i64p) if cap is not None else None, C.byref(h)))
        return DeviceResult(h, self)

    def krp_sum_many(self, batches: Sequence[DeviceBatch], weights: Sequence, widths, seeds: Sequence[RngSeed],
                     eps: float, max_rank=None, lanes: int = 8) -> List[DeviceResult]:
        """Independent sums side by side (ts_krp_sum_many):
        result i equals krp_sum(batches[i], weights[i], widths, seeds[i], eps, max_rank)."""
        n = len(batches)
        if len(weights) != n or len(seeds) != n:
            raise ValueError("krp_sum_many needs one weight vector and one seed per batch")
        ws = []
        for b, w in zip(batches, weights):
            w = np.ascontiguousarray(np.asarray(w, dtype=np.float64))
            if len(w) != b.count:
                raise ValueError("sum request needs matching, nonempty summands and weights")
            ws.append(w)
        wd = np.ascontiguousarray(np.asarray(widths, dtype=np.int64))
        if n and len(wd) != batches[0].order:
            raise ValueError("plan order does not match summand order")
        cap = None if max_rank is None else np.ascontiguousarray(np.asarray(max_rank, dtype=np.int64))
        bh = (C.c_void_p * max(1, n))(*[b.handle for b in batches])
        wp = (dptr * max(1, n))(*[_p(w) for w in ws])
        sd = np.ascontiguousarray([s.seed for s in seeds], dtype=np.uint64)
        st = np.ascontiguousarray([s.stream for s in seeds], dtype=np.uint64)
        out = (C.c_void_p * max(1, n))()
        _check(lib().ts_krp_sum_many(self.handle, i64(n), bh, wp, wd.ctypes.data_as(i64p),
                                     sd.ctypes.data_as(C.POINTER(C.c_uint64)), st.ctypes.data_as(C.POINTER(C.c_uint64)),
                                     C.c_double(eps), cap.ctypes.data_as(i64p) if cap is not None else None,
                                     C.c_int(lanes), out))
        return [DeviceResult(C.c_void_p(out[i]), self) for i in range(n)]

    def krp_sum_segmented(self, batch: DeviceBatch, segments, weights, widths, seeds: Sequence[RngSeed], eps: float,
                          max_rank=None) -> List[DeviceResult]:
        """Segmented independent sums (ts_krp_sum_segmented):
        sum s = the summands [segments[s], segments[s+1]) of `batch`, per-summand
        `weights`, shared plan `widths` / `max_rank`, own seed; every stage runs as
        one launch over all sums."""
        seg = np.ascontiguousarray(np.asarray(segments, dtype=np.int64))
        nsums = len(seg) - 1
        if nsums < 1 or len(seeds) != nsums:
            raise ValueError("krp_sum_segmented needs nsums + 1 segment bounds and one seed per sum")
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        if len(w) != batch.count:
            raise ValueError("sum request needs matching, nonempty summands and weights")
        wd = np.ascontiguousarray(np.asarray(widths, dtype=np.int64))
        if len(wd) != batch.order:
            raise ValueError("plan order does not match summand order")
        cap = None if max_rank is None else np.ascontiguousarray(np.asarray(max_rank, dtype=np.int64))
        sd = np.ascontiguousarray([x.seed for x in seeds], dtype=np.uint64)
        st = np.ascontiguousarray([x.stream for x in seeds], dtype=np.uint64)
        out = (C.c_void_p * nsums)()
        _check(lib().ts_krp_sum_segmented(self.handle, batch.handle, i64(nsums), seg.ctypes.data_as(i64p), _p(w),
                                          wd.ctypes.data_as(i64p), sd.ctypes.data_as(C.POINTER(C.c_uint64)),
                                          st.ctypes.data_as(C.POINTER(C.c_uint64)), C.c_double(eps),
                                          cap.ctypes.data_as(i64p) if cap is not None else None, out))
        return [DeviceResult(C.c_void_p(out[i]), self) for i in range(nsums)]

    def effective_subrank(self, batch: DeviceBatch, weights, eps: float, oversampling, strategy: "Strategy" = None):
        order = batch.order
        ov = np.asarray(oversampling if np.ndim(oversampling) else [oversampling] * order, dtype=np.int64)
        if len(ov) != order:
            raise ValueError("oversampling vector must have one entry per mode")
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        eff, tg, wd = (np.zeros(order, dtype=np.int64) for _ in range(3))
        fn = lib().ts_effective_subrank_kron if strategy == Strategy.Kron else lib().ts_effective_subrank
        _check(fn(self.handle, batch.handle, _p(w), C.c_double(eps), ov.ctypes.data_as(i64p),
                  eff.ctypes.data_as(i64p), tg.ctypes.data_as(i64p), wd.ctypes.data_as(i64p)))
        return [int(x) for x in eff], [int(x) for x in tg], [int(x) for x in wd]

    def close(self):
        if self.handle:
            lib().ts_ctx_destroy(self.handle)
            self.handle = None


_default_engine: Optional[Engine] = None


def default_engine() -> Engine:
    global _default_engine
    if _default_engine is None:
        _default_engine = Engine(int(os.environ.get("TUCKSUM_DEVICE", "0")))
    return _default_engine


# ---------------------------------------------------------------------------- reference entry points
def _validate_request(summands, weights):  # reference src/sketch.cpp:16-30
    if len(summands) == 0 or len(summands) != len(weights):
        raise ValueError("sum request needs matching, nonempty summands and weights")
    if any(x is None for x in summands):
        raise ValueError("sum request holds a null summand")
    dims = summands[0].dims
    if any(x.dims != dims for x in summands):
        raise ValueError("sum request summands must share dims")


def effective_subrank(summands, weights, eps, oversampling, strategy=Strategy.Krp, seed=RngSeed(),
                      engine: Optional[Engine] = None) -> SketchPlan:
    """Plan stage (reference src/sketch.cpp:272-358), on the GPU: Krp → uniform max target,
    Kron → kron_sketch_dims(targets), Lazy / Eager → the targets themselves (:340-346)."""
    _validate_request(summands, weights)
    if eps < 0:
        raise ValueError("tolerance must be nonnegative")
    order = len(summands[0].dims)
    ov = list(oversampling) if np.ndim(oversampling) else [int(oversampling)] * order
    if len(ov) != order:
        raise ValueError("oversampling vector must have one entry per mode")
    if any(p < 0 for p in ov):
        raise ValueError("oversampling must be nonnegative")
    eng = engine or default_engine()
    batch = eng.upload(summands)
    try:
        eff, tg, wd = eng.effective_subrank(batch, weights, eps, ov,
                                            Strategy.Kron if strategy == Strategy.Kron else Strategy.Krp)
    finally:
        batch.free()
    if strategy in (Strategy.Lazy, Strategy.Eager):
        wd = list(tg)
    return SketchPlan(strategy, eff, ov, tg, wd, eps, seed)


def krp_sum(req: SumRequest, plan: Optional[SketchPlan] = None, stats: Optional[SumStats] = None,
            engine: Optional[Engine] = None) -> TuckerTensor:
    """KRP sketched summation (reference src/sketch.cpp:66-181 via krp_sum, :360-362)."""
    return _sketched_sum(req, plan, stats, engine, Strategy.Krp)


def kron_sum(req: SumRequest, plan: Optional[SketchPlan] = None, stats: Optional[SumStats] = None,
             engine: Optional[Engine] = None) -> TuckerTensor:
    """Kronecker sketched summation (reference src/sketch.cpp:66-181 via kron_sum, :364-366)."""
    return _sketched_sum(req, plan, stats, engine, Strategy.Kron)


def _sketched_sum(req, plan, stats, engine, strategy):
    _validate_request(req.summands, req.weights)
    if req.eps < 0:
        raise ValueError("tolerance must be nonnegative")
    order = len(req.summands[0].dims)
    if order < 2:
        raise ValueError("sketched summation needs order >= 2")
    eng = engine or default_engine()
    batch = eng.upload(req.summands)
    try:
        if plan is None:
            ov = [int(req.oversampling)] * order
            if any(p < 0 for p in ov):
                raise ValueError("oversampling must be nonnegative")
            eff, tg, wd = eng.effective_subrank(batch, req.weights, req.eps, ov, strategy)
            plan = SketchPlan(strategy, eff, ov, tg, wd, req.eps, req.seed)
        if len(plan.mode_sketch_dims) != order:
            raise ValueError("plan order does not match summand order")
        if any(s < 1 for s in plan.mode_sketch_dims):
            raise ValueError("plan sketch widths must be positive")
        res = eng.krp_sum(batch, req.weights, plan.mode_sketch_dims, req.seed, req.eps, req.max_rank, strategy)
        out = res.to_tucker()
        res.free()
    finally:
        batch.free()
    if stats is not None:
        stats.plan = plan
        stats.has_plan = True
    return out


def tucker_rounding(x: TuckerTensor, tau: float, engine: Optional[Engine] = None, max_rank=None) -> TuckerTensor:
    """Lazy rounding (reference src/tucker.cpp:285-296) on the device: thin QR of
    every factor, R absorbed into the (block) core, st_hosvd, Q·P (ts_lazy_sum)."""
    if tau < 0:
        raise ValueError("tucker_rounding: tolerance must be nonnegative")
    eng = engine or default_engine()
    batch = eng.upload([x])
    try:
        res = eng.lazy_sum(batch, [1.0], tau, max_rank)
        out = res.to_tucker()
        res.free()
    finally:
        batch.free()
    return out


def tucker_norm(x: TuckerTensor, engine: Optional[Engine] = None) -> float:
    """Reference tucker_norm (src/tucker.cpp:159): orthogonalized-core norm, on the device."""
    eng = engine or default_engine()
    batch = eng.upload([x])
    try:
        return eng.tucker_norm(batch, [1.0])
    finally:
        batch.free()


def tucker_inner(x: TuckerTensor, y: TuckerTensor, engine: Optional[Engine] = None) -> float:
    """Reference tucker_inner (src/tucker.cpp:161-181) on the device."""
    if x.dims != y.dims:
        raise ValueError("tucker_inner: operands must share dims")
    eng = engine or default_engine()
    bx, by = eng.upload([x]), eng.upload([y])
    try:
        return eng.inner(bx, [1.0], by, [1.0])
    finally:
        bx.free()
        by.free()


def tucker_rel_error(x: TuckerTensor, ref: TuckerTensor, engine: Optional[Engine] = None) -> float:
    """Reference tucker_rel_error (src/tucker.cpp:298-303): ‖x − ref‖ / ‖ref‖ with
    both norms orthogonalized on the device (exact cancellation survives)."""
    eng = engine or default_engine()
    bd, br = eng.upload([x, ref]), eng.upload([ref])
    try:
        denom = eng.tucker_norm(br, [1.0])
        diff = eng.tucker_norm(bd, [1.0, -1.0])
    finally:
        bd.free()
        br.free()
    return diff if denom == 0.0 else diff / denom


def lazy_sum(req: SumRequest, engine: Optional[Engine] = None) -> TuckerTensor:
    """Strategy.Lazy (reference src/sketch.cpp:48-50): round the formal sum once."""
    if len(req.summands) == 0 or len(req.summands) != len(req.weights) or any(x is None for x in req.summands):
        raise ValueError("formal_sum: need matching, nonempty summands and weights")
    if any(x.dims != req.summands[0].dims for x in req.summands):
        raise ValueError("formal_sum: all summands must share dims")
    if req.eps < 0:
        raise ValueError("tucker_rounding: tolerance must be nonnegative")
    eng = engine or default_engine()
    batch = eng.upload(req.summands)
    try:
        res = eng.lazy_sum(batch, req.weights, req.eps, req.max_rank)
        out = res.to_tucker()
        res.free()
    finally:
        batch.free()
    return out


def eager_sum(req: SumRequest, stats: Optional[SumStats] = None, engine: Optional[Engine] = None) -> TuckerTensor:
    """Strategy.Eager (reference src/sketch.cpp:52-64): left fold, one device
    rounding per added summand; a single summand comes back scaled, unrounded."""
    _validate_request(req.summands, req.weights)
    if stats is not None:
        stats.eager_rank_trace = []
    acc = formal_sum([req.summands[0]], [req.weights[0]])
    for x, w in zip(req.summands[1:], req.weights[1:]):
        acc = tucker_rounding(tucker_axby(1.0, acc, w, x), req.eps, engine)
        if stats is not None:
            stats.eager_rank_trace.append(list(acc.ranks))
    return acc


def round_sum(req: SumRequest, plan: Optional[SketchPlan] = None, stats: Optional[SumStats] = None,
              engine: Optional[Engine] = None) -> TuckerTensor:
    """Strategy dispatcher (reference src/sketch.cpp:368-376), every strategy on the device."""
    if req.strategy == Strategy.Krp:
        return krp_sum(req, plan, stats, engine)
    if req.strategy == Strategy.Kron:
        return kron_sum(req, plan, stats, engine)
    if req.strategy == Strategy.Lazy:
        return lazy_sum(req, engine)
    if req.strategy == Strategy.Eager:
        return eager_sum(req, stats, engine)
    _validate_request(req.summands, req.weights)
    raise NotImplementedError(f"strategy {strategy_name(req.strategy)} is outside the B200 hot path (SURVEY.md §8)")
