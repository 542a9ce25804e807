"""Python mirror of the reference's hot-path API (namespace semikern), backed
by the CUDA library through the C-ABI.

Names, argument meaning and error classes follow the reference headers so a
caller (or a test ported from proj/tests/*.cpp) reads the same:

  proj/include/semikern/error.hpp     Error, DimensionError, DomainError,
                                      InvalidArgument, ParseError
  proj/include/semikern/semiring.hpp  Semiring, arithmetic_semiring() ...,
                                      kRelTol, kAbsTol, approx_equal(_scaled)
  proj/include/semikern/matrix.hpp    Triple, DenseMatrix, CsrMatrix, Matrix,
                                      csr_from_triples, to_dense, from_dense,
                                      nnz, storage_bytes, ewise_add/mul, mxm,
                                      dense_mxm_baseline
  proj/include/semikern/dnn.hpp       DnnModel, ForwardOptions, layer_step,
                                      relu_forward, dense_relu_forward,
                                      dense_layer_step

Matrices live in device memory; ``.numpy()`` / ``data()`` download.  The
extensions for the BASELINE workloads (sparse-activation forward, clip,
category set, device-side generators) are at the bottom.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from enum import IntEnum
from typing import Iterable, NamedTuple, Sequence

import numpy as np

from . import _lib
from ._lib import FwdOpts, vp

# ---- errors (error.hpp:24-58) ------------------------------------------------


class Error(RuntimeError):
    """Base class of every exception this library raises."""


class DimensionError(Error):
    pass


class DomainError(Error):
    pass


class InvalidArgument(Error):
    pass


class ParseError(Error):
    pass


class OutOfMemory(Error):
    """Device allocation failed (the bench maps it to a skipped run)."""


class CudaError(Error):
    """CUDA runtime failure, or no usable device."""


_STATUS = {1: Error, 2: DimensionError, 3: DomainError, 4: InvalidArgument, 5: ParseError,
           6: OutOfMemory, 7: CudaError}


def _check(rc: int):
    if rc != 0:
        msg = _lib.load().sk_last_error().decode(errors="replace")
        raise _STATUS.get(rc, Error)(msg)


# ---- semirings (semiring.hpp:32-153) ---------------------------------------------

class SemiringKind(IntEnum):
    arithmetic = 0
    max_plus = 1
    min_max = 2
    gf2 = 3


@dataclass(frozen=True)
class Semiring:
    kind: SemiringKind
    name: str
    zero: float
    one: float


def arithmetic_semiring() -> Semiring:
    return Semiring(SemiringKind.arithmetic, "arithmetic", 0.0, 1.0)


def max_plus_semiring() -> Semiring:
    return Semiring(SemiringKind.max_plus, "maxplus", -math.inf, 0.0)


def min_max_semiring() -> Semiring:
    return Semiring(SemiringKind.min_max, "minmax", math.inf, 0.0)


def gf2_semiring() -> Semiring:
    return Semiring(SemiringKind.gf2, "gf2", 0.0, 1.0)


def semiring_by_name(name: str) -> Semiring:
    table = {"arithmetic": arithmetic_semiring, "maxplus": max_plus_semiring,
             "minmax": min_max_semiring, "gf2": gf2_semiring}
    if name not in table:
        raise InvalidArgument(f"unknown semiring '{name}' (expected arithmetic|maxplus|minmax|gf2)")
    return table[name]()


kRelTol = np.float32(1e-5)
kAbsTol = np.float32(1e-6)


def approx_equal(x, y) -> bool:
    x, y = np.float32(x), np.float32(y)
    if x == y:
        return True
    return abs(x - y) <= max(kAbsTol, kRelTol * max(abs(x), abs(y)))


def approx_equal_scaled(x, y, scale) -> bool:
    x, y = np.float32(x), np.float32(y)
    if x == y:
        return True
    return abs(x - y) <= max(kAbsTol, kRelTol * np.float32(scale))


# ---- device context ------------------------------------------------------------------

LAYER_PATHS = ("empty", "exact", "esc", "engine", "dense")  # SK_PATH_* (sk_api.h)


class Context:
    """One CUDA device + stream (sk_ctx)."""

    def __init__(self, device: int = 0):
        self._L = _lib.load()
        h = vp()
        _check(self._L.sk_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def synchronize(self):
        _check(self._L.sk_ctx_synchronize(self.h))

    def set_timing(self, enable: bool):
        _check(self._L.sk_ctx_set_timing(self.h, int(enable)))

    def kernel_times_ms(self) -> np.ndarray:
        """Durations (ms) of the dominant-kernel launches recorded since
        set_timing(True) / the last call (CUDA events on this context's stream)."""
        cap = 1 << 16
        buf = np.zeros(cap, np.float32)
        n = C.c_size_t()
        _check(self._L.sk_ctx_kernel_times(self.h, buf.ctypes.data_as(_lib.f32p), cap,
                                           C.byref(n)))
        return buf[: min(n.value, cap)].copy()

    KERNEL_TAGS = {0: "other", 1: "k_exact_layer", 2: "k_sparse_engine", 3: "k_dense_engine",
                   4: "k_spmm_rows", 5: "k_gemm_packed", 6: "k_spgemm_rows", 7: "k_push_layer",
                   8: "k_exact_stream"}

    def kernel_times_tagged(self):
        """(durations ms, kernel names) of the timed launches since
        set_timing(True) / the last call; resets the list."""
        cap = 1 << 16
        buf = np.zeros(cap, np.float32)
        tags = np.zeros(cap, np.int32)
        n = C.c_size_t()
        _check(self._L.sk_ctx_kernel_times_tagged(self.h, buf.ctypes.data_as(_lib.f32p),
                                                  tags.ctypes.data_as(C.POINTER(C.c_int)), cap,
                                                  C.byref(n)))
        k = min(n.value, cap)
        return buf[:k].copy(), [self.KERNEL_TAGS.get(int(t), "other") for t in tags[:k]]

    def layer_stamps_ns(self, n: int) -> np.ndarray:
        """%globaltimer stamps of the last sparse forward: start + end of each layer."""
        buf = np.zeros(n, np.int64)
        _check(self._L.sk_ctx_layer_stamps(self.h, buf.ctypes.data_as(C.POINTER(C.c_longlong)), n))
        return buf

    def layer_paths(self, n: int) -> list:
        """Path names the first n layers of the last sparse forward took: "empty"
        (no work: empty input, biases <= 0), "exact", "esc", "engine", "dense"."""
        buf = np.zeros(max(n, 1), np.uint8)
        _check(self._L.sk_ctx_layer_paths(self.h, buf.ctypes.data_as(C.POINTER(C.c_ubyte)), n))
        return [LAYER_PATHS[int(x)] for x in buf[:n]]

    def set_density_switch(self, dense_above: float = 1.0 / 32, sparse_below: float = 1.0 / 128):
        """Activation density (fraction of m*n) above which relu_forward_sparse
        continues on the dense engine, and below which it returns to the sparse
        one.  dense_above <= 0 keeps the whole pass sparse.  Bitwise neutral."""
        _check(self._L.sk_ctx_set_density_switch(self.h, float(dense_above), float(sparse_below)))

    TUNING_KEYS = ("exact", "exact_kernel", "exact_group", "exact_records", "window_log2",
                   "exact_window_log2", "esc", "esc_ratio", "exact_fields", "exact_layout")

    def tuning(self) -> dict:
        """The context's kernel selection (sk_tuning; 0 = automatic)."""
        t = _lib.Tuning()
        _check(self._L.sk_ctx_get_tuning(self.h, C.byref(t)))
        return {k: getattr(t, k) for k in self.TUNING_KEYS}

    def set_tuning(self, **kw) -> dict:
        """Select kernel variants (sk_ctx_set_tuning): keys not given keep their
        value; returns the previous setting so callers can restore it.  Every
        choice computes the same fold bit for bit."""
        old = self.tuning()
        for k in kw:
            if k not in self.TUNING_KEYS:
                raise InvalidArgument(f"unknown tuning key {k!r}")
        new = dict(old, **kw)
        t = _lib.Tuning(**{k: (float(v) if k == "esc_ratio" else int(v)) for k, v in new.items()})
        _check(self._L.sk_ctx_set_tuning(self.h, C.byref(t)))
        return old

    def last_exact(self) -> dict:
        """What the last exact-layer launch ran (sk_ctx_last_exact): kernel
        ("generic" / "specialised"), windows per item, records per batch, window
        log2, accumulator fields per word, and the launch count."""
        e = _lib.ExactInfo()
        _check(self._L.sk_ctx_last_exact(self.h, C.byref(e)))
        return {"launches": int(e.launches),
                "kernel": {0: None, 1: "generic", 2: "specialised", 3: "push",
                           4: "flat", 5: "stream"}[e.kernel],
                "group": e.group, "records": e.records, "window_log2": e.window_log2,
                "fields": e.fields, "wraps": e.wraps,
                "layout": {0: "direct", 1: "padded", 3: "banked"}[e.layout]}

    def set_stream(self, stream_ptr: int | None):
        _check(self._L.sk_ctx_set_stream(self.h, vp(stream_ptr) if stream_ptr else None))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self._L.sk_ctx_destroy(self.h)
        except Exception:
            pass


_default_ctx: dict[int, Context] = {}
_current_device = 0


def set_device(device: int):
    global _current_device
    _current_device = device


def default_context() -> Context:
    if _current_device not in _default_ctx:
        _default_ctx[_current_device] = Context(_current_device)
    return _default_ctx[_current_device]


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


# ---- matrices (matrix.hpp:29-137) ---------------------------------------------------------

class Triple(NamedTuple):
    row: int
    col: int
    value: float


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


class DenseMatrix:
    """Row-major dense matrix in device memory; zeros are explicit."""

    def __init__(self, rows: int = 0, cols: int = 0, fill=0.0, *, ctx: Context | None = None,
                 _handle=None):
        self.ctx = _ctx(ctx)
        L = self.ctx._L
        if _handle is not None:
            self.h = _handle
        elif isinstance(fill, (list, tuple, np.ndarray)):
            data = _f32(fill).reshape(-1)
            if data.size != rows * cols:
                raise InvalidArgument(f"dense data length {data.size} does not equal rows*cols "
                                      f"for {rows}x{cols}")
            h = vp()
            _check(L.sk_dense_upload(self.ctx.h, rows, cols, data.ctypes.data, C.byref(h)))
            self.h = h
        else:
            h = vp()
            _check(L.sk_dense_create(self.ctx.h, rows, cols, float(fill), C.byref(h)))
            self.h = h
        r, c = C.c_uint32(), C.c_uint32()
        _check(L.sk_dense_shape(self.h, C.byref(r), C.byref(c)))
        self._rows, self._cols = r.value, c.value

    @classmethod
    def from_numpy(cls, a, ctx: Context | None = None) -> "DenseMatrix":
        a = _f32(a)
        if a.ndim != 2:
            raise InvalidArgument("expected a 2-D array")
        return cls(a.shape[0], a.shape[1], a, ctx=ctx)

    @staticmethod
    def identity(n: int, ctx: Context | None = None) -> "DenseMatrix":
        c = _ctx(ctx)
        h = vp()
        _check(c._L.sk_dense_identity(c.h, n, C.byref(h)))
        return DenseMatrix(ctx=c, _handle=h)

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    @property
    def shape(self):
        return (self._rows, self._cols)

    def numpy(self) -> np.ndarray:
        out = np.empty((self._rows, self._cols), np.float32)
        _check(self.ctx._L.sk_dense_download(self.ctx.h, self.h, out.ctypes.data))
        return out

    data = numpy

    def __call__(self, i: int, j: int) -> float:
        return float(self.numpy()[i, j])

    def write(self, a):
        """Overwrite the values in place from a host array of the same shape
        (sk_dense_write; stream-ordered).  Invalidates derived device copies."""
        a = np.ascontiguousarray(a, np.float32)
        if a.shape != (self.rows(), self.cols()):
            raise DimensionError(f"write of {a.shape} into {self.rows()}x{self.cols()}")
        _check(self.ctx._L.sk_dense_write(self.ctx.h, self.h, a.ctypes.data))
        self.ctx.synchronize()  # the host array is borrowed

    def device_ptr(self) -> int:
        return int(self.ctx._L.sk_dense_device_ptr(self.h) or 0)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx._L.sk_dense_free(self.h)
        except Exception:
            pass


class CsrMatrix:
    """CSR matrix in device memory (u32 row_ptr/col_idx, f32 values)."""

    def __init__(self, rows: int, cols: int, row_ptr=None, col_idx=None, values=None, *,
                 validate: bool = True, ctx: Context | None = None, _handle=None):
        self.ctx = _ctx(ctx)
        L = self.ctx._L
        if _handle is not None:
            self.h = _handle
        else:
            rp = _u32(row_ptr if row_ptr is not None else [0] * (rows + 1))
            ci = _u32(col_idx if col_idx is not None else [])
            v = _f32(values if values is not None else [])
            if validate:
                # checks the reference performs before touching the arrays (matrix.cpp:96-102)
                if rp.size != rows + 1:
                    raise InvalidArgument("row_ptr length must be rows+1")
                if rp[0] != 0:
                    raise InvalidArgument("row_ptr[0] must be 0")
                if rp[-1] != ci.size or ci.size != v.size:
                    raise InvalidArgument("row_ptr[rows], col_idx and values disagree on nnz")
            h = vp()
            _check(L.sk_csr_from_parts(self.ctx.h, rows, cols, rp.ctypes.data, ci.ctypes.data,
                                       v.ctypes.data, int(validate), C.byref(h)))
            self.h = h
        r, c, n = C.c_uint32(), C.c_uint32(), C.c_size_t()
        _check(L.sk_csr_shape(self.h, C.byref(r), C.byref(c), C.byref(n)))
        self._rows, self._cols, self._nnz = r.value, c.value, n.value
        self._host = None

    @staticmethod
    def from_parts_unchecked(rows, cols, row_ptr, col_idx, values, ctx=None) -> "CsrMatrix":
        return CsrMatrix(rows, cols, row_ptr, col_idx, values, validate=False, ctx=ctx)

    @staticmethod
    def from_pattern(rows, cols, row_ptr, col_idx, value: float = 1.0, *, validate=True,
                     ctx=None) -> "CsrMatrix":
        """Pattern-only upload: every stored value is `value` (set on the device),
        so only row_ptr and col_idx cross the host link (binary activations)."""
        c = _ctx(ctx)
        rp, ci = _u32(row_ptr), _u32(col_idx)
        if validate:
            if rp.size != rows + 1:
                raise InvalidArgument("row_ptr length must be rows+1")
            if rp[0] != 0:
                raise InvalidArgument("row_ptr[0] must be 0")
            if rp[-1] != ci.size:
                raise InvalidArgument("row_ptr[rows] and col_idx disagree on nnz")
        h = vp()
        _check(c._L.sk_csr_from_pattern(c.h, rows, cols, rp.ctypes.data, ci.ctypes.data,
                                        float(value), int(validate), C.byref(h)))
        return CsrMatrix(rows, cols, ctx=c, _handle=h)

    @staticmethod
    def from_pattern_async(rows, cols, row_ptr, col_idx, value: float = 1.0, *, stream: int,
                           ctx=None) -> "CsrMatrix":
        """from_pattern (unvalidated) with the copies on `stream` (a cudaStream_t
        handle, e.g. torch.cuda.Stream().cuda_stream): they overlap work already
        queued on the context's stream, and every later use of the matrix is
        ordered after them.  The host arrays are kept alive by the returned
        matrix; page-locked arrays (host_register) make the copies asynchronous."""
        c = _ctx(ctx)
        rp, ci = _u32(row_ptr), _u32(col_idx)
        if rp.size != rows + 1:
            raise InvalidArgument("row_ptr length must be rows+1")
        h = vp()
        _check(c._L.sk_csr_from_pattern_async(c.h, rows, cols, rp.ctypes.data, ci.ctypes.data,
                                              float(value), vp(stream), C.byref(h)))
        m = CsrMatrix(rows, cols, ctx=c, _handle=h)
        m._host_refs = (rp, ci)
        return m

    @staticmethod
    def from_pattern16_async(rows, cols, row_ptr, col_idx16, value: float = 1.0, *, stream: int,
                             ctx=None) -> "CsrMatrix":
        """from_pattern_async with 16-bit column indices (cols <= 65536): half the
        bytes over the host link; widened on the device (sk_csr_from_pattern16_async)."""
        c = _ctx(ctx)
        rp = _u32(row_ptr)
        ci = np.ascontiguousarray(col_idx16, dtype=np.uint16)
        if rp.size != rows + 1:
            raise InvalidArgument("row_ptr length must be rows+1")
        h = vp()
        _check(c._L.sk_csr_from_pattern16_async(c.h, rows, cols, rp.ctypes.data, ci.ctypes.data,
                                                float(value), vp(stream), C.byref(h)))
        m = CsrMatrix(rows, cols, ctx=c, _handle=h)
        m._host_refs = (rp, ci)
        return m

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def nnz(self) -> int:
        return self._nnz

    def extract(self):
        """extractTuples: host copies of (row_ptr, col_idx, values)."""
        if self._host is None:
            rp = np.empty(self._rows + 1, np.uint32)
            ci = np.empty(max(self._nnz, 1), np.uint32)
            v = np.empty(max(self._nnz, 1), np.float32)
            _check(self.ctx._L.sk_csr_extract(self.ctx.h, self.h, rp.ctypes.data, ci.ctypes.data,
                                              v.ctypes.data))
            self._host = (rp, ci[: self._nnz], v[: self._nnz])
        return self._host

    def row_ptr(self) -> np.ndarray:
        return self.extract()[0]

    def col_idx(self) -> np.ndarray:
        return self.extract()[1]

    def values(self) -> np.ndarray:
        return self.extract()[2]

    def row_cols(self, i: int) -> np.ndarray:
        rp, ci, _ = self.extract()
        return ci[rp[i]:rp[i + 1]]

    def row_values(self, i: int) -> np.ndarray:
        rp, _, v = self.extract()
        return v[rp[i]:rp[i + 1]]

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx._L.sk_csr_free(self.h)
        except Exception:
            pass


class Matrix:
    """Either representation behind uniform accessors (matrix.hpp:120-137)."""

    def __init__(self, m):
        if isinstance(m, Matrix):
            m = m._rep
        if not isinstance(m, (CsrMatrix, DenseMatrix)):
            raise InvalidArgument("Matrix holds a CsrMatrix or a DenseMatrix")
        self._rep = m

    def is_sparse(self) -> bool:
        return isinstance(self._rep, CsrMatrix)

    def rows(self) -> int:
        return self._rep.rows()

    def cols(self) -> int:
        return self._rep.cols()

    def csr(self) -> CsrMatrix:
        if not self.is_sparse():
            raise Error("matrix holds a dense representation")
        return self._rep

    def dense(self) -> DenseMatrix:
        if self.is_sparse():
            raise Error("matrix holds a sparse representation")
        return self._rep


# ---- Matrix Market exchange (matio.hpp) ------------------------------------------------


class MatrixFileKind(IntEnum):
    coordinate = 0
    array = 1


@dataclass
class MatrixFileInfo:  # matio.hpp:32-38
    path: str | None
    kind: MatrixFileKind
    rows: int
    cols: int
    entries: int


def _from_read(c, kind, hc, hd) -> "Matrix":
    if kind.value == 0:
        return Matrix(CsrMatrix(0, 0, ctx=c, _handle=hc))
    return Matrix(DenseMatrix(0, 0, ctx=c, _handle=hd))


def read_matrix(src, ctx: Context | None = None) -> "Matrix":
    """read_matrix(path) or read_matrix(file-like) (matio.hpp:46-51): coordinate
    files yield CSR, array files dense; ParseError carries "line N: ..."."""
    c = _ctx(ctx)
    kind, hc, hd = C.c_int(), vp(), vp()
    if hasattr(src, "read"):
        text = src.read()
        data = text.encode() if isinstance(text, str) else bytes(text)
        _check(c._L.sk_read_matrix_text(c.h, data, len(data), C.byref(kind), C.byref(hc),
                                        C.byref(hd)))
    else:
        _check(c._L.sk_read_matrix(c.h, str(src).encode(), C.byref(kind), C.byref(hc),
                                   C.byref(hd)))
    return _from_read(c, kind, hc, hd)


def write_matrix(a, dst, ctx: Context | None = None) -> MatrixFileInfo:
    """write_matrix(a, path) or write_matrix(a, file-like) (matio.hpp:43-44)."""
    m = a if isinstance(a, Matrix) else Matrix(a)
    rep = m._rep
    c = rep.ctx
    csr_h = rep.h if m.is_sparse() else None
    dense_h = None if m.is_sparse() else rep.h
    info = MatrixFileInfo(None, MatrixFileKind.coordinate if m.is_sparse() else
                          MatrixFileKind.array, m.rows(), m.cols(),
                          rep.nnz() if m.is_sparse() else m.rows() * m.cols())
    if hasattr(dst, "write"):
        n = C.c_size_t()
        _check(c._L.sk_format_matrix(c.h, csr_h, dense_h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(c._L.sk_format_matrix(c.h, csr_h, dense_h, buf, n.value + 1, C.byref(n)))
        dst.write(buf.raw[: n.value].decode())
    else:
        _check(c._L.sk_write_matrix(c.h, csr_h, dense_h, str(dst).encode()))
        info.path = str(dst)
    return info


def _unwrap(m):
    return m._rep if isinstance(m, Matrix) else m


# ---- construction and conversion ---------------------------------------------------------

def csr_from_triples(rows: int, cols: int, triples, ctx: Context | None = None) -> CsrMatrix:
    """Triples in any order; exact 0.0 dropped; InvalidArgument on an
    out-of-range index or a duplicate coordinate (matrix.cpp:145-189).
    ``triples`` is an iterable of (row, col, value) or a tuple of three arrays."""
    c = _ctx(ctx)
    if isinstance(triples, tuple) and len(triples) == 3 and hasattr(triples[0], "__len__") \
            and not isinstance(triples[0], tuple) \
            and not isinstance(triples[0], (int, np.integer)):
        r, cc, v = _u32(triples[0]), _u32(triples[1]), _f32(triples[2])
    else:
        t = list(triples)
        r = _u32([x[0] for x in t])
        cc = _u32([x[1] for x in t])
        v = _f32([x[2] for x in t])
    h = vp()
    _check(c._L.sk_csr_from_triples(c.h, rows, cols, r.ctypes.data, cc.ctypes.data,
                                    v.ctypes.data, len(v), C.byref(h)))
    return CsrMatrix(rows, cols, ctx=c, _handle=h)


def to_dense(a, ambient_zero: float = 0.0) -> DenseMatrix:
    a = _unwrap(a)
    if isinstance(a, DenseMatrix):
        return a
    h = vp()
    _check(a.ctx._L.sk_to_dense(a.ctx.h, a.h, float(ambient_zero), C.byref(h)))
    return DenseMatrix(ctx=a.ctx, _handle=h)


def from_dense(d: DenseMatrix) -> CsrMatrix:
    d = _unwrap(d)
    h = vp()
    _check(d.ctx._L.sk_from_dense(d.ctx.h, d.h, C.byref(h)))
    return CsrMatrix(d.rows(), d.cols(), ctx=d.ctx, _handle=h)


def nnz(a) -> int:
    a = _unwrap(a)
    if isinstance(a, CsrMatrix):
        return a.nnz()
    n = C.c_size_t()
    _check(a.ctx._L.sk_dense_nnz(a.ctx.h, a.h, C.byref(n)))
    return n.value


kIndexWidth = 4


def csr_storage_bytes(rows: int, nnz_count: int) -> int:
    return (rows + 1) * kIndexWidth + nnz_count * (kIndexWidth + 4)


def dense_storage_bytes(rows: int, cols: int) -> int:
    return rows * cols * 4


def storage_bytes(a) -> int:
    a = _unwrap(a)
    if isinstance(a, CsrMatrix):
        return csr_storage_bytes(a.rows(), a.nnz())
    return dense_storage_bytes(a.rows(), a.cols())


# ---- element-wise (matrix.hpp:175-191) --------------------------------------------------------

def _ewise(mul: int, a, b, s: Semiring):
    wrap = isinstance(a, Matrix) or isinstance(b, Matrix)
    a, b = _unwrap(a), _unwrap(b)
    L, c = a.ctx._L, a.ctx
    h = vp()
    if isinstance(a, DenseMatrix) and isinstance(b, DenseMatrix):
        _check(L.sk_ewise_dense(c.h, mul, a.h, b.h, int(s.kind), C.byref(h)))
        r = DenseMatrix(ctx=c, _handle=h)
    elif isinstance(a, CsrMatrix) and isinstance(b, CsrMatrix):
        _check(L.sk_ewise_csr(c.h, mul, a.h, b.h, int(s.kind), C.byref(h)))
        r = CsrMatrix(a.rows(), a.cols(), ctx=c, _handle=h)
    elif isinstance(a, CsrMatrix):
        _check(L.sk_ewise_mixed(c.h, mul, a.h, b.h, 1, int(s.kind), C.byref(h)))
        r = DenseMatrix(ctx=c, _handle=h)
    else:
        _check(L.sk_ewise_mixed(c.h, mul, b.h, a.h, 0, int(s.kind), C.byref(h)))
        r = DenseMatrix(ctx=c, _handle=h)
    return Matrix(r) if wrap else r


def ewise_add(a, b, s: Semiring):
    return _ewise(0, a, b, s)


def ewise_mul(a, b, s: Semiring):
    return _ewise(1, a, b, s)


# ---- mxm (matrix.hpp:193-218) -------------------------------------------------------------------

def mxm(a, b, s: Semiring, workers: int = 1):
    """C = A (+).(x) B.  CSR x dense -> dense, dense x dense -> dense,
    CSR x CSR -> CSR; dense x CSR is rejected.  ``workers`` is accepted for
    signature parity; results never depend on it."""
    if workers < 1:
        raise InvalidArgument("workers must be >= 1")
    wrap = isinstance(a, Matrix) or isinstance(b, Matrix)
    a, b = _unwrap(a), _unwrap(b)
    L, c = a.ctx._L, a.ctx
    h = vp()
    if isinstance(a, CsrMatrix) and isinstance(b, DenseMatrix):
        _check(L.sk_mxm_csr_dense(c.h, a.h, b.h, int(s.kind), C.byref(h)))
        r = DenseMatrix(ctx=c, _handle=h)
    elif isinstance(a, DenseMatrix) and isinstance(b, DenseMatrix):
        _check(L.sk_mxm_dense_dense(c.h, a.h, b.h, int(s.kind), C.byref(h)))
        r = DenseMatrix(ctx=c, _handle=h)
    elif isinstance(a, CsrMatrix) and isinstance(b, CsrMatrix):
        _check(L.sk_mxm_csr_csr(c.h, a.h, b.h, int(s.kind), C.byref(h)))
        r = CsrMatrix(a.rows(), b.cols(), ctx=c, _handle=h)
    else:
        raise Error("mxm: dense-by-sparse is not supported; densify the right operand")
    return Matrix(r) if wrap else r


def dense_mxm_baseline(a: DenseMatrix, b: DenseMatrix, workers: int = 1) -> DenseMatrix:
    a, b = _unwrap(a), _unwrap(b)
    h = vp()
    _check(a.ctx._L.sk_dense_mxm_baseline(a.ctx.h, a.h, b.h, C.byref(h)))
    return DenseMatrix(ctx=a.ctx, _handle=h)


# ---- DNN (dnn.hpp) ---------------------------------------------------------------------------------

Batch = DenseMatrix


def _as_model_csr(w) -> CsrMatrix:
    """Weights of a DnnModel on the device as CSR.  Dense weights keep every
    entry (explicit zeros included) so the fold is the dense kernel's fold."""
    w = _unwrap(w)
    if isinstance(w, CsrMatrix):
        return w
    d = w.numpy()
    m, l = d.shape
    rp = np.arange(0, (m + 1) * l, l, dtype=np.uint32)
    ci = np.tile(np.arange(l, dtype=np.uint32), m)
    return CsrMatrix.from_parts_unchecked(m, l, rp, ci, d.reshape(-1), ctx=w.ctx)


class DnnModel:
    """L square weight layers of one width plus L bias vectors (dnn.hpp:31-47)."""

    def __init__(self, weights: Sequence, biases: Sequence):
        weights = [_unwrap(w) for w in weights]
        biases = [_f32(b) for b in biases]
        if len(weights) == 0:
            raise InvalidArgument("model must have at least one layer")
        if len(weights) != len(biases):
            raise InvalidArgument(f"model has {len(weights)} weight matrices but "
                                  f"{len(biases)} bias vectors")
        m = weights[0].rows()
        for k, (w, b) in enumerate(zip(weights, biases)):
            if w.rows() != m or w.cols() != m:
                raise DimensionError(f"layer {k} weight is {w.rows()}x{w.cols()}; all layers "
                                     f"must be {m}x{m}")
            if b.size != m:
                raise DimensionError(f"layer {k} bias length {b.size} does not match {m} neurons")
        self._weights = weights
        self._biases = biases
        self._csr = [_as_model_csr(w) for w in weights]
        self.ctx = self._csr[0].ctx
        harr = (vp * len(self._csr))(*[w.h.value for w in self._csr])
        barr = (_lib.f32p * len(biases))(*[b.ctypes.data_as(_lib.f32p) for b in biases])
        h = vp()
        _check(self.ctx._L.sk_model_create(self.ctx.h, len(weights), harr, barr, C.byref(h)))
        self.h = h
        self._neurons = m

    def num_layers(self) -> int:
        return len(self._weights)

    def neurons(self) -> int:
        return self._neurons

    def weight(self, k: int):
        return Matrix(self._weights[k])

    def bias(self, k: int) -> np.ndarray:
        return self._biases[k]

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx._L.sk_model_free(self.h)
        except Exception:
            pass


@dataclass
class ForwardOptions:
    workers: int = 1
    materialize_bias: bool = False
    clip: float = 0.0  # extension: BASELINE cfg3-5 clip (0 = none, as the reference)

    def _c(self) -> FwdOpts:
        if self.workers < 1:
            raise InvalidArgument("workers must be >= 1")
        return FwdOpts(self.workers, int(self.materialize_bias), float(self.clip))


def layer_step(w, bias, y: DenseMatrix, relu_zero: DenseMatrix | None = None,
               opt: ForwardOptions | None = None) -> DenseMatrix:
    """Fused W.Y + b -> ReLU (dnn.cpp:86-103).  ``relu_zero`` is accepted for
    signature parity; the fused kernel never materialises it."""
    opt = opt or ForwardOptions()
    if isinstance(relu_zero, ForwardOptions):
        opt, relu_zero = relu_zero, None
    wc = _as_model_csr(w)
    b = _f32(bias)
    if y.rows() != wc.cols():
        raise DimensionError(f"weight is {wc.rows()}x{wc.cols()} but input has {y.rows()} rows")
    if b.size != wc.rows():
        raise DimensionError(f"bias length {b.size} does not match {wc.rows()} output rows")
    o = opt._c()
    h = vp()
    _check(y.ctx._L.sk_layer_step(y.ctx.h, wc.h, b.ctypes.data, y.h, C.byref(o), C.byref(h)))
    return DenseMatrix(ctx=y.ctx, _handle=h)


def relu_forward(model: DnnModel, input: DenseMatrix,
                 opt: ForwardOptions | None = None) -> DenseMatrix:
    o = (opt or ForwardOptions())._c()
    h = vp()
    _check(model.ctx._L.sk_relu_forward(model.ctx.h, model.h, input.h, C.byref(o), C.byref(h)))
    return DenseMatrix(ctx=model.ctx, _handle=h)


def relu_forward_host(model: DnnModel, y0: np.ndarray, opt: ForwardOptions | None = None,
                      out: np.ndarray | None = None) -> np.ndarray:
    """Host-buffer end-to-end call: H2D(y0) -> forward -> D2H(result)."""
    y0 = _f32(y0)
    if out is None:
        out = np.empty_like(y0)
    o = (opt or ForwardOptions())._c()
    if y0.shape[0] != model.neurons() or y0.ndim != 2 or y0.shape[1] < 1:
        raise DimensionError(f"input batch is {y0.shape}, expected {model.neurons()} rows")
    _check(model.ctx._L.sk_relu_forward_host(model.ctx.h, model.h, y0.shape[1], y0.ctypes.data,
                                             C.byref(o), out.ctypes.data))
    return out


def dense_layer_step(w: DenseMatrix, bias, y: DenseMatrix, workers: int = 1) -> DenseMatrix:
    w = _unwrap(w)
    b = _f32(bias)
    if b.size != w.rows():
        raise DimensionError(f"bias length {b.size} does not match {w.rows()} output rows")
    h = vp()
    _check(w.ctx._L.sk_dense_layer_step(w.ctx.h, w.h, b.ctypes.data, y.h, C.byref(h)))
    return DenseMatrix(ctx=w.ctx, _handle=h)


def dense_relu_forward(model: DnnModel, input: DenseMatrix) -> DenseMatrix:
    h = vp()
    _check(model.ctx._L.sk_dense_relu_forward(model.ctx.h, model.h, input.h, C.byref(h)))
    return DenseMatrix(ctx=model.ctx, _handle=h)


# ---- extensions for the BASELINE workloads -----------------------------------------------------

def relu_forward_sparse(model: DnnModel, y0: CsrMatrix, opt: ForwardOptions | None = None,
                        want_trace: bool = True):
    """Sparse-activation forward: returns (Y_L as CsrMatrix, nnz trace)."""
    o = (opt or ForwardOptions())._c()
    h = vp()
    trace = np.zeros(model.num_layers() + 1, np.uint64)
    _check(model.ctx._L.sk_relu_forward_sparse(model.ctx.h, model.h, y0.h, C.byref(o),
                                               C.byref(h),
                                               trace.ctypes.data if want_trace else None))
    return CsrMatrix(y0.rows(), y0.cols(), ctx=model.ctx, _handle=h), trace


def categories(y) -> np.ndarray:
    """Sorted sample (column) indices holding any nonzero."""
    y = _unwrap(y)
    L, c = y.ctx._L, y.ctx
    cnt = C.c_size_t()
    fn = L.sk_categories_csr if isinstance(y, CsrMatrix) else L.sk_categories_dense
    out = np.empty(max(y.cols(), 1), np.uint32)
    _check(fn(c.h, y.h, out.ctypes.data, out.size, C.byref(cnt)))
    return out[: cnt.value].copy()


def layer_seed(seed: int, layer: int) -> int:
    return int(_lib.load().sk_layer_seed(seed, layer))


def gen_layer_fixed(m: int, k: int, lseed: int, value: float = float("nan"),
                    ctx: Context | None = None) -> CsrMatrix:
    c = _ctx(ctx)
    h = vp()
    _check(c._L.sk_gen_layer_fixed(c.h, m, k, lseed, value, C.byref(h)))
    return CsrMatrix(m, m, ctx=c, _handle=h)


def gen_layer_density(m: int, density: float, lseed: int, ctx: Context | None = None) -> CsrMatrix:
    c = _ctx(ctx)
    h = vp()
    _check(c._L.sk_gen_layer_density(c.h, m, density, lseed, C.byref(h)))
    return CsrMatrix(m, m, ctx=c, _handle=h)


def gen_weight(m: int, inverse_sparsity: float, seed: int,
               ctx: Context | None = None) -> CsrMatrix:
    """The reference's gen_weight (matgen.cpp:50-87), bitwise, on the device."""
    c = _ctx(ctx)
    h = vp()
    _check(c._L.sk_gen_weight(c.h, m, float(inverse_sparsity), seed, C.byref(h)))
    return CsrMatrix(m, m, ctx=c, _handle=h)


def gen_input_dense(m: int, n: int, seed: int, ctx: Context | None = None) -> DenseMatrix:
    c = _ctx(ctx)
    h = vp()
    _check(c._L.sk_gen_input_dense(c.h, m, n, seed, C.byref(h)))
    return DenseMatrix(ctx=c, _handle=h)


def gen_input_binary(m: int, n: int, k: int, seed: int, sample_offset: int = 0,
                     ctx: Context | None = None) -> CsrMatrix:
    c = _ctx(ctx)
    h = vp()
    _check(c._L.sk_gen_input_binary(c.h, m, n, k, seed, sample_offset, C.byref(h)))
    return CsrMatrix(m, n, ctx=c, _handle=h)


def sparse_layer(w: CsrMatrix, bias, y: CsrMatrix, clip: float = 0.0) -> CsrMatrix:
    """One sparse-activation layer with a (possibly rectangular) weight block:
    W_ref rows = a block of output neurons.  The unit of the column-sharded
    forward pass (each GPU owns a block of output neurons)."""
    b = _f32(bias)
    if b.size != w.rows():
        raise DimensionError(f"bias length {b.size} does not match {w.rows()} output rows")
    h = vp()
    _check(y.ctx._L.sk_sparse_layer(y.ctx.h, w.h, b.ctypes.data, y.h, float(clip), C.byref(h)))
    return CsrMatrix(w.rows(), y.cols(), ctx=y.ctx, _handle=h)


def sparse_layer_dev(w: CsrMatrix, d_bias: int, dense_rows: int, negmin: float, y: CsrMatrix,
                     clip: float = 0.0) -> CsrMatrix:
    """sparse_layer with a device-resident bias (pointer to w.rows() floats) and
    its summaries precomputed (sk_sparse_layer_dev): dense_rows = rows with
    !(b <= 0), negmin = min of -b over b <= 0 (inf if none)."""
    h = vp()
    _check(y.ctx._L.sk_sparse_layer_dev(y.ctx.h, w.h, vp(d_bias), int(dense_rows), float(negmin),
                                        y.h, float(clip), C.byref(h)))
    return CsrMatrix(w.rows(), y.cols(), ctx=y.ctx, _handle=h)


class StagedLayer:
    """A column-shard layer computed up to its output count (sk_sparse_layer_stage);
    publish() writes the block into the exchange destinations with the layer's
    own gather kernel and releases it."""

    def __init__(self, ctx, h, nnz: int):
        self.ctx, self.h, self.nnz = ctx, h, nnz

    def publish(self, dst_rp, dst_ci, dst_v, row_off: int, nnz_off: int, write_last: bool):
        nd = len(dst_rp)
        arr = lambda xs: (vp * nd)(*[vp(x) for x in xs])  # noqa: E731
        h, self.h = self.h, None
        _check(self.ctx._L.sk_staged_publish(self.ctx.h, h, nd, arr(dst_rp), arr(dst_ci),
                                             arr(dst_v), row_off, nnz_off, int(write_last)))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx._L.sk_staged_free(self.h)
        except Exception:
            pass


def sparse_layer_stage(w: CsrMatrix, d_bias: int, dense_rows: int, negmin: float, y: CsrMatrix,
                       clip: float = 0.0) -> StagedLayer:
    h = vp()
    nnz = C.c_uint64()
    _check(y.ctx._L.sk_sparse_layer_stage(y.ctx.h, w.h, vp(d_bias), int(dense_rows),
                                          float(negmin), y.h, float(clip), C.byref(h),
                                          C.byref(nnz)))
    return StagedLayer(y.ctx, h, int(nnz.value))


def bias_summaries(bias) -> tuple[int, float]:
    """(dense_rows, negmin) of a bias vector, as sk_sparse_layer_dev expects."""
    b = _f32(bias)
    nonpos = b <= 0.0
    dense_rows = int(b.size - np.count_nonzero(nonpos))
    negmin = float(np.min(-b[nonpos].astype(np.float64))) if np.any(nonpos) else math.inf
    return dense_rows, negmin


def csr_device_arrays(a: CsrMatrix):
    """(row_ptr, col_idx, values) device pointers of a handle (zero-copy)."""
    rp, ci, v = vp(), vp(), vp()
    _check(a.ctx._L.sk_csr_device_arrays(a.h, C.byref(rp), C.byref(ci), C.byref(v)))
    return rp.value or 0, ci.value or 0, v.value or 0


def csr_from_device(rows: int, cols: int, nnz: int, rp_ptr: int, ci_ptr: int, v_ptr: int,
                    ctx: Context | None = None) -> CsrMatrix:
    c = _ctx(ctx)
    h = vp()
    _check(c._L.sk_csr_from_device(c.h, rows, cols, nnz, vp(rp_ptr), vp(ci_ptr), vp(v_ptr),
                                   C.byref(h)))
    return CsrMatrix(rows, cols, ctx=c, _handle=h)


def memcpy_d2d(dst_ptr: int, src_ptr: int, nbytes: int, ctx: Context | None = None):
    c = _ctx(ctx)
    _check(c._L.sk_memcpy_d2d(c.h, vp(dst_ptr), vp(src_ptr), nbytes))


# ---- column-sharded exchange over peer memory (sk_ipc_*, sk_csr_publish) ----------------

def ipc_alloc(nbytes: int, ctx: Context | None = None) -> tuple[int, bytes]:
    """A cudaMalloc'd device buffer and its 64-byte CUDA IPC handle."""
    c = _ctx(ctx)
    p = vp()
    h = C.create_string_buffer(64)
    _check(c._L.sk_ipc_alloc(c.h, max(int(nbytes), 16), C.byref(p), h))
    return p.value or 0, h.raw


def ipc_open(handle: bytes, ctx: Context | None = None) -> int:
    """Map a peer's buffer (peer access over NVLink)."""
    c = _ctx(ctx)
    p = vp()
    _check(c._L.sk_ipc_open(c.h, C.create_string_buffer(bytes(handle), 64), C.byref(p)))
    return p.value or 0


def ipc_close(ptr: int):
    _check(_lib.load().sk_ipc_close(vp(ptr)))


def ipc_free(ptr: int):
    _check(_lib.load().sk_ipc_free(vp(ptr)))


def csr_publish(blk: CsrMatrix, dst_rp, dst_ci, dst_v, row_off: int, nnz_off: int,
                write_last: bool):
    """One kernel writes `blk` into every destination (device pointers, peers'
    included): entries at nnz_off, row pointers at row_off shifted by nnz_off."""
    n = len(dst_rp)
    arr = vp * n
    _check(blk.ctx._L.sk_csr_publish(blk.ctx.h, blk.h, n, arr(*[vp(x) for x in dst_rp]),
                                     arr(*[vp(x) for x in dst_ci]),
                                     arr(*[vp(x) for x in dst_v]), int(row_off), int(nnz_off),
                                     1 if write_last else 0))
