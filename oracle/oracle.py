"""TEST INFRASTRUCTURE ONLY -- ctypes access to the two CPU checkers.

* ``Ref``  : the unmodified reference library (oracle/_ref/libsemikern_ref.so,
             built from /root/reference/proj/src by oracle/Makefile).
* ``Port`` : our C restatement of what the reference lacks
             (oracle/_build/libsk_oracle.so, from oracle/sk_oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  The product package
(paper_1708_02937_b200) never does.

Orientation is the reference's: W_ref m-by-m CSR with row i = in-edges of
output neuron i; Y_ref m-by-n neuron-major (proj/include/semikern/dnn.hpp:24-25).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsemikern_ref.so")
PORT_SO = os.path.join(HERE, "_build", "libsk_oracle.so")

u32p = C.POINTER(C.c_uint32)
f32p = C.POINTER(C.c_float)
u8p = C.POINTER(C.c_uint8)

SEMIRING = {"arithmetic": 0, "max_plus": 1, "min_max": 2, "gf2": 3}
STATUS_NAMES = {1: "Error", 2: "DimensionError", 3: "DomainError",
                4: "InvalidArgument", 5: "ParseError"}


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS_NAMES.get(code, "Error")


def _p(a, t):
    return a.ctypes.data_as(t)


@dataclass
class Csr:
    """Host CSR in the reference layout (u32 row_ptr/col_idx, f32 values)."""
    rows: int
    cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_dense(self, ambient: float = 0.0) -> np.ndarray:
        d = np.full((self.rows, self.cols), ambient, dtype=np.float32)
        for i in range(self.rows):
            s, e = self.row_ptr[i], self.row_ptr[i + 1]
            d[i, self.col_idx[s:e]] = self.values[s:e]
        return d

    def transpose(self) -> "Csr":
        port = Port.get()
        trp = np.zeros(self.cols + 1, np.uint32)
        tci = np.zeros(max(self.nnz, 1), np.uint32)
        tv = np.zeros(max(self.nnz, 1), np.float32)
        port.lib.sko_csr_transpose(self.rows, self.cols, _p(self.row_ptr, u32p),
                                   _p(self.col_idx, u32p), _p(self.values, f32p),
                                   _p(trp, u32p), _p(tci, u32p), _p(tv, f32p))
        return Csr(self.cols, self.rows, trp, tci[: self.nnz], tv[: self.nnz])

    def same_as(self, o: "Csr") -> bool:
        return (self.rows == o.rows and self.cols == o.cols
                and np.array_equal(self.row_ptr, o.row_ptr)
                and np.array_equal(self.col_idx, o.col_idx)
                and np.array_equal(self.values.view(np.uint32), o.values.view(np.uint32)))


def csr(rows, cols, row_ptr, col_idx, values) -> Csr:
    return Csr(int(rows), int(cols), np.ascontiguousarray(row_ptr, np.uint32),
               np.ascontiguousarray(col_idx, np.uint32),
               np.ascontiguousarray(values, np.float32))


class Ref:
    """The reference library itself, through oracle/ref_capi.cpp."""
    _inst = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def get(cls) -> "Ref":
        if cls._inst is None:
            cls._inst = cls()
        return cls._inst

    def __init__(self):
        L = C.CDLL(REF_SO)
        self.lib = L
        L.skref_last_error.restype = C.c_char_p
        L.skref_splitmix_at.restype = C.c_uint64
        L.skref_splitmix_at.argtypes = [C.c_uint64, C.c_uint64]
        L.skref_csr_nnz.restype = C.c_size_t
        L.skref_csr_rows.restype = C.c_uint32
        L.skref_csr_cols.restype = C.c_uint32
        L.skref_gen_weight.argtypes = [C.c_uint32, C.c_double, C.c_uint64, C.c_void_p]
        L.skref_gen_input.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, f32p]
        L.skref_gen_bias.argtypes = [C.c_uint32, C.c_uint64, C.c_int, f32p]
        vp_, sz = C.c_void_p, C.c_size_t
        L.skref_bench_analyze.argtypes = [sz, vp_, vp_, vp_, vp_, vp_, C.c_uint32, sz, vp_,
                                          C.POINTER(sz)]
        L.skref_bench_records_csv.argtypes = [sz, vp_, vp_, vp_, vp_, vp_, vp_, vp_, vp_,
                                              C.c_char_p, sz, C.POINTER(sz)]
        L.skref_bench_params_csv.argtypes = [sz, vp_, vp_, vp_, vp_, vp_, C.c_uint32,
                                             C.c_char_p, sz, C.POINTER(sz)]
        L.skref_bench_read_csv.argtypes = [C.c_char_p, sz, vp_, vp_, vp_, vp_, vp_, vp_, vp_,
                                           vp_, C.POINTER(sz)]
        L.skref_bench_validate.argtypes = [sz, vp_, sz, vp_, C.c_uint32, C.c_uint32, sz, vp_,
                                           C.c_int, C.c_int]
        L.skref_read_matrix_text.argtypes = [C.c_char_p, C.POINTER(C.c_int),
                                             C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                             C.POINTER(vp_), vp_, sz]
        L.skref_format_matrix.argtypes = [vp_, C.c_uint32, C.c_uint32, vp_, C.c_char_p, sz,
                                          C.POINTER(sz)]
        L.skref_to_dense.argtypes = [C.c_void_p, C.c_float, f32p]
        L.skref_layer_sparse_h.argtypes = [vp_, vp_, f32p, C.c_float, C.c_int,
                                           C.POINTER(vp_)]
        L.skref_csr_nnz.argtypes = [vp_]

    def _check(self, rc):
        if rc != 0:
            raise RefError(rc, self.lib.skref_last_error().decode())

    # -- handles --
    def _handle(self, a: Csr):
        h = C.c_void_p()
        self._check(self.lib.skref_csr_from_parts(
            C.c_uint32(a.rows), C.c_uint32(a.cols), _p(a.row_ptr, u32p),
            _p(a.col_idx, u32p), _p(a.values, f32p), C.byref(h)))
        return h

    def _take(self, h) -> Csr:
        L = self.lib
        rows, cols, nnz = L.skref_csr_rows(h), L.skref_csr_cols(h), L.skref_csr_nnz(h)
        rp = np.zeros(rows + 1, np.uint32)
        ci = np.zeros(max(nnz, 1), np.uint32)
        v = np.zeros(max(nnz, 1), np.float32)
        L.skref_csr_extract(h, _p(rp, u32p), _p(ci, u32p), _p(v, f32p))
        L.skref_csr_free(h)
        return Csr(rows, cols, rp, ci[:nnz], v[:nnz])

    def splitmix_at(self, seed: int, idx: int) -> int:
        return int(self.lib.skref_splitmix_at(seed, idx))

    # persistent handles (so timing loops measure the reference's kernels,
    # not the marshalling into its value types)
    def handle(self, a: Csr):
        return self._handle(a)

    def free(self, h):
        self.lib.skref_csr_free(h)

    def take(self, h) -> Csr:
        return self._take(h)

    def mxm_csr_csr_h(self, ha, hb, workers=1):
        h = C.c_void_p()
        self._check(self.lib.skref_mxm_csr_csr(ha, hb, 0, workers, C.byref(h)))
        return h

    def layer_sparse_h(self, hw, hy, bias, clip=0.0, workers=1):
        """One sparse-activation layer on reference handles: the reference's
        mxm(W_ref, Y_ref) + the restated epilogue (ref_capi.cpp).  Returns a new
        handle (the caller frees it)."""
        bias = np.ascontiguousarray(bias, np.float32)
        h = C.c_void_p()
        self._check(self.lib.skref_layer_sparse_h(hw, hy, _p(bias, f32p), clip, workers,
                                                  C.byref(h)))
        return h

    def nnz_h(self, h) -> int:
        return int(self.lib.skref_csr_nnz(h))

    def csr_from_triples(self, rows, cols, r, c, v) -> Csr:
        r = np.ascontiguousarray(r, np.uint32)
        c = np.ascontiguousarray(c, np.uint32)
        v = np.ascontiguousarray(v, np.float32)
        h = C.c_void_p()
        self._check(self.lib.skref_csr_from_triples(
            C.c_uint32(rows), C.c_uint32(cols), _p(r, u32p), _p(c, u32p), _p(v, f32p),
            C.c_size_t(len(v)), C.byref(h)))
        return self._take(h)

    def csr_validate(self, a: Csr) -> Csr:
        return self._take(self._handle(a))

    def from_dense(self, d: np.ndarray) -> Csr:
        d = np.ascontiguousarray(d, np.float32)
        h = C.c_void_p()
        self._check(self.lib.skref_csr_from_dense(C.c_uint32(d.shape[0]), C.c_uint32(d.shape[1]),
                                                  _p(d, f32p), C.byref(h)))
        return self._take(h)

    def to_dense(self, a: Csr, ambient: float = 0.0) -> np.ndarray:
        h = self._handle(a)
        out = np.zeros((a.rows, a.cols), np.float32)
        try:
            self._check(self.lib.skref_to_dense(h, C.c_float(ambient), _p(out, f32p)))
        finally:
            self.lib.skref_csr_free(h)
        return out

    def mxm_csr_dense(self, a: Csr, b: np.ndarray, semiring="arithmetic", workers=1):
        b = np.ascontiguousarray(b, np.float32)
        out = np.zeros((a.rows, b.shape[1]), np.float32)
        h = self._handle(a)
        try:
            self._check(self.lib.skref_mxm_csr_dense(
                h, C.c_uint32(b.shape[0]), C.c_uint32(b.shape[1]), _p(b, f32p),
                SEMIRING[semiring], workers, _p(out, f32p)))
        finally:
            self.lib.skref_csr_free(h)
        return out

    def mxm_dense_dense(self, a, b, semiring="arithmetic", workers=1):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.zeros((a.shape[0], b.shape[1]), np.float32)
        self._check(self.lib.skref_mxm_dense_dense(
            C.c_uint32(a.shape[0]), C.c_uint32(a.shape[1]), _p(a, f32p),
            C.c_uint32(b.shape[0]), C.c_uint32(b.shape[1]), _p(b, f32p),
            SEMIRING[semiring], workers, _p(out, f32p)))
        return out

    def mxm_csr_csr(self, a: Csr, b: Csr, semiring="arithmetic", workers=1) -> Csr:
        ha, hb = self._handle(a), self._handle(b)
        h = C.c_void_p()
        try:
            self._check(self.lib.skref_mxm_csr_csr(ha, hb, SEMIRING[semiring], workers,
                                                   C.byref(h)))
        finally:
            self.lib.skref_csr_free(ha)
            self.lib.skref_csr_free(hb)
        return self._take(h)

    def dense_mxm_baseline(self, a, b, workers=1):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.zeros((a.shape[0], b.shape[1]), np.float32)
        self._check(self.lib.skref_dense_mxm_baseline(
            C.c_uint32(a.shape[0]), C.c_uint32(a.shape[1]), _p(a, f32p),
            C.c_uint32(b.shape[0]), C.c_uint32(b.shape[1]), _p(b, f32p), workers,
            _p(out, f32p)))
        return out

    def ewise_dense(self, mul, a, b, semiring="arithmetic"):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        if a.shape != b.shape:
            rows, cols = a.shape
        out = np.zeros(a.shape, np.float32)
        self._check(self.lib.skref_ewise_dense(int(mul), C.c_uint32(a.shape[0]),
                                               C.c_uint32(a.shape[1]), _p(a, f32p),
                                               _p(b, f32p), SEMIRING[semiring], _p(out, f32p)))
        return out

    def ewise_csr(self, mul, a: Csr, b: Csr, semiring="arithmetic") -> Csr:
        ha, hb = self._handle(a), self._handle(b)
        h = C.c_void_p()
        try:
            self._check(self.lib.skref_ewise_csr(int(mul), ha, hb, SEMIRING[semiring],
                                                 C.byref(h)))
        finally:
            self.lib.skref_csr_free(ha)
            self.lib.skref_csr_free(hb)
        return self._take(h)

    def _model(self, weights, biases):
        hs = [self._handle(w) for w in weights]
        harr = (C.c_void_p * len(hs))(*[h.value for h in hs])
        bs = [np.ascontiguousarray(b, np.float32) for b in biases]
        barr = (f32p * len(bs))(*[_p(b, f32p) for b in bs])
        return hs, harr, bs, barr

    def relu_forward(self, weights, biases, y0, workers=1, materialize_bias=False):
        m, n = y0.shape
        y0 = np.ascontiguousarray(y0, np.float32)
        out = np.zeros((m, n), np.float32)
        hs, harr, bs, barr = self._model(weights, biases)
        try:
            self._check(self.lib.skref_relu_forward(
                C.c_uint32(m), C.c_uint32(len(weights)), harr, barr, C.c_uint32(n),
                _p(y0, f32p), workers, int(materialize_bias), _p(out, f32p)))
        finally:
            for h in hs:
                self.lib.skref_csr_free(h)
        return out

    def dense_relu_forward(self, weights, biases, y0):
        m, n = y0.shape
        y0 = np.ascontiguousarray(y0, np.float32)
        out = np.zeros((m, n), np.float32)
        hs, harr, bs, barr = self._model(weights, biases)
        try:
            self._check(self.lib.skref_dense_relu_forward(
                C.c_uint32(m), C.c_uint32(len(weights)), harr, barr, C.c_uint32(n),
                _p(y0, f32p), _p(out, f32p)))
        finally:
            for h in hs:
                self.lib.skref_csr_free(h)
        return out

    def layer_step(self, w: Csr, bias, y, workers=1):
        y = np.ascontiguousarray(y, np.float32)
        bias = np.ascontiguousarray(bias, np.float32)
        out = np.zeros((w.rows, y.shape[1]), np.float32)
        h = self._handle(w)
        try:
            self._check(self.lib.skref_layer_step(h, _p(bias, f32p), C.c_uint32(y.shape[1]),
                                                  _p(y, f32p), workers, _p(out, f32p)))
        finally:
            self.lib.skref_csr_free(h)
        return out

    def dense_layer_step(self, wd, bias, y, workers=1):
        wd = np.ascontiguousarray(wd, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        bias = np.ascontiguousarray(bias, np.float32)
        out = np.zeros((wd.shape[0], y.shape[1]), np.float32)
        self._check(self.lib.skref_dense_layer_step(
            C.c_uint32(wd.shape[0]), C.c_uint32(wd.shape[1]), _p(wd, f32p), _p(bias, f32p),
            C.c_uint32(y.shape[1]), _p(y, f32p), workers, _p(out, f32p)))
        return out

    def gen_weight(self, m, inverse_sparsity, seed) -> Csr:
        h = C.c_void_p()
        self._check(self.lib.skref_gen_weight(m, inverse_sparsity, seed, C.byref(h)))
        return self._take(h)

    def gen_input(self, m, batch, seed) -> np.ndarray:
        out = np.zeros((m, batch), np.float32)
        self._check(self.lib.skref_gen_input(m, batch, seed, _p(out, f32p)))
        return out

    def gen_bias(self, m, seed, uniform01=False) -> np.ndarray:
        out = np.zeros(m, np.float32)
        self._check(self.lib.skref_gen_bias(m, seed, int(uniform01), _p(out, f32p)))
        return out

    # ---- Matrix Market (proj/include/semikern/matio.hpp) ----

    def read_matrix_text(self, text: str):
        """('csr', Csr) or ('dense', ndarray) -- read_matrix(std::istream&)."""
        kind, r, c = C.c_int(), C.c_uint32(), C.c_uint32()
        h = C.c_void_p()
        cap = 1 << 24
        dense = np.zeros(cap, np.float32)
        self._check(self.lib.skref_read_matrix_text(
            text.encode(), C.byref(kind), C.byref(r), C.byref(c), C.byref(h),
            dense.ctypes.data_as(C.c_void_p), C.c_size_t(cap)))
        if kind.value == 0:
            return "csr", self._take(h)
        return "dense", dense[: r.value * c.value].reshape(r.value, c.value).copy()

    def format_matrix(self, a) -> str:
        """write_matrix(Matrix, std::ostream&) of a Csr or a dense ndarray."""
        if isinstance(a, Csr):
            h = self.handle(a)
            try:
                return self._text(self.lib.skref_format_matrix, h, C.c_uint32(0),
                                  C.c_uint32(0), None)
            finally:
                self.free(h)
        d = np.ascontiguousarray(a, np.float32)
        return self._text(self.lib.skref_format_matrix, None, C.c_uint32(d.shape[0]),
                          C.c_uint32(d.shape[1]), d.ctypes.data_as(C.c_void_p))

    # ---- benchmark sweep analysis / CSV (proj/include/semikern/bench.hpp) ----

    @staticmethod
    def _rec_arrays(records):
        """records: iterables of (m, is, impl(0 sparse / 1 dense), workers, mean,
        stddev, nnz, bytes)."""
        r = list(records)
        n = len(r)
        cols = list(zip(*r)) if n else [[]] * 8
        return (n, np.asarray(cols[0], np.uint32), np.asarray(cols[1], np.float64),
                np.asarray(cols[2], np.int32), np.asarray(cols[3], np.int32),
                np.asarray(cols[4], np.float64), np.asarray(cols[5], np.float64),
                np.asarray(cols[6], np.uint64), np.asarray(cols[7], np.uint64))

    def bench_analyze(self, records, reference_m):
        n, m, is_, impl, wk, mean, _, _, _ = self._rec_arrays(records)
        cap = 4096
        out = np.zeros(9 * cap)
        cnt = C.c_size_t()
        self._check(self.lib.skref_bench_analyze(
            C.c_size_t(n), m.ctypes.data_as(C.c_void_p), is_.ctypes.data_as(C.c_void_p),
            impl.ctypes.data_as(C.c_void_p), wk.ctypes.data_as(C.c_void_p),
            mean.ctypes.data_as(C.c_void_p), C.c_uint32(reference_m), C.c_size_t(cap),
            out.ctypes.data_as(C.c_void_p), C.byref(cnt)))
        return out[: 9 * cnt.value].reshape(cnt.value, 9)

    def _text(self, fn, *args):
        cap = 1 << 22
        buf = C.create_string_buffer(cap)
        ln = C.c_size_t()
        self._check(fn(*args, buf, C.c_size_t(cap), C.byref(ln)))
        return buf.value.decode()

    def bench_records_csv(self, records) -> str:
        n, m, is_, impl, wk, mean, sd, nnz, byt = self._rec_arrays(records)
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        return self._text(self.lib.skref_bench_records_csv, C.c_size_t(n), ptr(m), ptr(is_),
                          ptr(impl), ptr(wk), ptr(mean), ptr(sd), ptr(nnz), ptr(byt))

    def bench_params_csv(self, records, reference_m) -> str:
        n, m, is_, impl, wk, mean, _, _, _ = self._rec_arrays(records)
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        return self._text(self.lib.skref_bench_params_csv, C.c_size_t(n), ptr(m), ptr(is_),
                          ptr(impl), ptr(wk), ptr(mean), C.c_uint32(reference_m))

    def bench_read_csv(self, text: str):
        cap = 65536
        m = np.zeros(cap, np.uint32)
        is_ = np.zeros(cap)
        impl = np.zeros(cap, np.int32)
        wk = np.zeros(cap, np.int32)
        mean = np.zeros(cap)
        sd = np.zeros(cap)
        nnz = np.zeros(cap, np.uint64)
        byt = np.zeros(cap, np.uint64)
        cnt = C.c_size_t()
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(self.lib.skref_bench_read_csv(
            C.c_char_p(text.encode()), C.c_size_t(cap), ptr(m), ptr(is_), ptr(impl), ptr(wk),
            ptr(mean), ptr(sd), ptr(nnz), ptr(byt), C.byref(cnt)))
        k = cnt.value
        return [(int(m[i]), float(is_[i]), int(impl[i]), int(wk[i]), float(mean[i]),
                 float(sd[i]), int(nnz[i]), int(byt[i])) for i in range(k)]

    def bench_validate(self, sizes, inverse_sparsities, batch, layers, workers, repetitions,
                       warmup):
        sz = np.asarray(sizes, np.uint32)
        isx = np.asarray(inverse_sparsities, np.float64)
        wk = np.asarray(workers, np.int32)
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(self.lib.skref_bench_validate(
            C.c_size_t(sz.size), ptr(sz), C.c_size_t(isx.size), ptr(isx), C.c_uint32(batch),
            C.c_uint32(layers), C.c_size_t(wk.size), ptr(wk), C.c_int(repetitions),
            C.c_int(warmup)))


class Port:
    """Our C restatement (oracle/sk_oracle.c)."""
    _inst = None

    @classmethod
    def get(cls) -> "Port":
        if cls._inst is None:
            cls._inst = cls()
        return cls._inst

    def __init__(self):
        L = C.CDLL(PORT_SO)
        self.lib = L
        L.sko_splitmix_at.restype = C.c_uint64
        L.sko_splitmix_at.argtypes = [C.c_uint64, C.c_uint64]
        L.sko_layer_seed.restype = C.c_uint64
        L.sko_layer_seed.argtypes = [C.c_uint64, C.c_uint32]
        L.sko_gen_fixed_rows.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, u32p]
        L.sko_uniform_pm1.restype = C.c_float
        L.sko_uniform_pm1.argtypes = [C.c_uint64, C.c_uint64]
        L.sko_gen_layer_fixed.restype = C.c_size_t
        L.sko_gen_layer_fixed.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_float,
                                          u32p, u32p, f32p]
        L.sko_gen_layer_density.restype = C.c_size_t
        L.sko_gen_layer_density.argtypes = [C.c_uint32, C.c_double, C.c_uint64, u32p,
                                            C.c_void_p, C.c_void_p]
        L.sko_gen_input_dense.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, f32p]
        L.sko_gen_input_binary.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                           C.c_uint64, u32p, u32p, f32p]
        L.sko_layer_dense.argtypes = [C.c_uint32, C.c_uint32, u32p, u32p, f32p, f32p,
                                      C.c_float, C.c_uint32, f32p, f32p]
        L.sko_layer_sparse.restype = C.c_size_t
        L.sko_layer_sparse.argtypes = [C.c_uint32, C.c_uint32, u32p, u32p, f32p, f32p,
                                       C.c_float, C.c_uint32, u32p, u32p, f32p,
                                       C.POINTER(u32p), C.POINTER(u32p), C.POINTER(f32p)]
        L.sko_sparse_epilogue.restype = C.c_size_t
        L.sko_sparse_epilogue.argtypes = [C.c_uint32, C.c_uint32, u32p, u32p, f32p, f32p,
                                          C.c_float, C.POINTER(u32p), C.POINTER(u32p),
                                          C.POINTER(f32p)]
        L.sko_categories_sparse.argtypes = [C.c_uint32, C.c_uint32, u32p, u32p, f32p, u8p]
        L.sko_categories_dense.argtypes = [C.c_uint32, C.c_uint32, f32p, u8p]
        L.sko_free.argtypes = [C.c_void_p]
        L.sko_threads.restype = C.c_int
        L.sko_set_threads.argtypes = [C.c_int]

    def set_threads(self, n: int):
        self.lib.sko_set_threads(int(n))

    def threads(self) -> int:
        return int(self.lib.sko_threads())

    def layer_seed(self, seed, k):
        return int(self.lib.sko_layer_seed(seed, k))

    def splitmix_at(self, seed, idx):
        return int(self.lib.sko_splitmix_at(seed, idx))

    def gen_fixed_rows(self, rows, cols, k, seed) -> np.ndarray:
        out = np.zeros(rows * k, np.uint32)
        self.lib.sko_gen_fixed_rows(rows, cols, k, seed, _p(out, u32p))
        return out.reshape(rows, k)

    def gen_layer_fixed(self, m, k, layer_seed, value=float("nan")) -> Csr:
        rp = np.zeros(m + 1, np.uint32)
        ci = np.zeros(m * k, np.uint32)
        v = np.zeros(m * k, np.float32)
        self.lib.sko_gen_layer_fixed(m, k, layer_seed, value, _p(rp, u32p), _p(ci, u32p),
                                     _p(v, f32p))
        return Csr(m, m, rp, ci, v)

    def gen_layer_density(self, m, density, layer_seed) -> Csr:
        rp = np.zeros(m + 1, np.uint32)
        nnz = self.lib.sko_gen_layer_density(m, density, layer_seed, _p(rp, u32p), None, None)
        ci = np.zeros(max(nnz, 1), np.uint32)
        v = np.zeros(max(nnz, 1), np.float32)
        self.lib.sko_gen_layer_density(m, density, layer_seed, _p(rp, u32p),
                                       ci.ctypes.data, v.ctypes.data)
        return Csr(m, m, rp, ci[:nnz], v[:nnz])

    def gen_input_dense(self, m, n, seed) -> np.ndarray:
        y = np.zeros((m, n), np.float32)
        self.lib.sko_gen_input_dense(m, n, seed, _p(y, f32p))
        return y

    def gen_input_binary(self, m, n, k, seed, sample_offset=0) -> Csr:
        rp = np.zeros(m + 1, np.uint32)
        ci = np.zeros(n * k, np.uint32)
        v = np.zeros(n * k, np.float32)
        self.lib.sko_gen_input_binary(m, n, k, seed, sample_offset, _p(rp, u32p), _p(ci, u32p),
                                      _p(v, f32p))
        return Csr(m, n, rp, ci, v)

    def layer_dense(self, w: Csr, bias, y, clip=0.0) -> np.ndarray:
        y = np.ascontiguousarray(y, np.float32)
        bias = np.ascontiguousarray(bias, np.float32)
        out = np.zeros((w.rows, y.shape[1]), np.float32)
        self.lib.sko_layer_dense(w.rows, w.cols, _p(w.row_ptr, u32p), _p(w.col_idx, u32p),
                                 _p(w.values, f32p), _p(bias, f32p), clip, y.shape[1],
                                 _p(y, f32p), _p(out, f32p))
        return out

    def layer_sparse(self, w: Csr, bias, y: Csr, clip=0.0) -> Csr:
        bias = np.ascontiguousarray(bias, np.float32)
        orp, oci, ov = u32p(), u32p(), f32p()
        nnz = self.lib.sko_layer_sparse(w.rows, w.cols, _p(w.row_ptr, u32p),
                                        _p(w.col_idx, u32p), _p(w.values, f32p),
                                        _p(bias, f32p), clip, y.cols, _p(y.row_ptr, u32p),
                                        _p(y.col_idx, u32p), _p(y.values, f32p),
                                        C.byref(orp), C.byref(oci), C.byref(ov))
        rp = np.ctypeslib.as_array(orp, shape=(w.rows + 1,)).copy()
        ci = np.ctypeslib.as_array(oci, shape=(max(nnz, 1),))[:nnz].copy()
        v = np.ctypeslib.as_array(ov, shape=(max(nnz, 1),))[:nnz].copy()
        for p in (orp, oci, ov):
            self.lib.sko_free(C.cast(p, C.c_void_p))
        return Csr(w.rows, y.cols, rp, ci, v)

    def sparse_epilogue(self, z: Csr, bias, clip=0.0) -> Csr:
        bias = np.ascontiguousarray(bias, np.float32)
        orp, oci, ov = u32p(), u32p(), f32p()
        nnz = self.lib.sko_sparse_epilogue(z.rows, z.cols, _p(z.row_ptr, u32p), _p(z.col_idx, u32p),
                                           _p(z.values, f32p), _p(bias, f32p), clip,
                                           C.byref(orp), C.byref(oci), C.byref(ov))
        rp = np.ctypeslib.as_array(orp, shape=(z.rows + 1,)).copy()
        ci = np.ctypeslib.as_array(oci, shape=(max(nnz, 1),))[:nnz].copy()
        v = np.ctypeslib.as_array(ov, shape=(max(nnz, 1),))[:nnz].copy()
        for p in (orp, oci, ov):
            self.lib.sko_free(C.cast(p, C.c_void_p))
        return Csr(z.rows, z.cols, rp, ci, v)

    def categories_sparse(self, y: Csr) -> np.ndarray:
        f = np.zeros(y.cols, np.uint8)
        self.lib.sko_categories_sparse(y.rows, y.cols, _p(y.row_ptr, u32p),
                                       _p(y.col_idx, u32p), _p(y.values, f32p), _p(f, u8p))
        return np.nonzero(f)[0].astype(np.uint32)

    def categories_dense(self, y: np.ndarray) -> np.ndarray:
        y = np.ascontiguousarray(y, np.float32)
        f = np.zeros(y.shape[1], np.uint8)
        self.lib.sko_categories_dense(y.shape[0], y.shape[1], _p(y, f32p), _p(f, u8p))
        return np.nonzero(f)[0].astype(np.uint32)
