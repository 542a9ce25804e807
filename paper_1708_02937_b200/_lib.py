"""ctypes binding of libsk_b200.so (include/sk_api.h).

The product has exactly one compute path: the CUDA library.  If the shared
object is missing or no CUDA device is usable, every call raises -- there is
no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SK_LIB_PATH selects an alternative build (tuning experiments only)
LIB_PATH = os.environ.get("SK_LIB_PATH") or os.path.join(HERE, "libsk_b200.so")

u32p = C.POINTER(C.c_uint32)
f32p = C.POINTER(C.c_float)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p

SK_OK = 0

# every symbol include/sk_api.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "sk_last_error", "sk_version", "sk_kernel_launch_count",
    "sk_ctx_create", "sk_ctx_destroy", "sk_ctx_set_stream", "sk_ctx_stream",
    "sk_ctx_synchronize", "sk_ctx_set_timing", "sk_ctx_kernel_times", "sk_ctx_kernel_times_tagged",
    "sk_ctx_timer_start", "sk_ctx_timer_stop",
    "sk_ctx_layer_stamps", "sk_ctx_layer_paths", "sk_ctx_set_density_switch",
    "sk_ctx_set_tuning", "sk_ctx_get_tuning", "sk_ctx_last_exact",
    "sk_host_register", "sk_host_unregister",
    "sk_dense_create", "sk_dense_upload", "sk_dense_write", "sk_dense_download",
    "sk_dense_download_async", "sk_dense_shape", "sk_dense_device_ptr",
    "sk_dense_identity", "sk_dense_free",
    "sk_csr_from_triples", "sk_csr_from_parts", "sk_csr_from_pattern", "sk_csr_from_pattern_async",
    "sk_csr_from_pattern16_async",
    "sk_csr_shape",
    "sk_csr_extract",
    "sk_csr_free", "sk_to_dense", "sk_from_dense", "sk_dense_nnz",
    "sk_ewise_dense", "sk_ewise_csr", "sk_ewise_mixed",
    "sk_mxm_csr_dense", "sk_mxm_dense_dense", "sk_mxm_csr_csr", "sk_dense_mxm_baseline",
    "sk_model_create", "sk_model_shape", "sk_model_free",
    "sk_layer_step", "sk_relu_forward", "sk_relu_forward_host", "sk_relu_forward_sparse",
    "sk_categories_csr", "sk_categories_dense",
    "sk_sparse_layer", "sk_sparse_layer_dev", "sk_sparse_layer_stage", "sk_staged_publish",
    "sk_staged_free", "sk_csr_device_arrays", "sk_csr_from_device", "sk_memcpy_d2d",
    "sk_ipc_alloc", "sk_ipc_open", "sk_ipc_close", "sk_ipc_free", "sk_csr_publish",
    "sk_dense_layer_step", "sk_dense_relu_forward",
    "sk_gen_layer_fixed", "sk_gen_layer_density", "sk_gen_weight",
    "sk_read_matrix", "sk_read_matrix_text", "sk_write_matrix", "sk_format_matrix", "sk_gen_input_dense",
    "sk_gen_input_binary", "sk_layer_seed",
]


class FwdOpts(C.Structure):
    _fields_ = [("workers", C.c_int), ("materialize_bias", C.c_int), ("clip", C.c_float)]


class Tuning(C.Structure):  # sk_tuning
    _fields_ = [("exact", C.c_int), ("exact_kernel", C.c_int), ("exact_group", C.c_int),
                ("exact_records", C.c_int), ("window_log2", C.c_int),
                ("exact_window_log2", C.c_int), ("esc", C.c_int), ("esc_ratio", C.c_double),
                ("exact_fields", C.c_int), ("exact_layout", C.c_int)]


class ExactInfo(C.Structure):  # sk_exact_info
    _fields_ = [("launches", C.c_uint64), ("kernel", C.c_int), ("group", C.c_int),
                ("records", C.c_int), ("window_log2", C.c_int), ("fields", C.c_int),
                ("wraps", C.c_int), ("layout", C.c_int)]


_lib = None


def load() -> C.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `make -C paper_1708_02937_b200` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    L.sk_last_error.restype = C.c_char_p
    L.sk_version.restype = C.c_char_p
    L.sk_kernel_launch_count.restype = C.c_uint64
    L.sk_ctx_stream.restype = vp
    L.sk_ctx_stream.argtypes = [vp]
    L.sk_dense_device_ptr.restype = vp
    L.sk_dense_device_ptr.argtypes = [vp]
    L.sk_layer_seed.restype = C.c_uint64
    L.sk_layer_seed.argtypes = [C.c_uint64, C.c_uint32]
    for name in ("sk_ctx_destroy", "sk_dense_free", "sk_csr_free", "sk_model_free",
                 "sk_ctx_synchronize"):
        getattr(L, name).argtypes = [vp]
    L.sk_ctx_set_stream.argtypes = [vp, vp]
    L.sk_ctx_set_timing.argtypes = [vp, C.c_int]
    L.sk_ctx_kernel_times.argtypes = [vp, f32p, C.c_size_t, C.POINTER(C.c_size_t)]
    L.sk_ctx_kernel_times_tagged.argtypes = [vp, f32p, C.POINTER(C.c_int), C.c_size_t,
                                             C.POINTER(C.c_size_t)]
    L.sk_ctx_layer_stamps.argtypes = [vp, C.POINTER(C.c_longlong), C.c_size_t]
    L.sk_ctx_timer_start.argtypes = [vp]
    L.sk_ctx_timer_stop.argtypes = [vp, f32p]
    L.sk_ctx_layer_paths.argtypes = [vp, C.POINTER(C.c_ubyte), C.c_size_t]
    L.sk_ctx_set_density_switch.argtypes = [vp, C.c_double, C.c_double]
    L.sk_ctx_set_tuning.argtypes = [vp, C.POINTER(Tuning)]
    L.sk_ctx_get_tuning.argtypes = [vp, C.POINTER(Tuning)]
    L.sk_ctx_last_exact.argtypes = [vp, C.POINTER(ExactInfo)]
    L.sk_host_register.argtypes = [vp, C.c_size_t]
    L.sk_host_unregister.argtypes = [vp]
    L.sk_dense_create.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_float, C.POINTER(vp)]
    L.sk_dense_upload.argtypes = [vp, C.c_uint32, C.c_uint32, vp, C.POINTER(vp)]
    L.sk_dense_write.argtypes = [vp, vp, vp]
    L.sk_dense_download.argtypes = [vp, vp, vp]
    L.sk_dense_download_async.argtypes = [vp, vp, vp]
    L.sk_dense_shape.argtypes = [vp, u32p, u32p]
    L.sk_dense_identity.argtypes = [vp, C.c_uint32, C.POINTER(vp)]
    L.sk_csr_from_triples.argtypes = [vp, C.c_uint32, C.c_uint32, vp, vp, vp, C.c_size_t,
                                      C.POINTER(vp)]
    L.sk_csr_from_parts.argtypes = [vp, C.c_uint32, C.c_uint32, vp, vp, vp, C.c_int,
                                    C.POINTER(vp)]
    L.sk_csr_from_pattern.argtypes = [vp, C.c_uint32, C.c_uint32, vp, vp, C.c_float, C.c_int,
                                      C.POINTER(vp)]
    L.sk_csr_from_pattern_async.argtypes = [vp, C.c_uint32, C.c_uint32, vp, vp, C.c_float, vp,
                                            C.POINTER(vp)]
    L.sk_csr_from_pattern16_async.argtypes = [vp, C.c_uint32, C.c_uint32, vp, vp, C.c_float, vp,
                                              C.POINTER(vp)]
    L.sk_csr_shape.argtypes = [vp, u32p, u32p, C.POINTER(C.c_size_t)]
    L.sk_csr_extract.argtypes = [vp, vp, vp, vp, vp]
    L.sk_to_dense.argtypes = [vp, vp, C.c_float, C.POINTER(vp)]
    L.sk_from_dense.argtypes = [vp, vp, C.POINTER(vp)]
    L.sk_dense_nnz.argtypes = [vp, vp, C.POINTER(C.c_size_t)]
    L.sk_ewise_dense.argtypes = [vp, C.c_int, vp, vp, C.c_int, C.POINTER(vp)]
    L.sk_ewise_csr.argtypes = [vp, C.c_int, vp, vp, C.c_int, C.POINTER(vp)]
    L.sk_ewise_mixed.argtypes = [vp, C.c_int, vp, vp, C.c_int, C.c_int, C.POINTER(vp)]
    L.sk_mxm_csr_dense.argtypes = [vp, vp, vp, C.c_int, C.POINTER(vp)]
    L.sk_mxm_dense_dense.argtypes = [vp, vp, vp, C.c_int, C.POINTER(vp)]
    L.sk_mxm_csr_csr.argtypes = [vp, vp, vp, C.c_int, C.POINTER(vp)]
    L.sk_dense_mxm_baseline.argtypes = [vp, vp, vp, C.POINTER(vp)]
    L.sk_model_create.argtypes = [vp, C.c_uint32, C.POINTER(vp), C.POINTER(f32p),
                                  C.POINTER(vp)]
    L.sk_model_shape.argtypes = [vp, u32p, u32p]
    L.sk_layer_step.argtypes = [vp, vp, vp, vp, C.POINTER(FwdOpts), C.POINTER(vp)]
    L.sk_relu_forward.argtypes = [vp, vp, vp, C.POINTER(FwdOpts), C.POINTER(vp)]
    L.sk_relu_forward_host.argtypes = [vp, vp, C.c_uint32, vp, C.POINTER(FwdOpts), vp]
    L.sk_relu_forward_sparse.argtypes = [vp, vp, vp, C.POINTER(FwdOpts), C.POINTER(vp), vp]
    L.sk_sparse_layer.argtypes = [vp, vp, vp, vp, C.c_float, C.POINTER(vp)]
    L.sk_sparse_layer_dev.argtypes = [vp, vp, vp, C.c_uint64, C.c_double, vp, C.c_float,
                                      C.POINTER(vp)]
    L.sk_sparse_layer_stage.argtypes = [vp, vp, vp, C.c_uint64, C.c_double, vp, C.c_float,
                                        C.POINTER(vp), C.POINTER(C.c_uint64)]
    L.sk_staged_publish.argtypes = [vp, vp, C.c_uint32, C.POINTER(vp), C.POINTER(vp),
                                    C.POINTER(vp), C.c_uint32, C.c_uint64, C.c_int]
    L.sk_staged_free.argtypes = [vp]
    L.sk_csr_device_arrays.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]
    L.sk_csr_from_device.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_size_t, vp, vp, vp,
                                     C.POINTER(vp)]
    L.sk_memcpy_d2d.argtypes = [vp, vp, vp, C.c_size_t]
    L.sk_ipc_alloc.argtypes = [vp, C.c_size_t, C.POINTER(vp), C.c_char_p]
    L.sk_ipc_open.argtypes = [vp, C.c_char_p, C.POINTER(vp)]
    L.sk_ipc_close.argtypes = [vp]
    L.sk_ipc_free.argtypes = [vp]
    L.sk_csr_publish.argtypes = [vp, vp, C.c_uint32, C.POINTER(vp), C.POINTER(vp),
                                 C.POINTER(vp), C.c_uint32, C.c_uint64, C.c_int]
    L.sk_categories_csr.argtypes = [vp, vp, vp, C.c_size_t, C.POINTER(C.c_size_t)]
    L.sk_categories_dense.argtypes = [vp, vp, vp, C.c_size_t, C.POINTER(C.c_size_t)]
    L.sk_dense_layer_step.argtypes = [vp, vp, vp, vp, C.POINTER(vp)]
    L.sk_dense_relu_forward.argtypes = [vp, vp, vp, C.POINTER(vp)]
    L.sk_gen_layer_fixed.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint64, C.c_float,
                                     C.POINTER(vp)]
    L.sk_gen_weight.argtypes = [vp, C.c_uint32, C.c_double, C.c_uint64, C.POINTER(vp)]
    L.sk_read_matrix.argtypes = [vp, C.c_char_p, C.POINTER(C.c_int), C.POINTER(vp),
                                 C.POINTER(vp)]
    L.sk_read_matrix_text.argtypes = [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_int),
                                      C.POINTER(vp), C.POINTER(vp)]
    L.sk_write_matrix.argtypes = [vp, vp, vp, C.c_char_p]
    L.sk_format_matrix.argtypes = [vp, vp, vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
    L.sk_gen_layer_density.argtypes = [vp, C.c_uint32, C.c_double, C.c_uint64, C.POINTER(vp)]
    L.sk_gen_input_dense.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(vp)]
    L.sk_gen_input_binary.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                      C.c_uint64, C.POINTER(vp)]
    _lib = L
    return L


def launches() -> int:
    return int(load().sk_kernel_launch_count())
