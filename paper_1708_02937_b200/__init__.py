"""B200-native sparse ReLU DNN engine (Kepner et al., arXiv 1708.02937 hot path).

``semikern`` mirrors the reference's operator API; the compute is the CUDA
library libsk_b200.so (sm_100a) reached through include/sk_api.h.
"""
from . import _lib  # noqa: F401
from .semikern import *  # noqa: F401,F403
from .semikern import (  # noqa: F401
    Batch, Context, CsrMatrix, DenseMatrix, DnnModel, ForwardOptions, Matrix, Triple,
    categories, default_context, gen_input_binary, gen_input_dense, gen_layer_density,
    gen_layer_fixed, layer_seed, relu_forward_host, relu_forward_sparse, set_device,
)

__all__ = [n for n in dir() if not n.startswith("_")]
