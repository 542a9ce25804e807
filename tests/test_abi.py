"""CPU: the C-ABI library builds, loads and exports every symbol that
include/sk_api.h declares; without a device it fails loudly (no fallback)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "sk_api.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("sk_csr_from_triples", "sk_mxm_csr_dense", "sk_mxm_csr_csr", "sk_layer_step",
              "sk_relu_forward", "sk_relu_forward_sparse", "sk_from_dense", "sk_csr_extract",
              "sk_ewise_dense", "sk_dense_mxm_baseline", "sk_categories_csr"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1708_02937_b200 import _lib
    L = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == declared_symbols()


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_1708_02937_b200", "libsk_b200.so")
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    import paper_1708_02937_b200 as sk
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    with pytest.raises(sk.CudaError):
        sk.Context(0)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1708_02937_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "libsk_oracle", "libsemikern_ref", "skref_", "sko_"):
                    assert bad not in src, (f, bad)


def test_semiring_helpers_mirror_reference():
    import paper_1708_02937_b200 as sk
    assert sk.approx_equal(1.0, 1.0 + 5e-6)
    assert not sk.approx_equal(1.0, 1.0 + 5e-5)
    assert sk.approx_equal_scaled(0.0, 5e-6, 1.0)
    assert sk.semiring_by_name("maxplus").zero == float("-inf")
    with pytest.raises(sk.InvalidArgument):
        sk.semiring_by_name("tropical")
    assert sk.csr_storage_bytes(7, 12) == 8 * 4 + 12 * 8
    assert sk.dense_storage_bytes(32768, 32768) == 4 * 1024 ** 3
