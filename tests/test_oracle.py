"""CPU: the oracle (C restatement) pinned against the reference library and the
committed golden fixtures.  No GPU needed."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.oracle import csr


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_splitmix_matches_reference(port, ref):
    for seed, idx in [(0, 0), (42, 1), (2**63 + 5, 12345), (7, 2**40)]:
        assert port.splitmix_at(seed, idx) == ref.splitmix_at(seed, idx)


def test_gen_input_is_reference_formula(port, ref):
    assert np.array_equal(bits(port.gen_input_dense(37, 11, 9)), bits(ref.gen_input(37, 11, 9)))


def test_fixed_rows_generator_properties(port):
    rows = port.gen_fixed_rows(200, 1000, 32, 5)
    assert rows.shape == (200, 32)
    assert (np.diff(rows.astype(np.int64), axis=1) > 0).all()  # sorted, distinct
    assert rows.max() < 1000
    w = port.gen_layer_fixed(512, 16, 11)
    # exactly 16 nonzeros per row of W (Y.W orientation) == per column of W_ref
    assert np.array_equal(np.bincount(w.col_idx, minlength=512), np.full(512, 16))
    assert (w.values >= -1).all() and (w.values < 1).all() and (w.values != 0).all()


def test_binary_input_shards_concatenate(port):
    full = port.gen_input_binary(300, 40, 7, 3).to_dense()
    part = port.gen_input_binary(300, 15, 7, 3, sample_offset=25).to_dense()
    assert np.array_equal(full[:, 25:40], part)
    assert (full.sum(axis=0) == 7).all()


def test_layer_dense_bitwise_equals_reference_relu_forward(port, ref):
    seed, m, n, L = 5, 256, 96, 3
    Ws = [port.gen_layer_fixed(m, 16, port.layer_seed(seed, k)) for k in range(L)]
    bs = [np.full(m, -0.05, np.float32) for _ in range(L)]
    y = y0 = port.gen_input_dense(m, n, seed)
    for k in range(L):
        y = port.layer_dense(Ws[k], bs[k], y)
    assert np.array_equal(bits(y), bits(ref.relu_forward(Ws, bs, y0, workers=3)))


def test_layer_sparse_bitwise_equals_reference_csr_csr_plus_epilogue(port, ref):
    m, n = 2048, 64
    W = port.gen_layer_fixed(m, 32, 99, 1.0 / 16)
    Y = port.gen_input_binary(m, n, 150, 1)
    b = np.full(m, -0.05, np.float32)
    Z = ref.mxm_csr_csr(W, Y, workers=2)
    Zd = Z.to_dense()
    touched = np.zeros(Zd.shape, bool)
    for i in range(m):
        touched[i, Z.col_idx[Z.row_ptr[i]:Z.row_ptr[i + 1]]] = True
    z = (Zd + b[:, None]).astype(np.float32)
    z = np.where(z < 0, np.float32(0), z)
    z = np.where(z > 32, np.float32(32), z)
    expect = np.where(touched, z, 0).astype(np.float32)
    got = port.layer_sparse(W, b, Y, 32.0).to_dense()
    assert np.array_equal(bits(got), bits(expect))


def test_layer_sparse_equals_reference_dense_route(port, ref):
    # random U[-1,1) weights and dense U[0,1) input through the sparse route
    m, n = 300, 20
    W = port.gen_layer_fixed(m, 16, 4)
    y0 = port.gen_input_dense(m, n, 8)
    Y = ref.from_dense(y0)
    b = np.full(m, -0.05, np.float32)
    out = port.layer_sparse(W, b, Y, 0.0)
    assert np.array_equal(bits(out.to_dense()), bits(ref.layer_step(W, b, y0)))


def test_layer_sparse_positive_bias_densifies_like_reference(port, ref):
    m, n = 64, 9
    W = port.gen_layer_fixed(m, 4, 4)
    y0 = np.zeros((m, n), np.float32)
    y0[3, 2] = 1.0
    b = np.where(np.arange(m) % 3 == 0, 0.25, -0.5).astype(np.float32)
    out = port.layer_sparse(W, b, ref.from_dense(y0), 0.0)
    assert np.array_equal(bits(out.to_dense()), bits(ref.layer_step(W, b, y0)))


def test_golden_cfg1_regenerates(port):
    g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    m, n, L, k, seed = (int(g[x]) for x in ("m", "n", "L", "k", "seed"))
    Ws = [port.gen_layer_fixed(m, k, port.layer_seed(seed, i)) for i in range(L)]
    assert np.array_equal(Ws[0].row_ptr, g["w0_rp"]) and np.array_equal(Ws[0].col_idx, g["w0_ci"])
    y = port.gen_input_dense(m, n, seed)
    for i in range(L):
        y = port.layer_dense(Ws[i], np.full(m, g["bias"], np.float32), y)
    assert np.array_equal(bits(y), bits(g["yL"]))
    assert np.array_equal(port.categories_dense(y), g["categories"])


def test_golden_cfg2_small(port):
    g = np.load(os.path.join(GOLDEN, "cfg2_small.npz"))
    m, n, seed = int(g["m"]), int(g["n"]), int(g["seed"])
    y = port.gen_input_dense(m, n, seed)
    for d in (0.01, 0.001):
        key = f"d{d:g}".replace(".", "p")
        W = port.gen_layer_density(m, d, port.layer_seed(seed, 0))
        assert W.nnz == int(g[f"{key}_nnz"])
        out = port.layer_dense(W, np.full(m, -0.05, np.float32), y)
        assert np.array_equal(bits(out), bits(g[f"{key}_out"]))


def test_golden_cfg3_small(port):
    g = np.load(os.path.join(GOLDEN, "cfg3_small.npz"))
    m, n, L, kY, seed = (int(g[x]) for x in ("m", "n", "L", "kY", "seed"))
    Y = port.gen_input_binary(m, n, kY, seed)
    trace = [Y.nnz]
    for k in range(L):
        W = port.gen_layer_fixed(m, 32, port.layer_seed(seed, k), 1.0 / 16)
        Y = port.layer_sparse(W, np.full(m, -0.3, np.float32), Y, 32.0)
        trace.append(Y.nnz)
    assert trace == list(g["trace"])
    assert np.array_equal(Y.row_ptr, g["yL_rp"]) and np.array_equal(Y.col_idx, g["yL_ci"])


def test_golden_random_models_against_reference(ref):
    g = np.load(os.path.join(GOLDEN, "random_models.npz"))
    for t in range(12):
        mm, layers, nn = (int(x) for x in g[f"t{t}_meta"])
        Ws = [csr(mm, mm, g[f"t{t}_w{k}_rp"], g[f"t{t}_w{k}_ci"], g[f"t{t}_w{k}_v"])
              for k in range(layers)]
        bs = [g[f"t{t}_b{k}"] for k in range(layers)]
        out = ref.relu_forward(Ws, bs, g[f"t{t}_y0"])
        assert np.array_equal(bits(out), bits(g[f"t{t}_out"]))


def test_kat_fixture_matches_reference(ref):
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))
    assert kat["hand_layer"] == [[4.0], [0.0]]  # test_dnn.cpp:95-105
    assert kat["identity_clamp"] == [[3.0], [0.0]]  # test_dnn.cpp:85-93
    assert kat["mxm_arith"] == [[17.0], [39.0]]  # test_matrix.cpp:230-236
    assert kat["mxm_maxplus"] == [[8.0], [10.0]]  # test_matrix.cpp:237-243
    assert kat["triple_errors"]["duplicate"]["kind"] == "InvalidArgument"
    assert kat["validate_errors"]["stored_zero_ok"] is None
