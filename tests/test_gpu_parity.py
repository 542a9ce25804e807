"""GPU parity: the CUDA path (through the C-ABI) against the reference
library (oracle/_ref), the C restatement (oracle/_build) and the committed
golden fixtures.  Bitwise for the sparse path; the tensor-core dense leg is
checked with the reference's magnitude-scaled tolerance
(approx_equal_scaled, semiring.hpp:50-55, kRelTol = 1e-5)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.oracle import csr as hcsr

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def same_bits_nan(a, b):
    """Bitwise equal except NaN payloads: the GPU emits the canonical NaN
    (0x7fffffff) where x86 propagates the input payload, so NaN positions must
    match and every other value must be bit-identical."""
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(bits(a)[~na], bits(b)[~nb])


def dev_csr(sk, a):
    return sk.CsrMatrix(a.rows, a.cols, a.row_ptr, a.col_idx, a.values)


def host_csr(a):
    rp, ci, v = a.extract()
    return hcsr(a.rows(), a.cols(), rp, ci, v)


def assert_csr_bitwise(got, want, nan_payloads=False):
    g = host_csr(got)
    assert g.rows == want.rows and g.cols == want.cols
    assert np.array_equal(g.row_ptr, want.row_ptr)
    assert np.array_equal(g.col_idx, want.col_idx)
    if nan_payloads:  # NaN positions equal, payloads free (see same_bits_nan)
        assert same_bits_nan(g.values, want.values)
    else:
        assert np.array_equal(bits(g.values), bits(want.values))


# ---- known answers (proj/tests/test_dnn.cpp, test_matrix.cpp) ---------------------------

def test_known_answers(sk):
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))
    I2 = sk.DnnModel([sk.Matrix(sk.DenseMatrix.identity(2))], [[0.0, 0.0]])
    x = sk.DenseMatrix(2, 1, [3.0, -2.0])
    assert sk.relu_forward(I2, x).numpy().tolist() == kat["identity_clamp"]
    assert sk.dense_relu_forward(I2, x).numpy().tolist() == kat["identity_clamp"]
    W = sk.DenseMatrix(2, 2, [1, 2, 3, 4])
    model = sk.DnnModel([sk.Matrix(W)], [[1.0, -100.0]])
    assert sk.relu_forward(model, sk.DenseMatrix(2, 1, 1.0)).numpy().tolist() == kat["hand_layer"]
    assert sk.dense_relu_forward(model, sk.DenseMatrix(2, 1, 1.0)).numpy().tolist() == kat["hand_layer"]
    B = sk.DenseMatrix(2, 1, [5, 6])
    assert sk.mxm(W, B, sk.arithmetic_semiring()).numpy().tolist() == kat["mxm_arith"]
    assert sk.mxm(W, B, sk.max_plus_semiring()).numpy().tolist() == kat["mxm_maxplus"]
    neg = sk.DnnModel([sk.Matrix(sk.DenseMatrix(2, 2, [-1, -2, -3, -4]))], [[-1.0, -1.0]])
    assert sk.dense_relu_forward(neg, sk.DenseMatrix(2, 2, [1, 2, 1, 2])).numpy().tolist() == \
        kat["all_negative"]
    empty = sk.csr_from_triples(3, 3, [])
    assert sk.layer_step(sk.Matrix(empty), [0.0] * 3, sk.DenseMatrix(3, 2, 1.0)).numpy().tolist() \
        == kat["empty_w"]
    I4 = sk.Matrix(sk.DenseMatrix.identity(4))
    assert sk.layer_step(I4, [-1.0] * 4, sk.DenseMatrix(4, 3, 1.0)).numpy().tolist() == \
        kat["identity_minus1"]


def test_csr_from_triples_matches_reference(sk, ref):
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))
    t = sk.csr_from_triples(1, 3, [(0, 2, 3.0), (0, 0, 1.0), (0, 1, 2.0)])
    assert t.row_ptr().tolist() == kat["triples_sorted"]["rp"]
    assert t.col_idx().tolist() == kat["triples_sorted"]["ci"]
    assert t.values().tolist() == kat["triples_sorted"]["v"]
    t = sk.csr_from_triples(2, 2, [(0, 0, 0.0), (1, 1, 2.0)])
    assert t.nnz() == 1 and t.row_ptr().tolist() == kat["triples_zero_elided"]["rp"]
    cases = {"out_of_range": (2, 2, [2], [0], [1.0]),
             "duplicate": (2, 2, [0, 0], [1, 1], [1.0, 2.0]),
             "dup_after_sort": (3, 3, [2, 0, 2, 1], [1, 0, 1, 2], [1.0, 1.0, 5.0, 0.0]),
             "first_bad_in_input_order": (4, 4, [0, 9, 5], [0, 1, 0], [1., 1., 1.])}
    for name, (rows, cols, r, c, v) in cases.items():
        with pytest.raises(sk.InvalidArgument) as e:
            sk.csr_from_triples(rows, cols, (r, c, v))
        assert str(e.value) == kat["triple_errors"][name]["msg"], name
    # random triples, shuffled, with zeros: same CSR as the reference
    rng = np.random.default_rng(3)
    flat = rng.choice(300 * 200, size=5000, replace=False)
    r, c = (flat // 200).astype(np.uint32), (flat % 200).astype(np.uint32)
    v = rng.uniform(-1, 1, 5000).astype(np.float32)
    v[::7] = 0.0
    assert_csr_bitwise(sk.csr_from_triples(300, 200, (r, c, v)),
                       ref.csr_from_triples(300, 200, r, c, v))
    e = sk.csr_from_triples(2, 2, [])
    assert e.nnz() == 0 and e.row_ptr().tolist() == [0, 0, 0]


def test_csr_from_pattern(sk, port):
    Y = port.gen_input_binary(4096, 700, 50, 3)
    a = sk.CsrMatrix.from_pattern(Y.rows, Y.cols, Y.row_ptr, Y.col_idx, 1.0)
    assert_csr_bitwise(a, Y)
    b = sk.CsrMatrix.from_pattern(2, 3, [0, 1, 3], [2, 0, 1], -0.5)
    assert b.values().tolist() == [-0.5, -0.5, -0.5] and b.col_idx().tolist() == [2, 0, 1]
    with pytest.raises(sk.InvalidArgument):
        sk.CsrMatrix.from_pattern(1, 2, [0, 2], [1, 0], 1.0)  # not increasing
    e = sk.CsrMatrix.from_pattern(3, 3, [0, 0, 0, 0], [], 1.0)
    assert e.nnz() == 0


@pytest.mark.parametrize("c", [1.0, 0.375, -2.0, 0.0, float("nan"), 3e-39, 6.0])
def test_pattern_inputs_forward_like_explicit_values(sk, port, c):
    # a constant-valued input's statistics are known on the host (no device
    # pass): the forward must match the same matrix built from explicit values
    # and the oracle, whatever path the statistics select
    m, n, L = 2048, 1500, 3
    Y = port.gen_input_binary(m, n, 40, 9)
    vals = np.full(Y.nnz, c, np.float32)
    a = sk.CsrMatrix.from_pattern(m, n, Y.row_ptr, Y.col_idx, c)
    b = sk.CsrMatrix(m, n, Y.row_ptr, Y.col_idx, vals)
    hW = [port.gen_layer_fixed(m, 16, port.layer_seed(4, k), 1.0 / 8) for k in range(L)]
    bias = np.full(m, -0.25, np.float32)
    model = sk.DnnModel([dev_csr(sk, w) for w in hW], [bias] * L)
    oa, ta = sk.relu_forward_sparse(model, a, sk.ForwardOptions(clip=4.0))
    ob, tb = sk.relu_forward_sparse(model, b, sk.ForwardOptions(clip=4.0))
    from oracle.oracle import Csr
    y = Csr(m, n, Y.row_ptr, Y.col_idx, vals)
    for k in range(L):
        y = port.layer_sparse(hW[k], bias, y, 4.0)
    assert list(ta) == list(tb)
    assert_csr_bitwise(oa, y, nan_payloads=np.isnan(c))
    assert_csr_bitwise(ob, y, nan_payloads=np.isnan(c))


def test_csr_from_pattern_async(sk, port):
    # copies on another stream; every use is ordered after them (event on the
    # handle): extract, a forward, and freeing a handle nobody used
    import torch
    cs = torch.cuda.Stream()
    m, n, L = 4096, 2000, 2
    Y = port.gen_input_binary(m, n, 40, 11)
    a = sk.CsrMatrix.from_pattern_async(m, n, Y.row_ptr, Y.col_idx, 1.0, stream=cs.cuda_stream)
    assert_csr_bitwise(a, Y)
    hW = [port.gen_layer_fixed(m, 16, port.layer_seed(6, k), 1.0 / 8) for k in range(L)]
    bias = np.full(m, -0.2, np.float32)
    model = sk.DnnModel([dev_csr(sk, w) for w in hW], [bias] * L)
    ya = sk.CsrMatrix.from_pattern_async(m, n, Y.row_ptr, Y.col_idx, 1.0, stream=cs.cuda_stream)
    yb = sk.CsrMatrix.from_pattern(m, n, Y.row_ptr, Y.col_idx, 1.0)
    oa, ta = sk.relu_forward_sparse(model, ya, sk.ForwardOptions(clip=4.0))
    ob, tb = sk.relu_forward_sparse(model, yb, sk.ForwardOptions(clip=4.0))
    assert list(ta) == list(tb)
    assert_csr_bitwise(oa, host_csr(ob))
    unused = sk.CsrMatrix.from_pattern_async(m, n, Y.row_ptr, Y.col_idx, 2.0,
                                             stream=cs.cuda_stream)
    del unused
    torch.cuda.synchronize()


def test_validating_constructor_messages(sk):
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))["validate_errors"]
    cases = {"not_monotone": (3, 2, [0, 1, 0, 1], [0], [1.0]),
             "cols_not_increasing": (1, 2, [0, 2], [1, 0], [1.0, 2.0]),
             "col_out_of_range": (1, 2, [0, 1], [5], [1.0])}
    for name, (rows, cols, rp, ci, v) in cases.items():
        with pytest.raises(sk.InvalidArgument) as e:
            sk.CsrMatrix(rows, cols, rp, ci, v)
        assert str(e.value) == kat[name]["msg"]
    assert sk.CsrMatrix(1, 2, [0, 2], [0, 1], [0.0, 2.0]).nnz() == 2  # stored zero allowed
    with pytest.raises(sk.InvalidArgument):
        sk.CsrMatrix(2, 2, [0, 1], [0], [1.0])  # row_ptr length != rows+1


# ---- generators are bitwise the oracle's ------------------------------------------------

def test_device_generators_match_oracle(sk, port):
    a = sk.gen_layer_fixed(2048, 32, 77, 1.0 / 16)
    assert_csr_bitwise(a, port.gen_layer_fixed(2048, 32, 77, 1.0 / 16))
    a = sk.gen_layer_fixed(1024, 16, 78)
    assert_csr_bitwise(a, port.gen_layer_fixed(1024, 16, 78))
    a = sk.gen_layer_density(512, 0.05, 79)
    assert_csr_bitwise(a, port.gen_layer_density(512, 0.05, 79))
    y = sk.gen_input_dense(300, 70, 80)
    assert np.array_equal(bits(y.numpy()), bits(port.gen_input_dense(300, 70, 80)))
    b = sk.gen_input_binary(4096, 500, 60, 81, sample_offset=1234)
    assert_csr_bitwise(b, port.gen_input_binary(4096, 500, 60, 81, 1234))


# ---- the dense-activation path (K1) ---------------------------------------------------------

def test_cfg1_full_bitwise_vs_reference_golden(sk):
    g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    m, n, L, k, seed = (int(g[x]) for x in ("m", "n", "L", "k", "seed"))
    Ws = [sk.gen_layer_fixed(m, k, sk.layer_seed(seed, i)) for i in range(L)]
    model = sk.DnnModel(Ws, [np.full(m, g["bias"], np.float32)] * L)
    y0 = sk.gen_input_dense(m, n, seed)
    out = sk.relu_forward(model, y0)
    assert np.array_equal(bits(out.numpy()), bits(g["yL"]))
    assert np.array_equal(sk.categories(out), g["categories"])
    # the reference-facing host path (H2D -> forward -> D2H)
    host = sk.relu_forward_host(model, y0.numpy())
    assert np.array_equal(bits(host), bits(g["yL"]))
    # determinism / worker independence (dnn.hpp:75-76)
    for w in (1, 2, 7):
        again = sk.relu_forward(model, y0, sk.ForwardOptions(workers=w)).numpy()
        assert np.array_equal(bits(again), bits(g["yL"]))


def test_random_models_bitwise_vs_reference(sk):
    g = np.load(os.path.join(GOLDEN, "random_models.npz"))
    for t in range(12):
        mm, layers, nn = (int(x) for x in g[f"t{t}_meta"])
        Ws = [sk.CsrMatrix(mm, mm, g[f"t{t}_w{k}_rp"], g[f"t{t}_w{k}_ci"], g[f"t{t}_w{k}_v"])
              for k in range(layers)]
        model = sk.DnnModel(Ws, [g[f"t{t}_b{k}"] for k in range(layers)])
        y0 = sk.DenseMatrix.from_numpy(g[f"t{t}_y0"])
        out = sk.relu_forward(model, y0).numpy()
        assert np.array_equal(bits(out), bits(g[f"t{t}_out"])), t
        assert (out >= 0).all()
        dout = sk.dense_relu_forward(model, y0).numpy()
        want = g[f"t{t}_dense_out"]
        scale = np.maximum(np.abs(want), 1.0)
        assert (np.abs(dout - want) <= np.maximum(1e-6, 1e-5 * scale * mm)).all(), t


def test_cfg2_small_bitwise_vs_reference_golden(sk):
    g = np.load(os.path.join(GOLDEN, "cfg2_small.npz"))
    m, n, seed = int(g["m"]), int(g["n"]), int(g["seed"])
    y = sk.gen_input_dense(m, n, seed)
    for d in (0.01, 0.001):
        key = f"d{d:g}".replace(".", "p")
        W = sk.gen_layer_density(m, d, sk.layer_seed(seed, 0))
        assert W.nnz() == int(g[f"{key}_nnz"])
        out = sk.layer_step(sk.Matrix(W), np.full(m, -0.05, np.float32), y)
        assert np.array_equal(bits(out.numpy()), bits(g[f"{key}_out"]))


def test_layer_step_matches_reference_on_odd_shapes(sk, ref, port):
    rng = np.random.default_rng(11)
    for m, n in [(1, 1), (5, 3), (33, 1), (64, 130), (257, 257), (1000, 5)]:
        W = port.gen_layer_fixed(m, min(m, 7), int(rng.integers(1 << 30)))
        y = rng.uniform(-1, 1, (m, n)).astype(np.float32)
        y[rng.random((m, n)) < 0.2] = 0.0
        b = rng.uniform(-0.5, 0.5, m).astype(np.float32)
        got = sk.layer_step(sk.Matrix(dev_csr(sk, W)), b, sk.DenseMatrix.from_numpy(y)).numpy()
        assert np.array_equal(bits(got), bits(ref.layer_step(W, b, y))), (m, n)
        got = sk.layer_step(sk.Matrix(dev_csr(sk, W)), b, sk.DenseMatrix.from_numpy(y),
                            sk.ForwardOptions(clip=0.75)).numpy()
        assert np.array_equal(bits(got), bits(port.layer_dense(W, b, y, 0.75))), (m, n)


@pytest.mark.parametrize("m,n", [(300, 1024), (257, 1500), (64, 2052)])
def test_wide_batch_forward_matches_reference(sk, ref, port, m, n):
    """The dense engine's wide-batch variant (n >= 1024: a task is a row x 256
    columns, two 16-byte loads per in-edge and lane) against the reference's
    relu_forward (dnn.cpp:86-121 over matrix.cpp:403-424): rows of 0..70 stored
    entries (more than one 32-entry batch, leftovers of every size), a ragged
    last chunk (1500 = 5 x 256 + 220, 2052 = 8 x 256 + 4), three layers; and one
    clipped layer against the restated epilogue."""
    rng = np.random.default_rng(m + n)
    Ws, bs = [], []
    for k in range(3):
        lens = rng.integers(0, 71, size=m)
        lens[::13] = 0
        lens = np.minimum(lens, m)
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
        ci = np.concatenate([np.sort(rng.choice(m, size=int(c), replace=False)) for c in lens]
                            + [np.zeros(0, np.int64)]).astype(np.uint32)
        v = rng.uniform(-1, 1, len(ci)).astype(np.float32)
        Ws.append(hcsr(m, m, rp, ci, v))
        bs.append(rng.uniform(-0.2, 0.2, m).astype(np.float32))
    y0 = rng.uniform(0, 1, (m, n)).astype(np.float32)
    y0[rng.random((m, n)) < 0.3] = 0.0
    model = sk.DnnModel([dev_csr(sk, w) for w in Ws], bs)
    got = sk.relu_forward(model, sk.DenseMatrix.from_numpy(y0)).numpy()
    assert np.array_equal(bits(got), bits(ref.relu_forward(Ws, bs, y0, workers=2)))
    clipped = sk.relu_forward(sk.DnnModel([dev_csr(sk, Ws[0])] * 2, bs[:2]),
                              sk.DenseMatrix.from_numpy(y0), sk.ForwardOptions(clip=0.5)).numpy()
    want = port.layer_dense(Ws[0], bs[1], port.layer_dense(Ws[0], bs[0], y0, 0.5), 0.5)
    assert np.array_equal(bits(clipped), bits(want))


@pytest.mark.parametrize("m,n,inv", [(2048, 64, 1.0), (512, 64, 4.0), (700, 4, 2.0),
                                     (300, 12, 1.0), (1000, 36, 16.0), (64, 8, 1.0),
                                     (1024, 7, 1.0), (4096, 33, 2.0), (333, 64, 1.0)])
def test_narrow_activation_spmm_bitwise_vs_reference(sk, ref, m, n, inv):
    # n <= 64 (n % 4 == 0) takes the sub-warp-group SpMM (n/4 lanes a row,
    # rows of different lengths in one warp); other n the row-warp K1: the
    # paper sweep's batch-64 shapes, dense-ish rows included (inverse sparsity
    # 1 = m entries a row)
    w = sk.gen_weight(m, inv, 42 + m)
    hw = host_csr(w)
    rng = np.random.default_rng(m + n)
    y = rng.uniform(-1, 1, (m, n)).astype(np.float32)
    y[rng.random((m, n)) < 0.2] = 0.0
    b = rng.uniform(-0.5, 0.5, m).astype(np.float32)
    got = sk.layer_step(sk.Matrix(w), b, sk.DenseMatrix.from_numpy(y)).numpy()
    assert np.array_equal(bits(got), bits(ref.layer_step(hw, b, y)))
    got = sk.mxm(w, sk.DenseMatrix.from_numpy(y), sk.max_plus_semiring())
    assert np.array_equal(bits(got.numpy()), bits(ref.mxm_csr_dense(hw, y, "max_plus")))


def test_special_values_follow_reference_select(sk, ref):
    # NaN propagates, -0.0 survives the ReLU select, inf saturates (F4)
    m, n = 4, 6
    W = hcsr(4, 4, [0, 1, 2, 3, 4], [0, 1, 2, 3], [1.0, 1.0, 1.0, 1.0])
    y = np.array([[np.nan, 1, -1, 0, np.inf, -np.inf]] * 4, np.float32)
    y[1] = -0.0
    b = np.zeros(4, np.float32)
    got = sk.layer_step(sk.Matrix(dev_csr(sk, W)), b, sk.DenseMatrix.from_numpy(y)).numpy()
    want = ref.layer_step(W, b, y)
    assert same_bits_nan(got, want)
    assert np.isnan(got[0, 0]) and np.isinf(got[0, 4])


def test_dimension_errors(sk):
    model = sk.DnnModel([sk.csr_from_triples(3, 3, [(0, 0, 1.0)])], [[0.0] * 3])
    with pytest.raises(sk.DimensionError):
        sk.relu_forward(model, sk.DenseMatrix(4, 2, 0.0))
    with pytest.raises(sk.DimensionError):
        sk.layer_step(sk.Matrix(sk.DenseMatrix.identity(3)), [0.0] * 3, sk.DenseMatrix(2, 2, 1.0))
    with pytest.raises(sk.DimensionError):
        sk.layer_step(sk.Matrix(sk.DenseMatrix.identity(3)), [0.0] * 2, sk.DenseMatrix(3, 2, 1.0))
    with pytest.raises(sk.InvalidArgument):
        sk.DnnModel([], [])
    with pytest.raises(sk.DimensionError):
        sk.DnnModel([sk.csr_from_triples(2, 3, [])], [[0.0, 0.0]])
    with pytest.raises(sk.DimensionError):
        sk.mxm(sk.DenseMatrix(2, 3), sk.DenseMatrix(2, 2), sk.arithmetic_semiring())
    with pytest.raises(sk.Error):
        sk.mxm(sk.Matrix(sk.DenseMatrix(2, 2)), sk.Matrix(sk.csr_from_triples(2, 2, [])),
               sk.arithmetic_semiring())


# ---- semiring kernels against the reference -----------------------------------------

SEMIRINGS = ["arithmetic", "max_plus", "min_max", "gf2"]


def sample(kind, rng, shape):
    if kind == "arithmetic":
        v = rng.uniform(-2, 2, shape).astype(np.float32)
        v[v == 0] = 1
    elif kind == "max_plus":
        v = ((rng.integers(0, 1024, shape) - 512) / 64.0).astype(np.float32)
    elif kind == "min_max":
        v = rng.uniform(0, 10, shape).astype(np.float32)
    else:
        v = np.ones(shape, np.float32)
    return v


def rand_csr(rng, rows, cols, density, kind):
    mask = rng.random((rows, cols)) < density
    vals = sample(kind, rng, (rows, cols))
    rp = np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.uint32)
    ci = np.nonzero(mask)[1].astype(np.uint32)
    return hcsr(rows, cols, rp, ci, vals[mask])


def test_mxm_wide_batch_all_semirings_match_reference(sk, ref):
    """mxm(CsrMatrix, DenseMatrix) at n >= 1024 with rows of more than 16 entries
    takes the wide row kernel (a row x 256 columns per task) under every
    semiring: bitwise against the reference (matrix.cpp:403-424), ragged last
    chunk (1028 = 4 x 256 + 4)."""
    rng = np.random.default_rng(29)
    for kind in SEMIRINGS:
        s = getattr(sk, {"arithmetic": "arithmetic_semiring", "max_plus": "max_plus_semiring",
                         "min_max": "min_max_semiring", "gf2": "gf2_semiring"}[kind])()
        a = rand_csr(rng, 37, 90, 0.5, kind)
        assert a.nnz > 16 * 37
        b = rand_csr(rng, 90, 1028, 0.6, kind)
        bd = ref.to_dense(b, s.zero)
        got = sk.mxm(dev_csr(sk, a), sk.DenseMatrix.from_numpy(bd), s).numpy()
        assert np.array_equal(bits(got), bits(ref.mxm_csr_dense(a, bd, kind))), kind


def test_mxm_all_semirings_match_reference(sk, ref):
    rng = np.random.default_rng(13)
    for kind in SEMIRINGS:
        s = getattr(sk, {"arithmetic": "arithmetic_semiring", "max_plus": "max_plus_semiring",
                         "min_max": "min_max_semiring", "gf2": "gf2_semiring"}[kind])()
        for trial in range(8):
            m, l, n = (int(x) for x in rng.integers(1, 40, 3))
            a = rand_csr(rng, m, l, 0.2 + 0.6 * rng.random(), kind)
            b = rand_csr(rng, l, n, 0.2 + 0.6 * rng.random(), kind)
            bd = ref.to_dense(b, s.zero)
            ad = ref.to_dense(a, s.zero)
            got = sk.mxm(dev_csr(sk, a), sk.DenseMatrix.from_numpy(bd), s).numpy()
            assert np.array_equal(bits(got), bits(ref.mxm_csr_dense(a, bd, kind))), (kind, trial)
            got = sk.mxm(sk.DenseMatrix.from_numpy(ad), sk.DenseMatrix.from_numpy(bd), s).numpy()
            assert np.array_equal(bits(got), bits(ref.mxm_dense_dense(ad, bd, kind))), (kind, trial)
            got = sk.mxm(dev_csr(sk, a), dev_csr(sk, b), s)
            assert_csr_bitwise(got, ref.mxm_csr_csr(a, b, kind))


def test_ewise_all_semirings_match_reference(sk, ref):
    rng = np.random.default_rng(31)
    for kind in SEMIRINGS:
        s = getattr(sk, {"arithmetic": "arithmetic_semiring", "max_plus": "max_plus_semiring",
                         "min_max": "min_max_semiring", "gf2": "gf2_semiring"}[kind])()
        for trial in range(6):
            rows, cols = (int(x) for x in rng.integers(1, 10, 2))
            a = rand_csr(rng, rows, cols, 0.4, kind)
            b = rand_csr(rng, rows, cols, 0.4, kind)
            da, db = ref.to_dense(a, s.zero), ref.to_dense(b, s.zero)
            for mul in (0, 1):
                fn = sk.ewise_mul if mul else sk.ewise_add
                got = fn(sk.DenseMatrix.from_numpy(da), sk.DenseMatrix.from_numpy(db), s).numpy()
                assert np.array_equal(bits(got), bits(ref.ewise_dense(mul, da, db, kind)))
                got = fn(sk.Matrix(dev_csr(sk, a)), sk.Matrix(dev_csr(sk, b)), s)
                assert got.is_sparse()
                assert_csr_bitwise(got.csr(), ref.ewise_csr(mul, a, b, kind))
                got = fn(sk.Matrix(dev_csr(sk, a)), sk.Matrix(sk.DenseMatrix.from_numpy(db)), s)
                assert not got.is_sparse()
                want = ref.ewise_dense(mul, da, db, kind)
                assert np.array_equal(bits(got.dense().numpy()), bits(want))


def test_gf2_domain_error_surfaces_from_kernel(sk):
    a = sk.csr_from_triples(1, 1, [(0, 0, 2.0)])
    b = sk.DenseMatrix(1, 1, 1.0)
    with pytest.raises(sk.DomainError):
        sk.mxm(a, b, sk.gf2_semiring())
    with pytest.raises(sk.DomainError):
        sk.mxm(a, b, sk.gf2_semiring(), 4)
    # the context is usable afterwards
    assert sk.mxm(sk.csr_from_triples(1, 1, [(0, 0, 1.0)]), b, sk.gf2_semiring()).numpy()[0, 0] == 1


def test_conversions_and_counts(sk, ref):
    rng = np.random.default_rng(5)
    d = rng.uniform(-1, 1, (37, 91)).astype(np.float32)
    d[rng.random(d.shape) < 0.7] = 0.0
    dd = sk.DenseMatrix.from_numpy(d)
    assert_csr_bitwise(sk.from_dense(dd), ref.from_dense(d))
    assert sk.nnz(dd) == int((d != 0).sum())
    back = sk.to_dense(sk.from_dense(dd), 0.0).numpy()
    assert np.array_equal(bits(back), bits(d))
    e = sk.to_dense(sk.csr_from_triples(3, 3, []), float("-inf")).numpy()
    assert (e == -np.inf).all()


# ---- the sparse-activation path (K3) ---------------------------------------------------------

def test_cfg3_small_sparse_forward_bitwise_vs_golden(sk):
    g = np.load(os.path.join(GOLDEN, "cfg3_small.npz"))
    m, n, L, kY, seed = (int(g[x]) for x in ("m", "n", "L", "kY", "seed"))
    Ws = [sk.gen_layer_fixed(m, 32, sk.layer_seed(seed, k), 1.0 / 16) for k in range(L)]
    model = sk.DnnModel(Ws, [np.full(m, -0.3, np.float32)] * L)
    Y0 = sk.gen_input_binary(m, n, kY, seed)
    out, trace = sk.relu_forward_sparse(model, Y0, sk.ForwardOptions(clip=32.0))
    assert list(trace) == list(g["trace"])
    want = hcsr(m, n, g["yL_rp"], g["yL_ci"], g["yL_v"])
    assert_csr_bitwise(out, want)
    assert np.array_equal(sk.categories(out), np.unique(want.col_idx))


@pytest.mark.parametrize("m,n,kY,kW,value,bias,clip,L", [
    (16384, 2500, 246, 32, 1.0 / 16, -0.3, 32.0, 2),      # cfg3 construction, several windows
    (65536, 700, 262, 32, 1.0 / 16, -0.35, 32.0, 2),      # cfg4 construction
    (4096, 3000, 400, 32, 1.0 / 16, -0.05, 32.0, 3),      # live network (slow decay)
    (2048, 600, 1200, 24, float("nan"), -0.02, 0.0, 3),   # random weights, dense-ish Y: conflicts
    (1024, 257, 100, 16, float("nan"), 0.05, 0.0, 2),     # positive bias: rows densify
])
def test_sparse_forward_bitwise_vs_oracle(sk, port, m, n, kY, kW, value, bias, clip, L):
    seed = 17
    hW = [port.gen_layer_fixed(m, kW, port.layer_seed(seed, k), value) for k in range(L)]
    b = np.full(m, bias, np.float32)
    hY = port.gen_input_binary(m, n, kY, seed)
    model = sk.DnnModel([dev_csr(sk, w) for w in hW], [b] * L)
    out, trace = sk.relu_forward_sparse(model, dev_csr(sk, hY), sk.ForwardOptions(clip=clip))
    y = hY
    want_trace = [y.nnz]
    for k in range(L):
        y = port.layer_sparse(hW[k], b, y, clip)
        want_trace.append(y.nnz)
    assert list(trace) == want_trace
    assert_csr_bitwise(out, y)


def _rise_and_fall(port, sk, n=520):
    """A network whose activation density rises (positive bias) then decays
    (negative bias), so the density-adaptive forward switches both ways."""
    m, seed = 2048, 23
    hW = [port.gen_layer_fixed(m, 16, port.layer_seed(seed, k), float("nan")) for k in range(6)]
    bs = [np.full(m, b, np.float32) for b in (0.01, -0.2, -0.6, -0.9, -0.9, -0.9)]
    hY = port.gen_input_binary(m, n, 20, seed)
    want, trace = hY, [hY.nnz]
    for k in range(6):
        want = port.layer_sparse(hW[k], bs[k], want, 0.0)
        trace.append(want.nnz)
    model = sk.DnnModel([dev_csr(sk, w) for w in hW], bs)
    return model, dev_csr(sk, hY), want, trace, m * n


@pytest.mark.parametrize("mode", ["sparse_only", "default", "all_dense", "dense_after_first",
                                  "pingpong"])
def test_density_switch_is_bitwise_neutral(sk, port, mode):
    model, y0, want, want_trace, full = _rise_and_fall(port, sk)
    dens = np.array(want_trace[1:-1], np.float64) / full
    ctx = sk.default_context()
    try:
        if mode == "sparse_only":
            ctx.set_density_switch(0.0, 0.0)
        elif mode == "all_dense":  # Y0 itself is above the threshold
            ctx.set_density_switch(1e-9, 0.0)
        elif mode == "dense_after_first":  # Y0 (1%) sparse, layer 0 output dense
            ctx.set_density_switch(want_trace[0] / full * 2, 0.0)
        elif mode == "pingpong":
            t = float(np.sqrt(dens.max() * max(dens.min(), 1e-9)))
            ctx.set_density_switch(t, t)
        ctx.set_timing(True)
        ctx.kernel_times_ms()
        out, trace = sk.relu_forward_sparse(model, y0)
        segments = len(ctx.kernel_times_ms())
    finally:
        ctx.set_timing(False)
        ctx.set_density_switch()
    assert list(trace) == want_trace
    assert_csr_bitwise(out, want)
    if mode in ("sparse_only", "all_dense"):
        assert segments == 1
    if mode == "dense_after_first":
        assert segments == 2
    if mode == "pingpong":
        assert segments >= 3  # sparse -> dense -> sparse


@pytest.mark.parametrize("mode", ["all_dense", "pingpong"])
def test_density_switch_wide_batch(sk, port, mode):
    """The same rise-and-fall network at 1300 samples (5 x 256 + 20): the dense
    segments run the staged wide engine (K1b) with its intermediate activations
    in panel-major scratch -- six layers in one launch (all_dense: the first
    reads and the last writes row-major buffers), and a density stop mid-way
    (pingpong: the stopping layer's panels are copied back to rows before the
    sparse engine takes over); bitwise against the oracle's sparse layers."""
    model, y0, want, want_trace, full = _rise_and_fall(port, sk, n=1300)
    dens = np.array(want_trace[1:-1], np.float64) / full
    ctx = sk.default_context()
    try:
        if mode == "all_dense":
            ctx.set_density_switch(1e-9, 0.0)
        else:
            t = float(np.sqrt(dens.max() * max(dens.min(), 1e-9)))
            ctx.set_density_switch(t, t)
        out, trace = sk.relu_forward_sparse(model, y0)
        paths = ctx.layer_paths(6)
    finally:
        ctx.set_density_switch()
    assert list(trace) == want_trace
    assert_csr_bitwise(out, want)
    assert paths.count("dense") >= (6 if mode == "all_dense" else 2), paths


def test_density_switch_not_taken_with_nonfinite_weights(sk, port):
    # w * 0 = NaN for w = inf: the dense engine would differ, so the pass stays sparse
    m, n = 1024, 300
    W = port.gen_layer_fixed(m, 16, 9, 0.25)
    W.values[::97] = np.inf
    b = np.full(m, 0.01, np.float32)  # positive bias densifies
    Y = port.gen_input_binary(m, n, 300, 9)
    model = sk.DnnModel([dev_csr(sk, W)] * 3, [b] * 3)
    ctx = sk.default_context()
    ctx.set_density_switch(1e-9, 0.0)
    try:
        out, _ = sk.relu_forward_sparse(model, dev_csr(sk, Y))
    finally:
        ctx.set_density_switch()
    want = Y
    for _ in range(3):
        want = port.layer_sparse(W, b, want, 0.0)
    g = host_csr(out)
    assert np.array_equal(g.row_ptr, want.row_ptr) and np.array_equal(g.col_idx, want.col_idx)
    assert same_bits_nan(g.values, want.values)


def test_density_switch_argument_checks(sk):
    from paper_1708_02937_b200.semikern import InvalidArgument
    ctx = sk.default_context()
    with pytest.raises(InvalidArgument):
        ctx.set_density_switch(0.01, 0.5)
    with pytest.raises(InvalidArgument):
        ctx.set_density_switch(0.01, -1.0)
    ctx.set_density_switch()


@pytest.mark.parametrize("ymax,dense_rows", [(1, True), (300, True), (20000, True),
                                             (1, False), (300, False), (20000, False)])
def test_exact_fixed_point_layer_matches_oracle(sk, port, ymax, dense_rows):
    # Layer 0 with exactly representable partial sums takes the order-free
    # fixed-point path; ymax sets the partial-sum range and with it the packing
    # (range 7 -> four 8-bit fields per word, ~15 -> two 16-bit, ~21 -> int32).
    # Signed weights, rows with positive bias (dense rows) mixed in.
    from oracle.oracle import Csr
    m, n, L, seed = 4096, 3000, 2, 41
    rng = np.random.default_rng(seed)
    hW = []
    for k in range(L):
        w = port.gen_layer_fixed(m, 32, port.layer_seed(seed, k), float("nan"))
        q = np.round(w.values * 8.0)
        q[q == 0] = 1.0
        hW.append(Csr(m, m, w.row_ptr, w.col_idx, (q / 16.0).astype(np.float32)))
    ent = 60000
    flat = rng.choice(m * n, size=ent, replace=False)
    r, c = (flat // n).astype(np.uint32), (flat % n).astype(np.uint32)
    v = rng.integers(1, ymax + 1, ent).astype(np.float32)
    Y = sk.csr_from_triples(m, n, (r, c, v))
    hY = host_csr(Y)
    # positive-bias rows take the float fallback inside the exact kernel
    b = np.where(np.arange(m) % 13 == 0, 0.25 if dense_rows else -1.5, -0.5).astype(np.float32)
    model = sk.DnnModel([dev_csr(sk, w) for w in hW], [b] * L)
    out, trace = sk.relu_forward_sparse(model, Y, sk.ForwardOptions(clip=0.0))
    assert sk.default_context().layer_paths(1) == ["exact"]
    y, want_trace = hY, [hY.nnz]
    for k in range(L):
        y = port.layer_sparse(hW[k], b, y, 0.0)
        want_trace.append(y.nnz)
    assert list(trace) == want_trace
    assert_csr_bitwise(out, y)


@pytest.mark.parametrize("target", [127, 128, 32767, 32768, (1 << 24) - 1, 1 << 24])
@pytest.mark.parametrize("yvals", [(1.0,), (0.5, 1.0)])
def test_exact_path_field_boundaries(sk, port, target, yvals):
    # The fixed-point packing is chosen from qb = max row sum |w| * max|y| * 2^-gran:
    # qb <= 127 -> 8-bit fields, <= 32767 -> 16-bit, < 2^24 -> int32, else the
    # ordered path.  Rows whose partial sums reach exactly +-qb (one sample has
    # every neuron active) sit on each boundary; any overflow of a field shows.
    from oracle.oracle import Csr
    m, n = 64, 8
    scale = 2.0 if len(yvals) > 1 else 1.0  # lowbit(Y) = -1 doubles qb
    t = int(target / scale)
    pw = [float(1 << e) for e in range(25) if (t - 1) >> e & 1] + [1.0]  # sums to t
    rows, cols, vals = [], [], []
    for i in range(m):
        if i < 3:
            sign = [1.0, -1.0, None][i]
            for k, w in enumerate(sorted(pw)):
                s = sign if sign is not None else (1.0 if k % 2 == 0 else -1.0)
                rows.append(i), cols.append(k), vals.append(s * w)
        else:
            for k in sorted({(i * 7) % m, (i * 13 + 5) % m, (i * 3 + 1) % m}):
                rows.append(i), cols.append(k), vals.append(1.0 if (i + k) % 3 else -2.0)
    W = sk.csr_from_triples(m, m, (np.array(rows, np.uint32), np.array(cols, np.uint32),
                                   np.array(vals, np.float32)))
    hW = host_csr(W)
    rng = np.random.default_rng(target % 1000)
    yr, yc, yv = [], [], []
    for j in range(n):
        act = np.arange(m) if j == 0 else np.flatnonzero(rng.random(m) < 0.4)
        for k in act:
            yr.append(k), yc.append(j), yv.append(yvals[-1] if j == 0 else rng.choice(yvals))
    Y = sk.csr_from_triples(m, n, (np.array(yr, np.uint32), np.array(yc, np.uint32),
                                   np.array(yv, np.float32)))
    hY = host_csr(Y)
    b = np.full(m, -0.5, np.float32)
    model = sk.DnnModel([dev_csr(sk, Csr(m, m, hW.row_ptr, hW.col_idx, hW.values))] * 2, [b] * 2)
    out, trace = sk.relu_forward_sparse(model, Y, sk.ForwardOptions(clip=0.0))
    y, want_trace = hY, [hY.nnz]
    for k in range(2):
        y = port.layer_sparse(hW, b, y, 0.0)
        want_trace.append(y.nnz)
    assert list(trace) == want_trace
    assert_csr_bitwise(out, y)
    # the boundary row really reaches its bound t on sample 0 (z = t + b)
    first = port.layer_sparse(hW, b, hY, 0.0)
    assert first.col_idx[first.row_ptr[0]] == 0
    assert first.values[first.row_ptr[0]] == np.float32(t) + np.float32(-0.5)


def _thin_model(port, m, L, deg, seed, rng, special=False):
    from oracle.oracle import Csr
    hW = []
    for k in range(L):
        w = port.gen_layer_fixed(m, deg, port.layer_seed(seed, k), float("nan"))
        v = rng.uniform(-1.0, 1.0, w.values.size).astype(np.float32)  # not exact
        if special and k == 0:
            v[::97] = np.inf
        hW.append(Csr(m, m, w.row_ptr, w.col_idx, v))
    return hW


@pytest.mark.parametrize("m,n,L,entries", [(4096, 3000, 4, 5000), (4096, 3000, 3, 7),
                                           (70000, 70000, 2, 300), (70000, 70000, 2, 40)])
def test_esc_thin_layers_bitwise(sk, port, m, n, L, entries):
    # Thin inputs with every bias <= 0 take expand-sort-compress (stable sort of
    # (i, j) keys, ascending-k run fold); 70000 x 70000 needs 64-bit keys.
    rng = np.random.default_rng(m + entries)
    hW = _thin_model(port, m, L, 8, 17, rng, special=(entries == 5000))
    flat = rng.choice(m * n, size=entries, replace=False)
    r, c = (flat // n).astype(np.uint32), (flat % n).astype(np.uint32)
    v = rng.uniform(0.2, 3.0, entries).astype(np.float32)
    v[::11] = -0.0
    Y = sk.csr_from_triples(m, n, (r, c, v))
    hY = host_csr(Y)
    b = (-rng.uniform(0.0, 0.3, m)).astype(np.float32)
    b[::5] = 0.0
    model = sk.DnnModel([dev_csr(sk, w) for w in hW], [b] * L)
    out, trace = sk.relu_forward_sparse(model, Y, sk.ForwardOptions(clip=2.5))
    paths = sk.default_context().layer_paths(L)
    y, want_trace = hY, [hY.nnz]
    for k in range(L):
        y = port.layer_sparse(hW[k], b, y, 2.5)
        want_trace.append(y.nnz)
    assert list(trace) == want_trace
    assert_csr_bitwise(out, y)
    assert paths[0] == "esc", paths


@pytest.mark.parametrize("case", ["crowded_sample", "survivor_regrow"])
def test_sample_major_esc_fallback_and_regrow(sk, port, case):
    # The sample-major ESC sorts each sample's products in one warp's shared
    # buffer (512 products).  "crowded_sample": one sample holds 640 products,
    # so the layer must fall back to the global sort; "survivor_regrow": more
    # survivors than the first output allocation (65536), so the kernel reruns
    # with the exact count.  Both bitwise against the oracle.
    rng = np.random.default_rng(7 if case == "crowded_sample" else 8)
    m, n, L = 4096, 3000, 2
    hW = _thin_model(port, m, L, 8, 17, rng, special=False)
    entries = 2000 if case == "crowded_sample" else 24000
    flat = rng.choice(m * n, size=entries, replace=False)
    r, c = (flat // n).astype(np.uint32), (flat % n).astype(np.uint32)
    if case == "crowded_sample":
        extra = rng.choice(m, size=80, replace=False).astype(np.uint32)
        keep = c != 17
        r = np.concatenate([r[keep], extra])
        c = np.concatenate([c[keep], np.full(80, 17, np.uint32)])
    v = rng.uniform(0.2, 3.0, r.size).astype(np.float32)
    Y = sk.csr_from_triples(m, n, (r, c, v))
    hY = host_csr(Y)
    b = (-rng.uniform(0.0, 0.3, m)).astype(np.float32)
    if case == "survivor_regrow":
        b[:] = 0.0
    model = sk.DnnModel([dev_csr(sk, w) for w in hW], [b] * L)
    out, trace = sk.relu_forward_sparse(model, Y, sk.ForwardOptions(clip=32.0))
    y, want_trace = hY, [hY.nnz]
    for k in range(L):
        y = port.layer_sparse(hW[k], b, y, 32.0)
        want_trace.append(y.nnz)
    assert list(trace) == want_trace
    assert_csr_bitwise(out, y)
    if case == "survivor_regrow":
        assert want_trace[1] > 65536, want_trace


def test_empty_input_runs_and_positive_bias_after(sk, port):
    # an empty input stays empty through the layers with every bias <= 0 (no
    # work at all), then a layer with positive biases makes dense rows
    from oracle.oracle import Csr
    m, n, L = 2048, 500, 5
    rng = np.random.default_rng(3)
    hW = _thin_model(port, m, L, 8, 5, rng)
    bs = [np.full(m, -0.1, np.float32)] * 3 + [np.where(np.arange(m) % 7 == 0, 0.5, -0.2)
                                             .astype(np.float32)] + [np.full(m, -0.1, np.float32)]
    Y = sk.csr_from_triples(m, n, (np.zeros(0, np.uint32), np.zeros(0, np.uint32),
                                   np.zeros(0, np.float32)))
    model = sk.DnnModel([dev_csr(sk, w) for w in hW], bs)
    out, trace = sk.relu_forward_sparse(model, Y, sk.ForwardOptions(clip=0.0))
    paths = sk.default_context().layer_paths(L)
    y, want_trace = Csr(m, n, np.zeros(m + 1, np.uint32), np.zeros(0, np.uint32),
                        np.zeros(0, np.float32)), [0]
    for k in range(L):
        y = port.layer_sparse(hW[k], bs[k], y, 0.0)
        want_trace.append(y.nnz)
    assert list(trace) == want_trace and want_trace[4] > 0
    assert_csr_bitwise(out, y)
    assert paths[:3] == ["empty"] * 3 and paths[3] != "empty", paths


@pytest.mark.parametrize("entries,bias", [(1, -0.01), (40, -0.01), (40, -0.2), (900, 0.0)])
def test_sparse_forward_frontier_layers(sk, port, entries, bias):
    # near-empty inputs take the frontier path (only rows with an in-edge from an
    # active input row are processed); it must be invisible in the results
    m, n, L, seed = 8192, 3000, 5, 31
    rng = np.random.default_rng(seed)
    flat = rng.choice(m * n, size=entries, replace=False)
    r, c = (flat // n).astype(np.uint32), (flat % n).astype(np.uint32)
    v = rng.uniform(0.5, 2.0, entries).astype(np.float32)
    hY = port.csr_from_triples(m, n, r, c, v) if hasattr(port, "csr_from_triples") else None
    Y = sk.csr_from_triples(m, n, (r, c, v))
    if hY is None:
        hY = host_csr(Y)
    hW = [port.gen_layer_fixed(m, 32, port.layer_seed(seed, k), float("nan")) for k in range(L)]
    b = np.full(m, bias, np.float32)
    model = sk.DnnModel([dev_csr(sk, w) for w in hW], [b] * L)
    out, trace = sk.relu_forward_sparse(model, Y)
    y, want_trace = hY, [hY.nnz]
    for k in range(L):
        y = port.layer_sparse(hW[k], b, y, 0.0)
        want_trace.append(y.nnz)
    assert list(trace) == want_trace
    assert_csr_bitwise(out, y)


def test_sparse_forward_empty_and_tiny_inputs(sk, port):
    m = 512
    W = sk.gen_layer_fixed(m, 8, 3, 0.5)
    model = sk.DnnModel([W, W], [np.full(m, -0.1, np.float32)] * 2)
    empty = sk.CsrMatrix(m, 10, [0] * (m + 1), [], [])
    out, trace = sk.relu_forward_sparse(model, empty)
    assert out.nnz() == 0 and list(trace) == [0, 0, 0]
    one = sk.csr_from_triples(m, 1, [(5, 0, 3.0)])
    out, _ = sk.relu_forward_sparse(model, one)
    hW = host_csr(W)
    y = host_csr(one)
    for _ in range(2):
        y = port.layer_sparse(hW, np.full(m, -0.1, np.float32), y, 0.0)
    assert_csr_bitwise(out, y)


def test_sparse_route_equals_dense_route(sk):
    # the same network through K1 (dense Y) and K3 (sparse Y) agrees bitwise
    m, n = 2048, 300
    Ws = [sk.gen_layer_fixed(m, 32, sk.layer_seed(5, k)) for k in range(3)]
    model = sk.DnnModel(Ws, [np.full(m, -0.05, np.float32)] * 3)
    y0 = sk.gen_input_dense(m, n, 5)
    dense = sk.relu_forward(model, y0).numpy()
    sparse, _ = sk.relu_forward_sparse(model, sk.from_dense(y0))
    assert np.array_equal(bits(sk.to_dense(sparse).numpy()), bits(dense))


# ---- multi-GPU building blocks on one GPU ----------------------------------------------

@pytest.mark.parametrize("kind", ["mixed_bias", "nonpos_bias", "random_weights"])
def test_sparse_layer_on_a_row_block_matches_oracle(sk, port, kind):
    # a row block of W_ref (column sharding): binary Y x 1/16 weights take the
    # order-free kernel (with dense-sweep rows for positive biases, or the coarse
    # window table when every bias <= 0); random weights the windowed SpGEMM
    from oracle.oracle import Csr
    m, n = 4096, 700
    W = port.gen_layer_fixed(m, 32, 5, float("nan") if kind == "random_weights" else 1.0 / 16)
    Y = port.gen_input_binary(m, n, 300, 5)
    r0, r1 = 1000, 2500
    blk = Csr(r1 - r0, m, (W.row_ptr[r0:r1 + 1] - W.row_ptr[r0]).astype(np.uint32),
              W.col_idx[W.row_ptr[r0]:W.row_ptr[r1]], W.values[W.row_ptr[r0]:W.row_ptr[r1]])
    b = np.where(np.arange(r1 - r0) % 7 == 0, 0.01 if kind == "mixed_bias" else -0.2,
                 -0.05).astype(np.float32)
    got = sk.sparse_layer(dev_csr(sk, blk), b, dev_csr(sk, Y), 32.0)
    assert_csr_bitwise(got, port.layer_sparse(blk, b, Y, 32.0))


def test_csr_publish_to_several_destinations(sk, port):
    # the peer-exchange kernel: one launch writes a block into every destination
    # at its entry offset, row pointers shifted (here: two buffers on this GPU)
    import torch
    from paper_1708_02937_b200 import semikern as skm
    m, n = 300, 90
    blk_h = port.gen_input_binary(120, n, 7, 3)  # a 120-row block
    blk = dev_csr(sk, blk_h)
    row_off, nnz_off, total = 100, 5000, 5000 + blk_h.nnz
    dev = torch.device("cuda", 0)
    bufs = [(torch.full((m + 1,), 7, dtype=torch.int32, device=dev),
             torch.full((total,), 9, dtype=torch.int32, device=dev),
             torch.full((total,), -1.0, dtype=torch.float32, device=dev)) for _ in range(2)]
    for last in (False, True):
        skm.csr_publish(blk, [b[0].data_ptr() for b in bufs], [b[1].data_ptr() for b in bufs],
                        [b[2].data_ptr() for b in bufs], row_off, nnz_off, last)
        torch.cuda.synchronize()
        for rp, ci, v in bufs:
            rp, ci, v = rp.cpu().numpy(), ci.cpu().numpy(), v.cpu().numpy()
            assert np.array_equal(rp[row_off:row_off + 120],
                                  blk_h.row_ptr[:120].astype(np.int64) + nnz_off)
            assert rp[row_off + 120] == (total if last else 7)
            assert rp[row_off - 1] == 7
            assert np.array_equal(ci[nnz_off:], blk_h.col_idx.astype(np.int32))
            assert np.array_equal(bits(v[nnz_off:]), bits(blk_h.values))
            assert np.all(ci[:nnz_off] == 9)


@pytest.mark.parametrize("kind", ["exact", "engine"])
def test_staged_layer_publishes_from_its_gather(sk, port, kind):
    """sk_sparse_layer_stage + sk_staged_publish: a row block's layer written by
    its own gather kernel into several destinations (entries at nnz_off, row
    pointers shifted) equals sk_sparse_layer_dev's block, bit for bit.  "exact":
    the order-free path (the fused gather); "engine": a layer that is not
    provably exact (finished first, published from the block)."""
    import torch
    from paper_1708_02937_b200 import semikern as skm
    m, n, rows, r0 = 4096, 1500, 700, 1000
    val = 1.0 / 16 if kind == "exact" else float("nan")
    W = port.gen_layer_fixed(m, 32, port.layer_seed(5, 0), val)
    blk_h = hcsr(rows, m, (W.row_ptr[r0:r0 + rows + 1] - W.row_ptr[r0]).astype(np.uint32),
                 W.col_idx[W.row_ptr[r0]:W.row_ptr[r0 + rows]],
                 W.values[W.row_ptr[r0]:W.row_ptr[r0 + rows]])
    blk = dev_csr(sk, blk_h)
    b = np.full(rows, -0.2, np.float32)
    Y = dev_csr(sk, port.gen_input_binary(m, n, 300, 5))
    dev = torch.device("cuda", 0)
    db = torch.as_tensor(b, device=dev)
    torch.cuda.synchronize()
    dense_rows, negmin = skm.bias_summaries(b)
    want = host_csr(skm.sparse_layer_dev(blk, db.data_ptr(), dense_rows, negmin, Y, 32.0))
    assert want.nnz > 0
    st = skm.sparse_layer_stage(blk, db.data_ptr(), dense_rows, negmin, Y, 32.0)
    assert st.nnz == want.nnz
    nnz_off, row_off = 3000, r0
    total = nnz_off + want.nnz
    bufs = [(torch.full((m + 1,), 7, dtype=torch.int32, device=dev),
             torch.full((total,), 9, dtype=torch.int32, device=dev),
             torch.full((total,), -1.0, dtype=torch.float32, device=dev)) for _ in range(3)]
    st.publish([x[0].data_ptr() for x in bufs], [x[1].data_ptr() for x in bufs],
               [x[2].data_ptr() for x in bufs], row_off, nnz_off, True)
    sk.default_context().synchronize()
    for rp, ci, v in bufs:
        rp, ci, v = rp.cpu().numpy(), ci.cpu().numpy(), v.cpu().numpy()
        assert np.array_equal(rp[row_off:row_off + rows + 1],
                              want.row_ptr.astype(np.int64) + nnz_off)
        assert rp[row_off - 1] == 7 and rp[row_off + rows + 1] == 7
        assert np.array_equal(ci[nnz_off:], want.col_idx.astype(np.int32))
        assert np.array_equal(bits(v[nnz_off:]), bits(want.values))
        assert np.all(ci[:nnz_off] == 9)


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
def test_column_sharded_forward_single_rank_nccl(sk, port, exchange):
    import socket
    import torch
    import torch.distributed as dist
    from paper_1708_02937_b200.shard import relu_forward_sparse_colsharded
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
        s.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port_no}", rank=0,
                                world_size=1)
    m, n, L = 4096, 500, 6
    hW = [port.gen_layer_fixed(m, 32, port.layer_seed(8, k), 1.0 / 16) for k in range(L)]
    hY = port.gen_input_binary(m, n, 400, 8)
    # live layers, then a bias that empties the activations (the rest is skipped)
    bs = [np.full(m, x, np.float32) for x in (-0.05, -0.05, -0.05, -9.0, -0.05, -0.05)]
    try:
        y, trace = relu_forward_sparse_colsharded([dev_csr(sk, w) for w in hW], bs,
                                                  dev_csr(sk, hY), clip=32.0,
                                                  device=torch.device("cuda", 0),
                                                  exchange=exchange, exchange_single=True)
        want, want_trace = hY, [hY.nnz]
        for w, b in zip(hW, bs):
            want = port.layer_sparse(w, b, want, 32.0)
            want_trace.append(want.nnz)
        assert_csr_bitwise(y, want)
        assert list(trace) == want_trace
        assert want_trace[1] > 0 and want_trace[4] == 0
    finally:
        dist.destroy_process_group()


# ---- the dense comparator leg on tcgen05 (K4) ----------------------------------------

def scaled_ok(got, want, scale):
    """approx_equal_scaled (semiring.hpp:50-55): |x-y| <= max(kAbsTol, kRelTol*scale)."""
    return np.abs(got.astype(np.float64) - want.astype(np.float64)) <= np.maximum(1e-6, 1e-5 * scale)


@pytest.mark.parametrize("M,K,N", [(128, 32, 128), (130, 33, 7), (1000, 600, 257),
                                   (4096, 4096, 256), (1, 5, 1)])
def test_dense_mxm_baseline_tcgen05_within_scaled_tolerance(sk, ref, M, K, N):
    rng = np.random.default_rng(M + K + N)
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    b = rng.uniform(0, 1, (K, N)).astype(np.float32)
    a[rng.random(a.shape) < 0.3] = 0.0
    got = sk.dense_mxm_baseline(sk.DenseMatrix.from_numpy(a), sk.DenseMatrix.from_numpy(b)).numpy()
    exact = a.astype(np.float64) @ b.astype(np.float64)
    want = ref.dense_mxm_baseline(a, b, workers=8) if M * K * N < 2e9 else exact.astype(np.float32)
    scale = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64)
    assert scaled_ok(got, want, scale).all()
    # an fp32-class result (3xTF32): a single-pass tf32 product carries ~2^-11
    # relative error per term (median |err|/scale ~1e-4); 3xTF32 is ~1e-7
    rel = np.abs(got - exact) / np.maximum(scale, 1e-30)
    assert np.median(rel) < 1e-6 and rel.max() < 1e-5
    if M * K * N <= 1 << 22:
        # below the tensor-core threshold the comparator runs the reference's
        # own order (ascending k, no FMA): bitwise
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("m,n,L", [(25, 8, 3), (64, 8, 4), (4, 1, 1)])
def test_small_dense_forward_bitwise_and_within_reference_acceptance(sk, ref, port, m, n, L):
    # acceptance.cpp criterion 1 (proj/tests/acceptance.cpp:60-90) compares the
    # sparse pipeline with dense_relu_forward to 1e-5 relative PER ELEMENT; at
    # these sizes both legs fold in the reference's order, so they agree bitwise
    # with each other and with the reference.
    rng = np.random.default_rng(m * 131 + n)
    ws, bs = [], []
    for _ in range(L):
        w = rng.uniform(-1, 3, (m, m)).astype(np.float32)
        w[rng.random(w.shape) < 0.75] = 0.0
        ws.append(w)
        bs.append(rng.uniform(0, 1, m).astype(np.float32))
    y0 = rng.uniform(0, 1, (m, n)).astype(np.float32)
    model = sk.DnnModel([sk.Matrix(sk.DenseMatrix.from_numpy(w)) for w in ws], bs)
    dense = sk.dense_relu_forward(model, sk.DenseMatrix.from_numpy(y0)).numpy()
    sparse = sk.relu_forward(model, sk.DenseMatrix.from_numpy(y0)).numpy()
    want = y0
    for w, b in zip(ws, bs):
        want = ref.dense_layer_step(w, b, want, workers=1)
    assert np.array_equal(dense.view(np.uint32), want.view(np.uint32))
    assert np.array_equal(sparse.view(np.uint32), want.view(np.uint32))


def test_dense_layer_step_cfg2_density_matches_reference(sk, ref, port):
    m, n = 4096, 256
    W = port.gen_layer_density(m, 0.1, port.layer_seed(7, 0))
    wd = W.to_dense()
    y = port.gen_input_dense(m, n, 7)
    b = np.full(m, -0.05, np.float32)
    got = sk.dense_layer_step(sk.DenseMatrix.from_numpy(wd), b, sk.DenseMatrix.from_numpy(y)).numpy()
    want = ref.dense_layer_step(wd, b, y, workers=8)
    scale = np.abs(wd).astype(np.float64) @ np.abs(y).astype(np.float64)
    assert scaled_ok(got, want, scale).all()
    # ReLU pattern equal except where the pre-activation is within tolerance of 0
    pre = (wd.astype(np.float64) @ y.astype(np.float64)) + b[:, None]
    near = np.abs(pre) <= 1e-5 * scale + 1e-6
    assert ((got != 0) == (want != 0))[~near].all()


def test_dense_leg_packed_weights_cache(sk, ref, port):
    """K4 keeps the split/packed weights on the handle: repeated calls reuse it,
    an in-place write invalidates it, and dense_relu_forward's per-model copy
    gives the same result on every call (tolerance of approx_equal_scaled)."""
    m, n = 512, 128
    W = port.gen_layer_density(m, 0.1, port.layer_seed(11, 0))
    wd = W.to_dense()
    y = port.gen_input_dense(m, n, 11)
    b = np.full(m, -0.05, np.float32)
    Wd = sk.DenseMatrix.from_numpy(wd)
    yd = sk.DenseMatrix.from_numpy(y)

    def check(got, wmat):
        want = ref.dense_layer_step(wmat, b, y, workers=8)
        scale = np.abs(wmat).astype(np.float64) @ np.abs(y).astype(np.float64)
        assert (np.abs(got.astype(np.float64) - want) <= np.maximum(1e-6, 1e-5 * scale)).all()

    first = sk.dense_layer_step(Wd, b, yd).numpy()
    check(first, wd)
    assert np.array_equal(sk.dense_layer_step(Wd, b, yd).numpy(), first)  # cached pack
    wd2 = (wd * -0.5).astype(np.float32)
    Wd.write(wd2)  # invalidates the cached pack
    check(sk.dense_layer_step(Wd, b, yd).numpy(), wd2)
    model = sk.DnnModel([dev_csr(sk, W)] * 2, [b, b])
    r1 = sk.dense_relu_forward(model, yd).numpy()
    r2 = sk.dense_relu_forward(model, yd).numpy()
    assert np.array_equal(r1, r2)


def _in_degree_weights(m, maxdeg, seed):
    """W_ref with in-degrees 0..maxdeg (row i: (37 i) mod (maxdeg + 1) in-edges at
    distinct random inputs), every value 1/16: a constant increment."""
    from oracle.oracle import Csr
    rng = np.random.default_rng(seed)
    rp, ci = [0], []
    for i in range(m):
        d = (37 * i) % (maxdeg + 1)
        ci.extend(sorted(rng.choice(m, size=d, replace=False).tolist()))
        rp.append(len(ci))
    return Csr(m, m, np.array(rp, np.uint32), np.array(ci, np.uint32),
               np.full(len(ci), 1.0 / 16, np.float32))


# (m, samples, active inputs per sample, bias, clip, max in-degree, counter width)
STREAM_CASES = [
    (8192, 5000, 120, -0.3, 32.0, 64, 0),     # 4-bit counters, 8192-sample passes + a partial one
    (8192, 5000, 120, -0.3, 32.0, 64, 8),     # the same with 8-bit counters
    (4096, 700, 200, -0.45, 32.0, 40, 0),     # a batch narrower than one pass (t' = 7: 4-bit edge)
    (4096, 3000, 400, -0.5, 0.0, 96, 0),      # t' = 8: 8-bit counters; three in-edge slots
    (16384, 3000, 3000, -0.1, 2.0, 70, 0),    # 4-bit counters wrap (counts >= 10): the rerun;
                                              # clip 2 is active
    (2048, 20000, 4, -0.05, 32.0, 33, 0),     # 16384-sample passes, sparse passes (touched clear)
]


@pytest.mark.parametrize("layout", [2, 1, 3])
@pytest.mark.parametrize("case", STREAM_CASES)
def test_stream_kernel_regimes(sk, port, case, layout):
    """K7 (k_exact_stream, the order-free row stream) against the oracle's sparse
    layer (matrix.cpp:452-521 + dnn.cpp:86-103 restated) in the regimes its
    host logic chooses between: 4- vs 8-bit counters, a 4-bit counter wrapping
    (the layer is rerun with 8-bit ones), in-degrees up to 96 (one to three
    in-edge slots per lane, rows with none), a batch narrower than one pass,
    passes that end past the batch, the touched-word clear of sparse passes --
    each with Y read in place (layout 2), through the padded copy (1) and through
    the padded copy with bank-ordered pass slices (3: <= 8 passes, else 1)."""
    m, n, kY, bias, clip, maxdeg, fields = case
    hW = _in_degree_weights(m, maxdeg, m + n)
    hY = port.gen_input_binary(m, n, kY, 7)
    b = np.full(m, bias, np.float32)
    want = port.layer_sparse(hW, b, hY, clip)
    ctx = sk.default_context()
    # the wrapping case: 2048-sample passes (the widest that take 4-bit counters
    # is chosen narrower for this density)
    old = ctx.set_tuning(exact_kernel=5, exact_fields=fields, exact_layout=layout,
                         exact_group=2 if bias == -0.1 else 0)
    ctx.set_density_switch(0.0, 0.0)  # keep the activations sparse
    try:
        n0 = ctx.last_exact()["wraps"]
        model = sk.DnnModel([dev_csr(sk, hW)], [b])
        out, trace = sk.relu_forward_sparse(model, dev_csr(sk, hY), sk.ForwardOptions(clip=clip))
        info = ctx.last_exact()
    finally:
        ctx.set_tuning(**old)
        ctx.set_density_switch()
    assert ctx.layer_paths(1) == ["exact"] and info["kernel"] == "stream", info
    assert info["layout"] in {2: ("direct",), 1: ("padded",), 3: ("banked", "padded")}[layout], info
    assert list(trace) == [hY.nnz, want.nnz]
    assert_csr_bitwise(out, want)
    if fields == 8 or bias == -0.5:
        assert info["fields"] == 4, info  # 8-bit counters: four per word
    if bias == -0.1:
        assert want.nnz > 100000 and info["wraps"] > n0, info  # the 4-bit pass wrapped


@pytest.mark.parametrize("n,group", [(20000, 0), (40000, 0), (9000, 1), (3000, 0)])
def test_stream_in_place_row_boundaries(sk, port, n, group):
    """K7 reading Y in place: a 16-byte unit at a row's start or end also holds
    entries of the neighbouring rows, and those must not count (the slice's side
    unit replaces it -- the pass table's head / tail flags).  Rows of 0..9
    entries at random samples (most rows start and end inside a unit, many
    consist of one unit, neighbours' samples fall into the same pass), 2 / 3 /
    9 / 1 passes; bitwise against the oracle's sparse layer and against the
    padded copy."""
    from oracle.oracle import Csr
    m = 3001
    rng = np.random.default_rng(n + group)
    lens = rng.integers(0, 10, size=m)
    lens[::97] = 0
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
    ci = np.concatenate([np.sort(rng.choice(n, size=int(c), replace=False)) for c in lens]
                        ).astype(np.uint32)
    hY = Csr(m, n, rp, ci, np.ones(len(ci), np.float32))
    hW = _in_degree_weights(m, 64, 11)
    b = np.full(m, -0.05, np.float32)
    want = port.layer_sparse(hW, b, hY, 32.0)
    ctx = sk.default_context()
    outs = []
    for layout in (2, 1):
        old = ctx.set_tuning(exact_kernel=5, exact_layout=layout, esc=-1,
                             exact_group=group)
        ctx.set_density_switch(0.0, 0.0)
        try:
            model = sk.DnnModel([dev_csr(sk, hW)], [b])
            out, trace = sk.relu_forward_sparse(model, dev_csr(sk, hY),
                                                sk.ForwardOptions(clip=32.0))
            info = ctx.last_exact()
        finally:
            ctx.set_tuning(**old)
            ctx.set_density_switch()
        assert info["kernel"] == "stream", info
        assert info["layout"] == {2: "direct", 1: "padded"}[layout], info
        assert list(trace) == [hY.nnz, want.nnz]
        assert_csr_bitwise(out, want)
        outs.append(out)
    assert want.nnz > 1000


def test_pattern16_upload_matches_pattern(sk, port):
    """sk_csr_from_pattern16_async (16-bit column indices widened on the device,
    the bench's end-to-end upload) gives the same CSR as the 32-bit upload:
    odd nnz (the widening kernel's tail), the largest column 65535, empty rows."""
    import torch
    m, n = 3000, 65536
    Y = port.gen_input_binary(m, n, 7, 3)
    rp = Y.row_ptr.copy()
    ci = Y.col_idx.copy()
    ci[rp[5]:rp[6]] = np.arange(65536 - (rp[6] - rp[5]), 65536, dtype=np.uint32)  # top columns
    rp2 = np.concatenate([rp[:11], rp[11:] - (rp[11] - rp[10])]).astype(np.uint32)
    ci2 = np.concatenate([ci[:rp[10]], ci[rp[11]:]]).astype(np.uint32)   # row 10 emptied
    ci2 = ci2[:-1]                                                        # odd nnz
    rp2[-1] -= 1
    rp2 = np.minimum(rp2, rp2[-1])
    s = torch.cuda.Stream()
    a = sk.CsrMatrix.from_pattern16_async(m, n, rp2, ci2.astype(np.uint16), 1.0,
                                          stream=s.cuda_stream)
    b = sk.CsrMatrix.from_pattern(m, n, rp2, ci2, 1.0, validate=True)
    for x, y in zip(a.extract(), b.extract()):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    with pytest.raises(Exception):
        sk.CsrMatrix.from_pattern16_async(m, n + 1, rp2, ci2.astype(np.uint16), 1.0,
                                          stream=s.cuda_stream)


# (m, samples, active inputs per sample, bias, max in-degree, 4-bit wrap expected)
CHAIN_CASES = [
    (8192, 5000, 120, -0.45, 64, False),   # layer 1 leaves a few entries: the tiny ESC takes layer 2
    (8192, 5000, 120, -0.2, 64, False),    # layer 1 leaves thousands: the tiny ESC declines
    (16384, 3000, 3000, -0.1, 70, True),   # a 4-bit counter wraps: the synchronous fallback
]


@pytest.mark.parametrize("case", CHAIN_CASES)
def test_exact_layer_chained_with_tiny_esc(sk, port, case):
    """The exact layer and the tiny ESC of the next layer issued with one host
    round trip (the layer-1 count stays on the device): both outcomes of the
    tiny kernel (it takes the layer / declines and the host goes on its usual
    way) and the fallback when a 4-bit counter wraps -- three layers against
    the oracle's sparse layer, layer by layer."""
    m, n, kY, bias, maxdeg, wraps = case
    L = 3
    hW = [_in_degree_weights(m, maxdeg, m + n + 7 * k) for k in range(L)]
    hY = port.gen_input_binary(m, n, kY, 11)
    b = np.full(m, bias, np.float32)
    y, want_trace = hY, [hY.nnz]
    for k in range(L):
        y = port.layer_sparse(hW[k], b, y, 32.0)
        want_trace.append(y.nnz)
    ctx = sk.default_context()
    old = ctx.set_tuning(exact_kernel=5, exact_group=2 if wraps else 0)
    ctx.set_density_switch(0.0, 0.0)
    try:
        w0 = ctx.last_exact()["wraps"]
        model = sk.DnnModel([dev_csr(sk, w) for w in hW], [b] * L)
        out, trace = sk.relu_forward_sparse(model, dev_csr(sk, hY), sk.ForwardOptions(clip=32.0))
        paths = ctx.layer_paths(L)
        info = ctx.last_exact()
    finally:
        ctx.set_tuning(**old)
        ctx.set_density_switch()
    assert list(trace) == want_trace
    assert_csr_bitwise(out, y)
    assert paths[0] == "exact", paths
    if want_trace[1] <= 512 and want_trace[1] * maxdeg <= 2048:
        assert paths[1] == "esc", (paths, want_trace)
    if wraps:
        assert info["wraps"] > w0, info
