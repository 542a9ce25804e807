"""GPU parity at the bench's own scale: the inputs `bench.py` times.

* cfg3 / cfg4 / cfg5 (BASELINE configs[2..4]) at 60000 samples with the
  bench's seeds: the whole L-layer forward (nnz trace, output CSR, category
  set) bitwise against the C restatement of the reference's sparse layer
  (oracle/sk_oracle.c, pinned to proj/src/matrix.cpp:452-521 + dnn.cpp:86-121),
  and the kernel the bench runs asserted (sk_ctx_last_exact): K7 (the row
  stream, k_exact_stream.cu).
* Layer 1 of each at full scale with EVERY exact-layer variant forced through
  the per-context tuning (K7 at 1 / 2 / 4 / 8 / 16 windows per pass x 4-bit
  (where the threshold allows) / 8-bit counters;
  generic / specialised kernel x 64 / 192 records x
  4..64 windows per item, i.e. 1..16 accumulator passes per item, plus the
  other window sizes), at the bench bias and at a less negative bias whose
  output holds millions of entries -- so the multi-pass items, the candidate
  marking and the emit are checked where they do real work.
* The windowed engine and its frontier path at full scale (exact / ESC off).
* BASELINE configs[1] at its full size (W 4096 x 4096, Y 4096 x 1024) for all
  five densities, sparse leg (K1, including the light-row kU=4 variant taken at
  d <= 1e-3) bitwise against the reference's layer_step, dense leg (K4) within
  the reference's approx_equal_scaled.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 42       # bench.py SEED
B = 60000       # bench batch per GPU
# name: (neurons, layers, active inputs per sample, bench bias, a "live" bias)
CFG = {
    "cfg3": (16384, 120, 246, -0.3, -0.2),
    "cfg4": (65536, 480, 262, -0.35, -0.1),
    "cfg5": (262144, 120, 262, -0.45, -0.1),
}
# the records / kernel the bench takes on layer 1 (profiles/r01 launch lists)
BENCH_KERNEL = {"cfg3": (0, "stream"), "cfg4": (0, "stream"), "cfg5": (0, "stream")}


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_same(got, want, what):
    rp, ci, v = got.extract()
    assert got.rows() == want.rows and got.cols() == want.cols, what
    assert np.array_equal(rp, want.row_ptr), f"{what}: row pointers differ"
    assert np.array_equal(ci, want.col_idx), f"{what}: columns differ"
    assert np.array_equal(bits(v), bits(want.values)), f"{what}: values differ"


_host = {}


def host_inputs(port, cfg):
    """Layer-0/1 weights and Y0 on the host (the oracle's generators; the device
    generators are bitwise equal to them, test_device_generators_match_oracle)."""
    if cfg not in _host:
        m, L, kY, _, _ = CFG[cfg]
        W = [port.gen_layer_fixed(m, 32, port.layer_seed(SEED, k), 1.0 / 16) for k in range(2)]
        Y0 = port.gen_input_binary(m, B, kY, SEED)
        _host[cfg] = (W, Y0)
    return _host[cfg]


_want1 = {}


def oracle_layer1(port, cfg, bias):
    key = (cfg, bias)
    if key not in _want1:
        (W, Y0), m = host_inputs(port, cfg), CFG[cfg][0]
        _want1[key] = port.layer_sparse(W[0], np.full(m, bias, np.float32), Y0, 32.0)
    return _want1[key]


@pytest.fixture
def ctx(sk):
    c = sk.default_context()
    old = c.set_tuning()
    yield c
    c.set_tuning(**old)
    c.set_density_switch()


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4", "cfg5"])
def test_bench_forward_full_scale(sk, port, ctx, cfg):
    """The bench's workload exactly (device-generated weights and inputs, all L
    layers, clip 32) against the oracle run layer by layer; layers after the
    activations die are empty in both (every bias <= 0)."""
    m, L, kY, bias, _ = CFG[cfg]
    Ws = [sk.gen_layer_fixed(m, 32, sk.layer_seed(SEED, k), 1.0 / 16) for k in range(L)]
    b = np.full(m, bias, np.float32)
    model = sk.DnnModel(Ws, [b] * L)
    del Ws
    Y0 = sk.gen_input_binary(m, B, kY, SEED)
    n0 = ctx.last_exact()["launches"]
    out, trace = sk.relu_forward_sparse(model, Y0, sk.ForwardOptions(clip=32.0))
    info = ctx.last_exact()
    paths = ctx.layer_paths(L)

    (hW, hY0) = host_inputs(port, cfg)
    y, want = hY0, [hY0.nnz]
    for k in range(L):
        if y.nnz == 0:  # empty input, bias <= 0: every later layer is empty
            want += [0] * (L - k)
            break
        w = hW[k] if k < 2 else port.gen_layer_fixed(m, 32, port.layer_seed(SEED, k), 1.0 / 16)
        y = port.layer_sparse(w, b, y, 32.0)
        want.append(y.nnz)
    assert [int(x) for x in trace] == want
    assert_same(out, y, f"{cfg} Y_L")
    assert np.array_equal(sk.categories(out), port.categories_sparse(y))
    # the kernel the bench times ran on layer 1
    assert paths[0] == "exact" and info["launches"] == n0 + 1
    assert (info["records"], info["kernel"]) == BENCH_KERNEL[cfg], info
    del model


def _layer1_model(sk, cfg, bias):
    m = CFG[cfg][0]
    W0 = sk.gen_layer_fixed(m, 32, sk.layer_seed(SEED, 0), 1.0 / 16)
    return sk.DnnModel([W0], [np.full(m, bias, np.float32)])


@pytest.mark.parametrize("cfg,which", [(c, w) for c in ("cfg3", "cfg4", "cfg5")
                                       for w in ("bench", "live")])
def test_exact_layer_every_variant_full_scale(sk, port, ctx, cfg, which):
    m, _, kY, bench_bias, live_bias = CFG[cfg]
    bias = bench_bias if which == "bench" else live_bias
    want = oracle_layer1(port, cfg, bias)
    if which == "live":
        assert want.nnz > 10000  # the emit does real work
    model = _layer1_model(sk, cfg, bias)
    Y0 = sk.gen_input_binary(m, B, kY, SEED)
    combos = [dict(exact_kernel=k, exact_records=r, exact_group=g)
              for k in (1, 2) for r in (64, 192) for g in (4, 8, 16, 32, 64)]
    combos += [dict(exact_kernel=1, exact_window_log2=s) for s in (8, 9, 11, 12)]
    combos += [dict(exact_kernel=3), dict(exact_kernel=4)]
    combos += [dict(exact_kernel=5, exact_group=g, exact_fields=f)
               for g in (1, 2, 4, 8, 16) for f in (0, 8)]
    for c in combos:
        ctx.set_tuning(**dict(dict(exact_kernel=0, exact_records=0, exact_group=0,
                                   exact_window_log2=0, exact_fields=0), **c))
        out, trace = sk.relu_forward_sparse(model, Y0, sk.ForwardOptions(clip=32.0))
        info = ctx.last_exact()
        assert ctx.layer_paths(1) == ["exact"], c
        assert_same(out, want, f"{cfg} bias {bias} {c}")
        if c["exact_kernel"] == 3:  # push where the counters fit, else the windowed kernel
            assert info["kernel"] == ("push" if m <= 65536 else "specialised"), (c, info)
            continue
        if c["exact_kernel"] == 4:  # flattened products (the specialised kernel's shape)
            assert info["kernel"] == "flat", (c, info)
            continue
        if c["exact_kernel"] == 5:  # K7: windows per pass as asked (8-bit: at most 8)
            g = min(c["exact_group"], 8) if c["exact_fields"] == 8 else c["exact_group"]
            assert (info["kernel"], info["group"]) == ("stream", g), (c, info)
            if c["exact_fields"] == 8:
                assert info["fields"] == 4, (c, info)
            continue
        assert info["kernel"] == {1: "generic", 2: "specialised"}[c["exact_kernel"]], (c, info)
        if "exact_records" in c:
            assert (info["records"], info["group"]) == (c["exact_records"], c["exact_group"])
        else:
            assert info["window_log2"] == c["exact_window_log2"]


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4"])
def test_windowed_engine_full_scale(sk, port, ctx, cfg):
    """Two layers with the order-free kernel and ESC disabled: layer 1 on the
    windowed engine's ordered path (float accumulation, touched lists), layer 2
    on the ordered path again (cfg3: 136 K inputs) or on the frontier path (cfg4:
    24 inputs) -- at the full 60000 samples."""
    m, _, kY, bias, _ = CFG[cfg]
    (hW, hY0) = host_inputs(port, cfg)
    b = np.full(m, bias, np.float32)
    y1 = oracle_layer1(port, cfg, bias)
    y2 = port.layer_sparse(hW[1], b, y1, 32.0)
    Ws = [sk.gen_layer_fixed(m, 32, sk.layer_seed(SEED, k), 1.0 / 16) for k in range(2)]
    model = sk.DnnModel(Ws, [b] * 2)
    Y0 = sk.gen_input_binary(m, B, kY, SEED)
    ctx.set_tuning(exact=-1, esc=-1)
    ctx.set_density_switch(0.0, 0.0)  # keep it on the sparse engine
    out, trace = sk.relu_forward_sparse(model, Y0, sk.ForwardOptions(clip=32.0))
    assert ctx.layer_paths(2)[0] == "engine"
    assert [int(x) for x in trace] == [hY0.nnz, y1.nnz, y2.nnz]
    assert_same(out, y2, f"{cfg} engine 2 layers")


@pytest.mark.parametrize("d", [0.5, 0.1, 0.01, 0.001, 0.0001])
def test_cfg2_full_size_both_legs(sk, ref, port, d):
    """BASELINE configs[1] at 4096 x 4096 . 4096 x 1024 (tools/cfg2_sweep.py's
    seeds): the sparse leg bitwise vs the reference's layer_step (dnn.cpp:86-103),
    the dense tcgen05 leg within approx_equal_scaled of its dense_layer_step."""
    m, n, seed = 4096, 1024, 42
    hW = port.gen_layer_density(m, d, port.layer_seed(seed, 0))
    y = port.gen_input_dense(m, n, seed)
    b = np.full(m, -0.05, np.float32)
    W = sk.gen_layer_density(m, d, sk.layer_seed(seed, 0))
    assert np.array_equal(W.row_ptr(), hW.row_ptr) and np.array_equal(W.col_idx(), hW.col_idx)
    yd = sk.DenseMatrix.from_numpy(y)
    want = ref.layer_step(hW, b, y, workers=8)
    got = sk.layer_step(sk.Matrix(W), b, yd).numpy()
    assert np.array_equal(bits(got), bits(want))
    # dense leg (K4, 3xTF32 on tcgen05): the reference's magnitude-scaled criterion
    wd = hW.to_dense()
    got_d = sk.dense_layer_step(sk.DenseMatrix.from_numpy(wd), b, yd).numpy()
    scale = np.abs(wd).astype(np.float64) @ np.abs(y).astype(np.float64)
    tol = np.maximum(1e-6, 1e-5 * scale)
    assert (np.abs(got_d.astype(np.float64) - want.astype(np.float64)) <= tol).all()


def test_staged_wide_task_standalone_and_saturated_forward(sk, ref, port):
    """K1b (the shared-memory-staged wide task with in-order task claiming):
    * standalone, where the activations exceed the L2 budget (4096 x 4100:
      67 MB, ragged last chunk): layer_step bitwise against the reference
      (dnn.cpp:86-103 over matrix.cpp:403-424) and mxm(CsrMatrix, DenseMatrix)
      under max-plus against the reference's mxm;
    * in the engine on a saturating network (cfg3's construction at 2048
      neurons, 50 % binary inputs, 6000 samples, 5 layers: every layer dense,
      intermediate activations in panel-major scratch): relu_forward_sparse
      bitwise against the oracle's sparse layers."""
    m, n, seed = 4096, 4100, 7
    hW = port.gen_layer_fixed(m, 24, port.layer_seed(seed, 0), float("nan"))
    rng = np.random.default_rng(seed)
    y = rng.uniform(0, 1, (m, n)).astype(np.float32)
    y[rng.random((m, n)) < 0.25] = 0.0
    b = rng.uniform(-0.3, 0.1, m).astype(np.float32)
    W = sk.CsrMatrix(m, m, hW.row_ptr, hW.col_idx, hW.values)
    yd = sk.DenseMatrix.from_numpy(y)
    got = sk.layer_step(sk.Matrix(W), b, yd).numpy()
    assert np.array_equal(bits(got), bits(ref.layer_step(hW, b, y, workers=8)))
    got = sk.mxm(W, yd, sk.max_plus_semiring()).numpy()
    assert np.array_equal(bits(got), bits(ref.mxm_csr_dense(hW, y, "max_plus")))
    del got, yd, y

    m, n, L = 2048, 6000, 5
    hWs = [port.gen_layer_fixed(m, 32, port.layer_seed(SEED, k), 1.0 / 16) for k in range(L)]
    bs = [np.full(m, -0.3, np.float32)] * L
    hY = port.gen_input_binary(m, n, m // 2, SEED)
    want, trace = hY, [hY.nnz]
    for k in range(L):
        want = port.layer_sparse(hWs[k], bs[k], want, 32.0)
        trace.append(want.nnz)
    assert trace[-1] > 0.9 * m * n  # saturated
    ctx = sk.default_context()
    model = sk.DnnModel([sk.CsrMatrix(m, m, w.row_ptr, w.col_idx, w.values) for w in hWs], bs)
    Y0 = sk.CsrMatrix(m, n, hY.row_ptr, hY.col_idx, hY.values)
    out, tr = sk.relu_forward_sparse(model, Y0, sk.ForwardOptions(clip=32.0))
    assert ctx.layer_paths(L).count("dense") >= L - 1
    assert [int(x) for x in tr] == trace
    assert_same(out, want, "saturated forward")
