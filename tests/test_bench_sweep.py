"""The paper's benchmark sweep (proj/include/semikern/bench.hpp): analysis,
CSV formats and configuration checks pinned against the reference library
(CPU), the device gen_weight bitwise against the reference's, and a small
sweep on the GPU."""
import io
import math

import numpy as np
import pytest

from paper_1708_02937_b200 import bench_sweep as bs
from paper_1708_02937_b200 import semikern as skm


def refmsg(e):
    """The reference's message inside an oracle RefError ("Kind: message")."""
    return str(e).split(": ", 1)[1]


def _recs():
    rng = np.random.default_rng(5)
    out = []
    for m in (256, 512, 1024):
        for s in (1.0, 2.0, 4.0, 16.0, 1000.5):
            for impl in (0, 1):
                for wk in (1, 4):
                    out.append((m, s, impl, wk, float(rng.uniform(1e-6, 1e-1)),
                                float(rng.uniform(0, 1e-3)), int(rng.integers(0, 1 << 40)),
                                int(rng.integers(0, 1 << 40))))
    return out


def _as_records(raw):
    return [bs.BenchRecord(m, s, bs.Impl(i), w, me, sd, nz, b) for m, s, i, w, me, sd, nz, b in raw]


def test_analyze_matches_reference(ref):
    raw = _recs()
    want = ref.bench_analyze(raw, 512)
    got = bs.analyze(_as_records(raw), 512)
    assert len(got) == len(want)
    for p, w in zip(got, want):
        vals = [p.m, p.ratio_dense, p.slope, p.saturation, p.blas_per_element,
                p.ratio_dense_normalized, p.slope_normalized, p.saturation_normalized,
                p.blas_per_element_normalized]
        assert vals == list(w)  # identical double arithmetic


def test_csv_formats_match_reference(ref):
    raw = _recs()
    raw += [(8, 1e-05 + 1, 0, 1, 1e-05, 0.0, 0, 0), (8, 1e20, 1, 2, 123456.789, 1e-300, 1, 2),
            (8, 3.0, 0, 3, 0.1 + 0.2, 1 / 3, 5, 6), (8, 1.5, 1, 1, 2.0 ** -30, 1e16, 7, 8)]
    buf = io.StringIO()
    bs.write_records_csv(_as_records(raw), buf)
    assert buf.getvalue() == ref.bench_records_csv(raw)
    buf = io.StringIO()
    bs.write_params_csv(bs.analyze(_as_records(_recs()), 256), buf)
    assert buf.getvalue() == ref.bench_params_csv(_recs(), 256)


def test_number_matches_to_chars(ref):
    vals = [0.0, 1.0, -2.5, 1e-4, 1e-5, 0.0001234, 123456789.0, 1e15, 1e16, 1e17, 1e21,
            3.0e-7, 2.0 ** -52, 5e-324, 1.7976931348623157e308, 0.1, 1 / 3, 1234.5678e10]
    raw = [(1, 1.0, 0, 1, v, 0.0, 0, 0) for v in vals]
    lines = ref.bench_records_csv(raw).strip().split("\n")[1:]
    for v, line in zip(vals, lines):
        assert bs.number(v) == line.split(",")[4], v


def test_read_csv_round_trip_and_errors(ref):
    raw = _recs()
    text = ref.bench_records_csv(raw)
    got = bs.read_records_csv(io.StringIO(text))
    want = ref.bench_read_csv(text)
    assert [(r.m, r.inverse_sparsity, int(r.implementation), r.workers, r.mean_layer_seconds,
             r.stddev_seconds, r.nnz, r.matrix_bytes) for r in got] == want
    head = bs.RECORD_HEADER
    bad = {
        "empty": "",
        "header": "m,x\n",
        "fields": head + "\n1,1,sparse,1,1,1,1\n",
        "impl": head + "\n1,1,sparse\r\n2,1,both,1,1,1,1,1\n",
        "int": head + "\n+1,1,sparse,1,1,1,1,1\n",
        "neg_uint": head + "\n-1,1,sparse,1,1,1,1,1\n",
        "double": head + "\n1, 1,sparse,1,1,1,1,1\n",
        "plus_double": head + "\n1,+1,sparse,1,1,1,1,1\n",
        "hex": head + "\n1,0x10,sparse,1,1,1,1,1\n",
        "overflow_int": head + "\n1,1,sparse,99999999999,1,1,1,1\n",
        "blank_ok_then_bad": head + "\n\n1,1,dense,1,1,1,1,1\n1,1,dense,1,1,1,1,x\n",
    }
    for name, t in bad.items():
        with pytest.raises(Exception) as want_e:
            ref.bench_read_csv(t)
        with pytest.raises(skm.Error) as got_e:
            bs.read_records_csv(io.StringIO(t))
        assert str(got_e.value) == refmsg(want_e.value), name


def test_analyze_errors_match_reference(ref):
    raw = [r for r in _recs() if not (r[0] == 512 and r[1] == 4.0 and r[2] == 0)]
    cases = {"missing_point": (raw, 256), "no_records": ([], 256),
             "bad_reference": (_recs(), 999),
             "no_sparse": ([r for r in _recs() if r[2] == 1], 256)}
    for name, (recs, refm) in cases.items():
        with pytest.raises(Exception) as want_e:
            ref.bench_analyze(recs, refm)
        with pytest.raises(skm.Error) as got_e:
            bs.analyze(_as_records(recs), refm)
        assert str(got_e.value) == refmsg(want_e.value), name


def test_config_validation_matches_reference(ref):
    base = dict(sizes=[64], inverse_sparsities=[1.0], batch=8, layers=1, workers=[1],
                repetitions=5, warmup=1)
    cases = [dict(sizes=[]), dict(inverse_sparsities=[]), dict(workers=[]), dict(workers=[0]),
             dict(repetitions=2), dict(warmup=0), dict(layers=0), dict(sizes=[0]),
             dict(batch=0), dict(inverse_sparsities=[0.5]), dict(inverse_sparsities=[math.nan])]
    for c in cases:
        kw = dict(base, **c)
        with pytest.raises(Exception) as want_e:
            ref.bench_validate(kw["sizes"], kw["inverse_sparsities"], kw["batch"], kw["layers"],
                               kw["workers"], kw["repetitions"], kw["warmup"])
        with pytest.raises(skm.InvalidArgument) as got_e:
            bs.BenchConfig(**kw).validate()
        assert str(got_e.value) == refmsg(want_e.value), c
    ref.bench_validate(**{k: v for k, v in base.items()})
    bs.BenchConfig(**base).validate()


def test_gen_bias_matches_reference(ref):
    for m, seed in ((1, 0), (1000, 7), (4096, 12345)):
        assert np.array_equal(bs.gen_bias(bs.GenSpec(m, 1.0, 1, seed), bs.BiasMode.uniform01),
                              ref.gen_bias(m, seed, True))
        assert np.array_equal(bs.gen_bias(bs.GenSpec(m, 1.0, 1, seed)), ref.gen_bias(m, seed))


@pytest.mark.gpu
def test_device_gen_weight_matches_reference(sk, ref):
    for m, s, seed in ((1, 1.0, 0), (300, 1.0, 3), (1000, 4.0, 7), (2048, 100.0, 11),
                       (777, 3.3, 2)):
        got = sk.gen_weight(m, s, seed)
        want = ref.gen_weight(m, s, seed)
        rp, ci, v = got.extract()
        assert np.array_equal(rp, want.row_ptr) and np.array_equal(ci, want.col_idx)
        assert np.array_equal(np.asarray(v).view(np.uint32), want.values.view(np.uint32))
    with pytest.raises(sk.InvalidArgument, match="inverse_sparsity must be >= 1"):
        sk.gen_weight(10, 0.5, 0)


@pytest.mark.gpu
def test_small_sweep_runs_and_analyzes(sk):
    cfg = bs.BenchConfig(sizes=[256, 512], inverse_sparsities=[1, 4, 64], batch=64,
                         repetitions=3, warmup=1)
    res = bs.run_sweep(cfg)
    assert len(res.records) == 2 * 3 * 2 and not res.skipped
    assert [r.key() for r in res.records] == sorted(r.key() for r in res.records)
    assert all(r.mean_layer_seconds > 0 for r in res.records)
    params = bs.analyze(res.records, 256)
    assert [p.m for p in params] == [256, 512] and params[0].ratio_dense_normalized == 1.0
    buf = io.StringIO()
    bs.write_records_csv(res.records, buf)
    back = bs.read_records_csv(io.StringIO(buf.getvalue()))
    assert [r.key() for r in back] == [r.key() for r in res.records]
