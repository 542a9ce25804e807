"""The paper's benchmark sweep on the B200 (proj/include/semikern/bench.hpp,
proj/src/bench.cpp; the experiment behind Kepner et al.'s sparse-vs-dense
timing curves).

For every (size m, inverse sparsity) cell the weights are generated once with
the reference's own ``gen_weight`` (device-side, bitwise: ``sk_gen_weight``),
the input with ``gen_input`` and the bias with ``gen_bias``; the dense leg times
``dense_layer_step`` on the explicit-zero dense form of the same weights (K4,
tcgen05), the sparse leg ``layer_step`` (K1).  A sample is ``layers``
consecutive steps from the same input, the recorded time is per layer (CUDA
events on the library's stream around the steps: device time of the whole API
calls), ``warmup`` samples are discarded, mean and sample standard deviation
over ``repetitions`` (bench.cpp ``time_step`` / ``mean_stddev``).

``analyze``, the CSV writers/reader and ``BenchConfig.validate`` restate
bench.cpp exactly (same formulas, field formatting -- std::to_chars shortest
round trip -- and error messages); tests/test_bench_sweep.py pins them against
the reference library.
"""
from __future__ import annotations

import argparse
import dataclasses
import math
import re
import sys
from enum import IntEnum
from typing import IO, Iterable, Sequence

import numpy as np

from . import semikern as sk

RECORD_HEADER = ("m,inverse_sparsity,implementation,workers,mean_layer_seconds,"
                 "stddev_seconds,nnz,matrix_bytes")
PARAMS_HEADER = ("m,ratio_dense,slope,saturation,blas_per_element,ratio_dense_normalized,"
                 "slope_normalized,saturation_normalized,blas_per_element_normalized")


class Impl(IntEnum):  # bench.hpp: enum class Impl { sparse, dense }
    sparse = 0
    dense = 1


def impl_name(impl: Impl) -> str:
    return "sparse" if impl == Impl.sparse else "dense"


class BiasMode(IntEnum):  # matgen.hpp
    zero = 0
    uniform01 = 1


@dataclasses.dataclass
class GenSpec:  # matgen.hpp:29-37
    m: int = 0
    inverse_sparsity: float = 1.0
    batch: int = 64
    seed: int = 0

    def validate(self) -> None:
        if self.m < 1:
            raise sk.InvalidArgument("GenSpec: m must be >= 1")
        if self.batch < 1:
            raise sk.InvalidArgument("GenSpec: batch must be >= 1")
        if not (self.inverse_sparsity >= 1.0):
            raise sk.InvalidArgument("GenSpec: inverse_sparsity must be >= 1")


@dataclasses.dataclass
class BenchConfig:  # bench.hpp:37-51
    sizes: list = dataclasses.field(default_factory=list)
    inverse_sparsities: list = dataclasses.field(default_factory=list)
    batch: int = 64
    layers: int = 1
    workers: list = dataclasses.field(default_factory=lambda: [1])
    repetitions: int = 5
    warmup: int = 1
    seed: int = 0
    bias_mode: BiasMode = BiasMode.zero
    output: str | None = None

    def validate(self) -> None:  # bench.cpp BenchConfig::validate
        if not self.sizes:
            raise sk.InvalidArgument("sweep needs at least one size")
        if not self.inverse_sparsities:
            raise sk.InvalidArgument("sweep needs at least one inverse sparsity")
        if not self.workers:
            raise sk.InvalidArgument("sweep needs a workers list")
        for w in self.workers:
            if w < 1:
                raise sk.InvalidArgument("workers must be >= 1")
        if self.repetitions < 3:
            raise sk.InvalidArgument("repetitions must be >= 3")
        if self.warmup < 1:
            raise sk.InvalidArgument("warmup must be >= 1")
        if self.layers < 1:
            raise sk.InvalidArgument("layers must be >= 1")
        for m in self.sizes:
            for s in self.inverse_sparsities:
                GenSpec(m, s, self.batch, self.seed).validate()


@dataclasses.dataclass
class BenchRecord:  # bench.hpp:53-62
    m: int = 0
    inverse_sparsity: float = 1.0
    implementation: Impl = Impl.sparse
    workers: int = 1
    mean_layer_seconds: float = 0.0
    stddev_seconds: float = 0.0
    nnz: int = 0
    matrix_bytes: int = 0

    def key(self):
        return (self.m, self.inverse_sparsity, int(self.implementation), self.workers)


@dataclasses.dataclass
class SkippedRun:
    m: int
    inverse_sparsity: float
    implementation: Impl
    workers: int
    reason: str


@dataclasses.dataclass
class SweepResult:
    records: list
    skipped: list


@dataclasses.dataclass
class CurveParams:  # bench.hpp:97-107
    m: int = 0
    ratio_dense: float = 0.0
    slope: float = 0.0
    saturation: float = 0.0
    blas_per_element: float = 0.0
    ratio_dense_normalized: float = 0.0
    slope_normalized: float = 0.0
    saturation_normalized: float = 0.0
    blas_per_element_normalized: float = 0.0


# ---- generators (matgen.cpp; the weights and inputs run on the device) -----------------

_M64 = (1 << 64) - 1


def _splitmix_at(seed: int, idx: np.ndarray) -> np.ndarray:
    """rng.hpp SplitMix64::at, vectorised (wrapping uint64 arithmetic)."""
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) + (idx.astype(np.uint64) + np.uint64(1)) *
             np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _stream_seed(seed: int, which: int) -> int:
    return int(_splitmix_at(seed, np.array([which], np.uint64))[0])


def gen_bias(spec: GenSpec, mode: BiasMode = BiasMode.zero) -> np.ndarray:
    """matgen.cpp gen_bias: zero, or float(to_unit(at(stream kBias = 3, i)))."""
    spec.validate()
    if mode != BiasMode.uniform01:
        return np.zeros(spec.m, np.float32)
    bits = _splitmix_at(_stream_seed(spec.seed, 3), np.arange(spec.m, dtype=np.uint64))
    return ((bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53).astype(np.float32)


# ---- timing --------------------------------------------------------------------------

def _mean_stddev(samples: Sequence[float]) -> tuple[float, float]:
    mean = 0.0
    for x in samples:
        mean += x
    mean /= len(samples)
    ss = 0.0
    for x in samples:
        ss += (x - mean) * (x - mean)
    sd = math.sqrt(ss / (len(samples) - 1)) if len(samples) > 1 else 0.0
    return mean, sd


def _time_step(y0, layers: int, warmup: int, repetitions: int, step, stream) -> tuple:
    import torch
    samples = []
    for rep in range(warmup + repetitions):
        y = y0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(layers):
            y = step(y)
        e1.record(stream)
        e1.synchronize()
        if rep >= warmup:
            samples.append(e0.elapsed_time(e1) / 1e3 / layers)
    return _mean_stddev(samples)


def run_sweep(config: BenchConfig, progress: IO | None = None) -> SweepResult:
    """bench.cpp run_sweep on the GPU: CUDA events on a dedicated stream that the
    library is pointed at (the legacy default stream has handle 0, which
    set_stream reads as "the library's own stream": events recorded there would
    not bracket the kernels)."""
    import torch
    config.validate()
    ctx = sk.default_context()
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    res = SweepResult([], [])
    try:
        _sweep_into(res, config, stream, progress)
    finally:
        ctx.synchronize()
        ctx.set_stream(None)  # back to the library's own stream before `stream` goes away
    res.records.sort(key=BenchRecord.key)
    return res


def _sweep_into(res: SweepResult, config: BenchConfig, stream, progress) -> None:
    workers = sorted(set(config.workers))
    for m in sorted(set(config.sizes)):
        for s in sorted(set(config.inverse_sparsities)):
            spec = GenSpec(m, s, config.batch, config.seed)
            w = sk.gen_weight(m, s, config.seed)
            bias = gen_bias(spec, config.bias_mode)
            y0 = sk.gen_input_dense(m, config.batch, config.seed)
            nnz = w.nnz()
            sparse_bytes = (m + 1) * 4 + nnz * 8  # storage_bytes(Matrix(w))
            for wk in workers:
                try:
                    wd = sk.to_dense(w, 0.0)
                    mean, sd = _time_step(
                        y0, config.layers, config.warmup, config.repetitions,
                        lambda y, wd=wd, wk=wk: sk.dense_layer_step(wd, bias, y, workers=wk),
                        stream)
                    res.records.append(BenchRecord(m, s, Impl.dense, wk, mean, sd, nnz, m * m * 4))
                    if progress:
                        print(f"m={m} is={s:g} dense workers={wk} mean={mean:g}s", file=progress)
                except sk.OutOfMemory:
                    res.skipped.append(SkippedRun(
                        m, s, Impl.dense, wk, f"allocation of {m * m * 4} dense bytes failed"))
                    if progress:
                        print(f"m={m} is={s:g} dense workers={wk} skipped (allocation failed)",
                              file=progress)
            wm = sk.Matrix(w)
            for wk in workers:
                mean, sd = _time_step(
                    y0, config.layers, config.warmup, config.repetitions,
                    lambda y, wk=wk: sk.layer_step(wm, bias, y, None,
                                                   sk.ForwardOptions(workers=wk)),
                    stream)
                res.records.append(BenchRecord(m, s, Impl.sparse, wk, mean, sd, nnz, sparse_bytes))
                if progress:
                    print(f"m={m} is={s:g} sparse workers={wk} mean={mean:g}s", file=progress)


# ---- analysis (bench.cpp analyze) ---------------------------------------------------------

def _g(x: float) -> str:
    """operator<< of a double with default stream precision (%g)."""
    return f"{x:g}"


def analyze(records: Iterable[BenchRecord], reference_m: int) -> list[CurveParams]:
    records = list(records)
    sizes = sorted({r.m for r in records})
    if not sizes:
        raise sk.Error("analyze: no records")

    def require_time(m, impl, s):
        for r in records:
            if r.m == m and r.implementation == impl and r.inverse_sparsity == s and \
                    r.workers == 1:
                return r.mean_layer_seconds
        raise sk.Error(f"analyze: no {impl_name(impl)} record at inverse sparsity {_g(s)} "
                       f"for m={m} (workers=1)")

    params = []
    for m in sizes:
        max_is = 0.0
        for r in records:
            if r.m == m and r.implementation == Impl.sparse and r.workers == 1:
                max_is = max(max_is, r.inverse_sparsity)
        if max_is == 0.0:
            raise sk.Error(f"analyze: no sparse records for m={m} (workers=1)")
        t_s1 = require_time(m, Impl.sparse, 1.0)
        t_s4 = require_time(m, Impl.sparse, 4.0)
        t_sat = require_time(m, Impl.sparse, max_is)
        t_d1 = require_time(m, Impl.dense, 1.0)
        elements = float(m) * m
        params.append(CurveParams(m, t_s1 / t_d1, (t_s1 - t_s4) / (0.75 * elements),
                                  t_sat / float(m), t_d1 / elements))
    ref = next((p for p in params if p.m == reference_m), None)
    if ref is None:
        raise sk.Error(f"analyze: reference size m={reference_m} has no records")
    r = dataclasses.replace(ref)
    for p in params:
        p.ratio_dense_normalized = p.ratio_dense / r.ratio_dense
        p.slope_normalized = p.slope / r.slope
        p.saturation_normalized = p.saturation / r.saturation
        p.blas_per_element_normalized = p.blas_per_element / r.blas_per_element
    return params


# ---- CSV (bench.cpp) ----------------------------------------------------------------------

def number(v: float) -> str:
    """std::to_chars(double): shortest round-trip digits, in fixed or
    scientific notation, whichever is shorter (fixed on a tie), %e-style
    exponent with at least two digits."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    fixed = np.format_float_positional(v, unique=True, trim="-")
    sci = np.format_float_scientific(v, unique=True, trim="-", exp_digits=2)
    return fixed if len(fixed) <= len(sci) else sci


def write_records_csv(records: Iterable[BenchRecord], out: IO | str) -> None:
    lines = [RECORD_HEADER]
    for r in records:
        lines.append(f"{r.m},{number(r.inverse_sparsity)},{impl_name(r.implementation)},"
                     f"{r.workers},{number(r.mean_layer_seconds)},{number(r.stddev_seconds)},"
                     f"{r.nnz},{r.matrix_bytes}")
    text = "\n".join(lines) + "\n"
    if isinstance(out, str):
        try:
            with open(out, "w") as f:
                f.write(text)
        except OSError:
            raise sk.Error(f"cannot open '{out}' for writing") from None
    else:
        out.write(text)


def write_params_csv(params: Iterable[CurveParams], out: IO | str) -> None:
    lines = [PARAMS_HEADER]
    for p in params:
        lines.append(",".join([str(p.m)] + [number(x) for x in (
            p.ratio_dense, p.slope, p.saturation, p.blas_per_element, p.ratio_dense_normalized,
            p.slope_normalized, p.saturation_normalized, p.blas_per_element_normalized)]))
    text = "\n".join(lines) + "\n"
    if isinstance(out, str):
        try:
            with open(out, "w") as f:
                f.write(text)
        except OSError:
            raise sk.Error(f"cannot open '{out}' for writing") from None
    else:
        out.write(text)


# std::from_chars accepts exactly these (no leading '+', no whitespace, no hex
# in general format); integers are plain decimal digits (a '-' only for signed)
_DOUBLE = re.compile(r"-?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|(?i:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?))")
_UINT = re.compile(r"\d+")
_SINT = re.compile(r"-?\d+")


def _parse_double(tok: str, line: int) -> float:
    if not _DOUBLE.fullmatch(tok):
        raise sk.ParseError(f"line {line}: malformed number '{tok}'")
    v = float(tok)
    if math.isinf(v) and "inf" not in tok.lower():  # from_chars: result_out_of_range
        raise sk.ParseError(f"line {line}: malformed number '{tok}'")
    return v


def _parse_int(tok: str, line: int, signed: bool, bits: int) -> int:
    if not (_SINT if signed else _UINT).fullmatch(tok):
        raise sk.ParseError(f"line {line}: malformed integer '{tok}'")
    v = int(tok)
    lo, hi = (-(1 << (bits - 1)), (1 << (bits - 1)) - 1) if signed else (0, (1 << bits) - 1)
    if not (lo <= v <= hi):
        raise sk.ParseError(f"line {line}: malformed integer '{tok}'")
    return v


def read_records_csv(src: IO | str) -> list[BenchRecord]:
    if isinstance(src, str):
        try:
            with open(src) as f:
                text = f.read()
        except OSError:
            raise sk.Error(f"cannot open '{src}' for reading") from None
    else:
        text = src.read()
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # getline does not produce a final empty line
    if not lines:
        raise sk.ParseError("line 1: empty CSV")
    head = lines[0][:-1] if lines[0].endswith("\r") else lines[0]
    if head != RECORD_HEADER:
        raise sk.ParseError(f"line 1: unexpected CSV header '{head}'")
    out = []
    for no, line in enumerate(lines[1:], start=2):
        if line.endswith("\r"):
            line = line[:-1]
        if not line:
            continue
        f = line.split(",")
        if len(f) != 8:
            raise sk.ParseError(f"line {no}: expected 8 fields, found {len(f)}")
        r = BenchRecord()
        r.m = _parse_int(f[0], no, False, 32)
        r.inverse_sparsity = _parse_double(f[1], no)
        if f[2] == "sparse":
            r.implementation = Impl.sparse
        elif f[2] == "dense":
            r.implementation = Impl.dense
        else:
            raise sk.ParseError(f"line {no}: unknown implementation '{f[2]}'")
        r.workers = _parse_int(f[3], no, True, 32)
        r.mean_layer_seconds = _parse_double(f[4], no)
        r.stddev_seconds = _parse_double(f[5], no)
        r.nnz = _parse_int(f[6], no, False, 64)
        r.matrix_bytes = _parse_int(f[7], no, False, 64)
        out.append(r)
    return out


# ---- command line (the sweep binary of the reference: semikern bench) ---------------------

def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--sizes", default="1024,2048,4096")
    ap.add_argument("--inverse-sparsities", default="1,2,4,8,16,32,64,128,256,512,1024")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--workers", default="1")
    ap.add_argument("--repetitions", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--bias", choices=["zero", "uniform01"], default="zero")
    ap.add_argument("--reference-m", type=int, default=0)
    ap.add_argument("--output", default="sweep.csv")
    ap.add_argument("--params", default="")
    a = ap.parse_args(argv)
    cfg = BenchConfig([int(x) for x in a.sizes.split(",")],
                      [float(x) for x in a.inverse_sparsities.split(",")], a.batch, a.layers,
                      [int(x) for x in a.workers.split(",")], a.repetitions, a.warmup, a.seed,
                      BiasMode[a.bias], a.output)
    res = run_sweep(cfg, progress=sys.stderr)
    write_records_csv(res.records, a.output)
    for s in res.skipped:
        print(f"skipped m={s.m} is={s.inverse_sparsity:g} {impl_name(s.implementation)}: "
              f"{s.reason}", file=sys.stderr)
    if a.params:
        write_params_csv(analyze(res.records, a.reference_m or min(cfg.sizes)), a.params)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
