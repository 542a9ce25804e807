#!/usr/bin/env python
"""Benchmark of the sparse ReLU DNN inference path (Y_{k+1} = ReLU(Y_k W_k + b_k)).

Default workload: BASELINE.json configs[3] ("cfg4"), the configuration the
metric is quoted on at 1/2/4/8 GPUs: 480 layers, N = 65536 neurons, W_k with
exactly 32 nonzeros per row (value 1/16), bias -0.35, ReLU clipped at 32,
Y0 binary with round(0.4% * N) = 262 active neurons per sample, ONE batch of
60000 samples.  At N > 1 the batch is split into contiguous sample shards
(batch-row sharding, replicated W, no collective on the data path; the
partition is the reference's count*w/nw rule, proj/src/detail/parallel.hpp:
29-43): strong scaling, 7500 samples per GPU at N = 8 (`--scaling weak` gives
every GPU its own 60000 instead).  One step = one full 480-layer inference.

The line also carries a `sustained` object: the cfg3 network driven into its
saturated regime (every layer does full work), because the
BASELINE configs as specified die after 1-2 layers.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4|cfg3|cfg5|cfg1]
    python bench.py --impl reference ...   # the reference's CPU path, rank 0 only

Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edges/sec (nnz(W)·batch MACs/s)"

WORKLOADS = {
    # name: (neurons, layers, per-rank batch, W nnz/row, value, bias, clip, Y0 kind, Y0 k)
    "cfg4": dict(m=65536, L=480, B=60000, kW=32, value=1.0 / 16, bias=-0.35, clip=32.0,
                 y0="binary", density=0.004,
                 desc="BASELINE configs[3]: 480-layer sparse DNN, N=65536, 32 nnz/row (1/16), "
                      "bias -0.35, ReLU clip 32, Y0 binary 0.4%/sample, 60000 samples"),
    "cfg3": dict(m=16384, L=120, B=60000, kW=32, value=1.0 / 16, bias=-0.3, clip=32.0,
                 y0="binary", density=0.015,
                 desc="BASELINE configs[2]: 120-layer sparse DNN, N=16384, 32 nnz/row (1/16), "
                      "bias -0.3, ReLU clip 32, Y0 binary 1.5%/sample, 60000 samples"),
    # Not a BASELINE config: the cfg3 network driven into its saturated regime
    # (Y0 50% ones -> every activation clips at 32 from layer 1 on), so every
    # layer carries full work.  Exercises the density-adaptive hand-off to the
    # dense engine; reported separately, never as the headline.
    "cfg3_saturated": dict(m=16384, L=120, B=60000, kW=32, value=1.0 / 16, bias=-0.3,
                           clip=32.0, y0="binary", density=0.5,
                           desc="sustained-work variant of BASELINE configs[2] (NOT a BASELINE "
                                "config): cfg3 network, Y0 binary 50%/sample -> activations "
                                "saturate (dense) from layer 2, 60000 samples"),
    "cfg5": dict(m=262144, L=120, B=60000, kW=32, value=1.0 / 16, bias=-0.45, clip=32.0,
                 y0="binary", density=0.001,
                 desc="BASELINE configs[4]: 120-layer sparse DNN, N=262144, 32 nnz/row (1/16), "
                      "bias -0.45, ReLU clip 32, Y0 binary 0.1%/sample, 60000 samples"),
    "cfg1": dict(m=1024, L=4, B=256, kW=16, value=float("nan"), bias=-0.05, clip=0.0,
                 y0="dense", density=1.0,
                 desc="BASELINE configs[0]: 4-layer sparse DNN, N=1024, 16 nnz/row U[-1,1), "
                      "bias -0.05, Y0 dense U[0,1), batch 256"),
}
E2E_DEPTH = 2  # inputs in flight ahead of the forward in the end-to-end loop
SEED = 42


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ---------------------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md "clocks line")

class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed
    region.  In-process NVML (nvidia_ml_py) from a background thread: spawning
    nvidia-smi stalls CUDA API calls while it initialises NVML, which lands in
    short timed regions.  NVML is initialised and queried once before the region
    starts; a sample is also taken at entry and exit so short regions still get
    samples.  Falls back to `nvidia-smi -lms` if NVML is unavailable."""

    PERIOD_S = 0.05

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []  # (sm_mhz, max_mhz, reasons_bitmask)
        self.nv = None
        self.h = None
        self.thread = None
        self.proc = None
        self.path = os.path.join("/tmp", f"sk_clocks_{os.getpid()}_{gpu_index}.csv")
        if os.environ.get("SK_BENCH_NO_CLOCKS"):  # diagnostics only
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = None
            try:  # the CUDA device's own GPU (NVML ignores CUDA_VISIBLE_DEVICES)
                import torch
                uuid = str(torch.cuda.get_device_properties(self.gpu).uuid)
                self.h = pynvml.nvmlDeviceGetHandleByUUID(
                    uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self.rows.clear()
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.rows.append((float(sm), float(self.max_mhz), int(reasons)))

    def _loop(self):
        import threading  # noqa: F401
        while not self.stop.wait(self.PERIOD_S):
            try:
                self._sample()
            except Exception:
                return

    def __enter__(self):
        if os.environ.get("SK_BENCH_NO_CLOCKS"):
            return self
        if self.nv is not None:
            import threading
            self.stop = threading.Event()
            self._sample()
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
            return self
        try:  # fallback: nvidia-smi, started well before the region
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            t0 = time.time()
            while time.time() - t0 < 10 and os.path.getsize(self.path) == 0:
                time.sleep(0.05)
            time.sleep(0.5)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.thread is not None:
            self.stop.set()
            self.thread.join()
            try:
                self._sample()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if self.nv is not None and self.rows:
            nv = self.nv
            bits = [getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
                    getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                    getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                    getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4)]
            sm = [r[0] for r in self.rows]
            mx = max(r[1] for r in self.rows)
            reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2] & bits[i]})
            loaded = [x for x in sm if x > 0.5 * mx] or sm
            return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                    "samples": len(self.rows), "source": "nvml"}
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 7 and parts[0].replace(".", "").isdigit():
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows]
        mx = max(float(r[1]) for r in rows)
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "source": "nvidia-smi"}


# ---------------------------------------------------------------------------------------
# workload construction

def kY_of(w):
    return max(1, int(round(w["density"] * w["m"])))


def edges_per_inference(w, batch):
    return w["L"] * w["m"] * w["kW"] * batch


def build_model(sk, w):
    Ws = [sk.gen_layer_fixed(w["m"], w["kW"], sk.layer_seed(SEED, k), w["value"])
          for k in range(w["L"])]
    b = np.full(w["m"], w["bias"], np.float32)
    return sk.DnnModel(Ws, [b] * w["L"]), Ws


def sparse_layer_bytes(nnz_in, nnz_out, batch, m, nnzW):
    """8 nnz(Y_k) + 8 nnz(Y_k+1) + 8(B+1) + 4(N+1) + 8 nnz(W) + 4N."""
    return 8 * nnz_in + 8 * nnz_out + 8 * (batch + 1) + 4 * (m + 1) + 8 * nnzW + 4 * m


def dense_layer_bytes(batch, m, nnzW):
    """8 B N + 4(N+1) + 8 nnz(W) + 4N."""
    return 8 * batch * m + 4 * (m + 1) + 8 * nnzW + 4 * m


def useful_products(trace, paths, m, batch, nnzW, layer1_products):
    """Multiply-adds the forward actually needs: layer 1 counted exactly
    (sum over input neurons of out-degree x active samples), later sparse
    layers at their expected count nnz(Y_k) nnz(W_k) / N, dense-engine layers
    every MAC (the engine folds all of them).  Empty layers need none."""
    tot = 0.0
    for k in range(len(trace) - 1):
        if k == 0 and layer1_products is not None:
            tot += layer1_products
        elif paths and paths[k] == "dense":
            tot += nnzW[k] * batch
        else:
            tot += trace[k] * nnzW[k] / m
    return tot


def measured_traffic(workload):
    """Per-launch DRAM traffic of the dominant kernel from the committed ncu
    capture (profiles/r02/traffic.json, else r01) and the unit that binds it."""
    for r in ("r02", "r01"):
        try:
            t = json.load(open(os.path.join(ROOT, "profiles", r, "traffic.json")))
            return t[workload]["bytes"], t[workload]["report"], t[workload].get("limiter")
        except Exception:
            continue
    return None, None, None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# ---------------------------------------------------------------------------------------
# the reference's CPU implementation (oracle/_ref): reference arm and cpu_baseline

def host_weight_handles(R, P, w, cores):
    """The L weight matrices as reference CsrMatrix handles (generated by the
    oracle's C generators in parallel; setup, never timed)."""
    from concurrent.futures import ThreadPoolExecutor

    def one(k):
        x = P.gen_layer_fixed(w["m"], w["kW"], P.layer_seed(SEED, k), w["value"])
        return R.handle(x)

    with ThreadPoolExecutor(max_workers=max(1, cores)) as ex:
        return list(ex.map(one, range(w["L"])))


def cpu_reference_run(w, batch, steps, warmup, workers):
    """Times the reference's CPU path on the FULL workload (`batch` samples, all
    L layers), mirroring time_step (proj/src/bench.cpp:82-95): each step
    restarts from Y0.  Sparse-activation configs: per layer the reference's
    mxm(CsrMatrix W_ref, CsrMatrix Y_ref) (proj/src/matrix.cpp:541-547 ->
    452-521) with `workers` threads, followed by the sparse epilogue the
    reference lacks (restated in oracle/ref_capi.cpp), Y kept as a reference
    CsrMatrix between layers.  Dense-input configs: the reference's relu_forward
    (proj/src/dnn.cpp:111-121).  Returns (per-step seconds, per-step per-layer
    seconds)."""
    from oracle.oracle import Port, Ref
    R, P = Ref.get(), Port.get()
    m = w["m"]
    b = np.full(m, w["bias"], np.float32)
    times, per_layer = [], []
    if w["y0"] == "dense":
        W_host = [P.gen_layer_fixed(m, w["kW"], P.layer_seed(SEED, k), w["value"])
                  for k in range(w["L"])]
        y0 = P.gen_input_dense(m, batch, SEED)
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            R.relu_forward(W_host, [b] * w["L"], y0, workers=workers)
            if it >= warmup:
                times.append(time.perf_counter() - t0)
        return times, per_layer
    hW = host_weight_handles(R, P, w, workers)
    hY0 = R.handle(P.gen_input_binary(m, batch, kY_of(w), SEED))
    try:
        for it in range(warmup + steps):
            lt, hy = [], hY0
            for k in range(w["L"]):
                t0 = time.perf_counter()
                hn = R.layer_sparse_h(hW[k], hy, b, w["clip"], workers)
                lt.append(time.perf_counter() - t0)
                if hy is not hY0:
                    R.free(hy)
                hy = hn
            if hy is not hY0:
                R.free(hy)
            if it >= warmup:
                times.append(sum(lt))
                per_layer.append(lt)
    finally:
        for h in hW:
            R.free(h)
        R.free(hY0)
    return times, per_layer


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_sample_desc(w, cores, per_layer):
    if w["y0"] == "dense":
        return (f"full workload ({w['B']} samples, {w['L']} layers): reference relu_forward "
                f"workers={cores}")
    s = (f"full workload ({w['B']} samples, all {w['L']} layers, nothing extrapolated): per "
         f"layer the reference's mxm(CsrMatrix,CsrMatrix) workers={cores} + the restated "
         f"sparse epilogue (oracle/ref_capi.cpp skref_layer_sparse_h)")
    if per_layer:
        pl = np.mean(np.array(per_layer), axis=0) * 1e3
        s += f"; mean ms per layer: layer 1 {pl[0]:.1f}, layer 2 {pl[1]:.1f}" if len(pl) > 1 else ""
        if len(pl) > 2:
            s += f", layers 3-{len(pl)} total {float(np.sum(pl[2:])):.1f}"
    return s


def run_reference(args, w):
    """--impl reference: rank 0 times the reference's CPU path on the same
    workload (the global batch, every layer); other ranks exit without work."""
    rank, _, world = env_rank()
    if rank != 0:
        return
    cores = cpu_cores()
    times, per_layer = cpu_reference_run(w, w["B"], args.steps, args.warmup, cores)
    t = statistics.mean(times)
    value = edges_per_inference(w, w["B"]) / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.scaling == "strong" else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": w["desc"], "global_batch": w["B"], "cpu_batch": w["B"],
                   "layers": w["L"]},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": cores,
                         "kind": "reference", "sample": cpu_sample_desc(w, cores, per_layer),
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# our arm

class Rank:
    def __init__(self, args):
        import torch
        self.rank, self.local, self.world = env_rank()
        torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1 or (args.shard == "cols" and "MASTER_ADDR" in os.environ):
            import torch.distributed as dist
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.dist = dist

    def barrier(self):
        import torch
        if self.dist is not None:
            self.dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(self, x):
        import torch
        t = torch.tensor([float(x)], device="cuda")
        if self.dist is not None:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


def timed_steps(R, stream, steps, fn):
    """K steps of fn() between barriers, CUDA events on the library's stream;
    returns the max over ranks of the elapsed ms."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R.barrier()
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    R.barrier()
    return R.max_over_ranks(e0.elapsed_time(e1))


def layer1_products(W0, host_rp):
    """Exact multiply-add count of layer 1: sum over input neurons k of
    out-degree(k) (column count of W_ref) x active samples of neuron k."""
    ci = np.asarray(W0.col_idx(), np.int64)
    outdeg = np.bincount(ci, minlength=len(host_rp) - 1).astype(np.float64)
    return float(np.dot(outdeg, np.diff(host_rp.astype(np.int64)).astype(np.float64)))


def run_sustained(sk, ctx, stream, R, args, pk, b0, Bl, Bg):
    """The `sustained` object: the cfg3 network in its saturated regime
    (WORKLOADS['cfg3_saturated'], not a BASELINE config), every layer full work;
    the dense engine dominates.  Same timing rules as the headline."""
    w = WORKLOADS["cfg3_saturated"]
    model, Ws = build_model(sk, w)
    nnzW = [x.nnz() for x in Ws]
    del Ws
    Y0 = sk.gen_input_binary(w["m"], Bl, kY_of(w), SEED, sample_offset=b0)
    run = lambda: sk.relu_forward_sparse(model, Y0, sk.ForwardOptions(clip=w["clip"]))  # noqa
    trace = None
    for _ in range(3):
        _, trace = run()
    steps = 3
    ctx.set_timing(True)
    ctx.kernel_times_tagged()
    ms = timed_steps(R, stream, steps, run) / steps
    kt, tags = ctx.kernel_times_tagged()
    ctx.set_timing(False)
    paths = ctx.layer_paths(w["L"])
    tr = [int(x) for x in trace]
    dense_layers = paths.count("dense")
    dense_ms = float(sum(t for t, g in zip(kt, tags) if g == "k_dense_engine")) / steps
    byts = dense_layers * dense_layer_bytes(Bl, w["m"], nnzW[0])
    macs = dense_layers * nnzW[0] * Bl
    achieved = byts / (dense_ms / 1e3) / 1e9 if dense_ms > 0 else 0.0
    fma_peak = ctx_fma_peak(sk)
    edges = edges_per_inference(w, Bg)
    useful = useful_products(tr, paths, w["m"], Bl, nnzW, None)
    # per-layer DRAM traffic of the engine from the committed ncu capture (one
    # saturated 60000-sample layer), scaled to this rank's batch
    tb, trep, _ = measured_traffic("cfg3_saturated_wide")
    if tb is not None:
        tb = int(tb * Bl / 60000)
    sustained_extra = {
        "traffic_per_layer": tb, "traffic_source": trep,
        "algorithmic_bytes_per_layer": dense_layer_bytes(Bl, w["m"], nnzW[0]),
        "l2_to_sm_gbs": 4.0 * macs / (dense_ms / 1e3) / 1e9 if dense_ms > 0 else 0.0,
        "measured_limiter": "L1/TEX data pipe 85 % (cp.async writes + shared reads of the staged "
                            "activation segments), L2 76 %, issue 67 %; 4 B per MAC cross "
                            "L2 -> SM (no on-chip reuse for a random W), DRAM traffic 1.02x the "
                            "algorithmic bytes (profiles/r02/engine_staged_b60000_brief.txt)",
    }
    return {
        "workload": w["desc"], "value": edges / (ms / 1e3), "unit": "edges/s",
        "ms_per_step": ms, "steps": steps, "warmup": 3,
        "useful_products_per_s": useful * (Bg / Bl) / (ms / 1e3),
        "nnz_trace": tr[:4] + ["..."] + tr[-1:],
        "layer_paths": {p_: paths.count(p_) for p_ in sorted(set(paths))},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": None,
                     "kernel": "k_dense_engine_bulk (K1b, dense-activation layers: fused SpMM + "
                               "bias/ReLU/clip; activation segments staged through shared "
                               "memory by cp.async, tasks claimed in panel order)",
                     "algorithmic_bytes": byts, "launch_ms": dense_ms,
                     "kernel_share_of_step": dense_ms / ms,
                     "fp32_macs_per_s": macs / (dense_ms / 1e3) if dense_ms > 0 else 0.0,
                     "fp32_frac": (macs / (dense_ms / 1e3)) / fma_peak if dense_ms > 0 else 0.0,
                     "fp32_peak_macs_per_s": fma_peak,
                     "fp32_note": "non-fused mul + add (bitwise parity): 2 FP32 pipe ops per "
                                  "MAC; peak = SMs x 128 lanes x max SM clock / 2",
                     **sustained_extra},
    }


def ctx_fma_peak(sk):
    """Non-fused FP32 multiply-add peak (MAC/s): 2 pipe ops per MAC."""
    import torch
    p = torch.cuda.get_device_properties(torch.cuda.current_device())
    clk = 1965e6
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        clk = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM) * 1e6
    except Exception:
        pass
    return p.multi_processor_count * 128 * clk / 2


def sample_plan(Bg, world, rank, cols, strong):
    """(first sample, samples on this rank, samples of the whole job).  Column
    sharding: every rank holds the whole batch.  Strong batch-row scaling: the one
    global batch split by the reference's count*w/nw rule
    (proj/src/detail/parallel.hpp:29-43).  Weak: every rank its own Bg samples."""
    from paper_1708_02937_b200 import shard
    if cols:
        return 0, Bg, Bg
    if strong:
        b0, Bl = shard.batch_shard(Bg, world, rank)
        return b0, Bl, Bg
    return rank * Bg, Bg, Bg * world


def run_ours(args, w):
    import torch
    R = Rank(args)
    rank, local, world, dist = R.rank, R.local, R.world, R.dist
    import paper_1708_02937_b200 as sk
    from paper_1708_02937_b200 import shard
    sk.set_device(local)
    ctx = sk.default_context()
    # a dedicated stream: the library launches on it and the timing events are
    # recorded on it (torch's legacy default stream would map to the library's
    # own private stream)
    stream = torch.cuda.Stream(device=local)
    ctx.set_stream(stream.cuda_stream)

    m, L, Bg = w["m"], w["L"], w["B"]
    cols = args.shard == "cols" and w["y0"] == "binary"
    strong = args.scaling == "strong"
    b0, Bl, job_batch = sample_plan(Bg, world, rank, cols, strong)
    layer1 = None
    if cols:
        # column sharding: this rank owns output neurons [r0, r1) of every W_ref and
        # the whole batch; one exchange of the sparse activations per layer
        dev = torch.device("cuda", local)
        r0, r1 = shard.block_range(m, world, rank)
        blocks, nnzW = [], []
        for k in range(L):
            wf = sk.gen_layer_fixed(m, w["kW"], sk.layer_seed(SEED, k), w["value"])
            nnzW.append(wf.nnz())
            blocks.append(shard.row_block(wf, r0, r1, dev))
            del wf
        bblocks = [np.full(r1 - r0, w["bias"], np.float32)] * L
        Y0 = sk.gen_input_binary(m, Bg, kY_of(w), SEED)
        peer = shard.PeerExchange(m, ctx=ctx) if args.exchange == "peer" else None
        plan = shard.ColShardPlan(blocks, bblocks, device=dev)  # device biases, agreed flags
        run = lambda y: shard.relu_forward_sparse_colsharded(  # noqa
            blocks, bblocks, y, w["clip"], device=dev, exchange=args.exchange, peer=peer,
            plan=plan)
        host_rp, host_ci, host_v = (np.array(a) for a in Y0.extract())
        nnz0 = int(host_rp[-1])
    elif w["y0"] == "binary":
        model, Ws = build_model(sk, w)
        nnzW = [x.nnz() for x in Ws]
        Y0 = sk.gen_input_binary(m, Bl, kY_of(w), SEED, sample_offset=b0)
        run = lambda y: sk.relu_forward_sparse(model, y, sk.ForwardOptions(clip=w["clip"]))  # noqa
        host_rp, host_ci, host_v = (np.array(a) for a in Y0.extract())
        nnz0 = int(host_rp[-1])
        layer1 = layer1_products(Ws[0], host_rp)
        del Ws
    else:
        model, Ws = build_model(sk, w)
        nnzW = [x.nnz() for x in Ws]
        Y0 = sk.gen_input_dense(m, Bl, SEED)
        run = lambda y: (sk.relu_forward(model, y, sk.ForwardOptions(clip=w["clip"])), None)  # noqa
        host_y = Y0.numpy()
        nnz0 = m * Bl
    torch.cuda.synchronize()
    sampler = ClockSampler(local)  # NVML initialised well before the timed region

    trace = None
    for _ in range(args.warmup):
        out, trace = run(Y0)
        del out
    R.barrier()

    # ---- timed region: resident inputs ----------------------------------------------
    ctx.set_timing(True)
    ctx.kernel_times_tagged()
    launches0 = sk._lib.launches()
    if rank == 0:  # where a launch list (ncu -s) of the timed region starts
        print(f"bench: {launches0} library launches before the timed region", file=sys.stderr)
    res = {}

    def step():
        out, res["trace"] = run(Y0)
        del out

    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/ (launch lists)
    with sampler as clocks:
        ms_max = timed_steps(R, stream, args.steps, step)
    torch.cuda.nvtx.range_pop()
    trace = res.get("trace", trace)
    launches = sk._lib.launches() - launches0
    ktimes, ktags = ctx.kernel_times_tagged()
    ctx.set_timing(False)
    ms_step = ms_max / args.steps
    edges = edges_per_inference(w, job_batch)
    value = edges / (ms_step / 1e3)

    # ---- e2e: host buffers in, result read back, through the public API ---------------
    if w["y0"] == "binary":
        # Y0 is binary: only its pattern crosses the host link (sk_csr_from_pattern);
        # with <= 65536 samples its column indices travel as 16-bit words
        # (sk_csr_from_pattern16_async: half the bytes, widened on the device)
        assert np.all(host_v == 1.0), "pattern upload needs a binary Y0"
        ncols = Y0.cols()
        narrow = ncols <= 65536
        up_ci = host_ci.astype(np.uint16) if narrow else host_ci
        for a in (host_rp, up_ci):
            sk._lib.load().sk_host_register(a.ctypes.data, a.nbytes)
        h2d = host_rp.nbytes + up_ci.nbytes
        copy_stream = torch.cuda.Stream(device=local)

        def upload():
            # on a copy stream: overlaps the forward already queued on the compute stream
            if narrow:
                return sk.CsrMatrix.from_pattern16_async(m, ncols, host_rp, up_ci, 1.0,
                                                         stream=copy_stream.cuda_stream)
            return sk.CsrMatrix.from_pattern_async(m, ncols, host_rp, up_ci, 1.0,
                                                   stream=copy_stream.cuda_stream)

        # steady-state input pipeline: every step issues exactly one upload (the
        # input of the step E2E_DEPTH ahead) before its own forward, so a timed
        # region of K steps holds K uploads and K forwards; the inputs of its
        # first E2E_DEPTH steps were issued during warm-up and the last E2E_DEPTH
        # uploads feed the steps after the region -- the region's closing
        # synchronize still waits for them (same work, no pipeline fill or drain)
        pending = collections.deque()

        def e2e_step():
            while len(pending) < E2E_DEPTH:  # first call only: fill the pipeline
                pending.append(upload())
            pending.append(upload())
            y = pending.popleft()
            out, tr = run(y)
            cats = sk.categories(out)
            return cats.nbytes + 8 * (L + 1)
    else:
        sk._lib.load().sk_host_register(host_y.ctypes.data, host_y.nbytes)
        h2d = host_y.nbytes
        out_host = np.empty_like(host_y)
        sk._lib.load().sk_host_register(out_host.ctypes.data, out_host.nbytes)

        def e2e_step():
            sk.relu_forward_host(model, host_y, sk.ForwardOptions(clip=w["clip"]), out=out_host)
            return out_host.nbytes
    for _ in range(max(1, args.warmup)):
        e2e_step()
    d2h = [0]

    def e2e_timed():
        d2h[0] = e2e_step()

    t0 = time.perf_counter()
    e2e_ms = timed_steps(R, stream, args.steps, e2e_timed)
    e2e_wall = R.max_over_ranks((time.perf_counter() - t0) * 1e3)
    e2e_step_ms = max(e2e_ms, e2e_wall) / args.steps
    e2e_value = edges / (e2e_step_ms / 1e3)
    # the host link alone: the same per-step input uploads back to back (what the
    # overlapped e2e step cannot go below)
    h2d_ms = None
    if w["y0"] == "binary":
        pending.clear()  # the inputs still in flight go back to the pool first
        torch.cuda.synchronize()
        upload()  # the pool now holds one input's worth of free blocks
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record(copy_stream)
        for _ in range(args.steps):
            upload()  # released at once: the next upload reuses its blocks
        ev1.record(copy_stream)
        torch.cuda.synchronize()
        h2d_ms = ev0.elapsed_time(ev1) / args.steps

    # ---- roofline of the dominant kernel ---------------------------------------------
    pk, pk_kind = peaks()
    tr = [int(x) for x in trace] if trace is not None else [nnz0] * (L + 1)
    paths = ctx.layer_paths(L) if not cols else []
    kt = np.array(ktimes, np.float64)
    roof = None
    if len(kt):
        by_kernel = {}
        for t_, g_ in zip(kt, ktags):
            by_kernel[g_] = by_kernel.get(g_, 0.0) + float(t_) / args.steps
        dom = max(by_kernel, key=by_kernel.get)
        t_dom = by_kernel[dom] / 1e3  # s per inference
        if cols:
            mg = shard.block_range(m, world, rank)[1] - shard.block_range(m, world, rank)[0]
            nnzb = [x.nnz() for x in blocks]
            byts = sum(sparse_layer_bytes(tr[k], tr[k + 1] * mg // m, Bl, mg, nnzb[k])
                       for k in range(L) if tr[k] > 0)
            desc = "this rank's output-neuron block per layer (k_exact_layer / k_spgemm_rows)"
        elif dom in ("k_exact_layer", "k_exact_stream"):
            byts = sum(sparse_layer_bytes(tr[k], tr[k + 1], Bl, m, nnzW[k])
                       for k in range(L) if paths[k] == "exact")
            desc = ("k_exact_layer (order-free fixed-point windowed SpGEMM + bias/ReLU/clip + "
                    "prune; its partial sums provably exact)" if dom == "k_exact_layer" else
                    "k_exact_stream (K7: order-free fixed-point SpGEMM, one output row per "
                    "warp, in-edge slices of a padded Y streamed as coalesced 16-byte units "
                    "into shared-memory 8-bit counters + bias/ReLU/clip + prune; partial sums "
                    "provably exact)")
        elif dom == "k_dense_engine":
            byts = sum(dense_layer_bytes(Bl, m, nnzW[k]) for k in range(L)
                       if w["y0"] == "dense" or paths[k] == "dense")
            desc = "k_dense_engine (per layer fused SpMM + bias/ReLU)"
        else:
            byts = sum(sparse_layer_bytes(tr[k], tr[k + 1], Bl, m, nnzW[k])
                       for k in range(L) if paths and paths[k] in ("engine",))
            desc = dom
        achieved = byts / t_dom / 1e9 if t_dom > 0 else 0.0
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": None, "kernel": desc,
                "algorithmic_bytes": byts, "launch_ms": t_dom * 1e3,
                "kernel_share_of_step": float(t_dom * 1e3 / ms_step), "peak_kind": pk_kind,
                "timed_kernels_ms_per_step": by_kernel,
                "rest_of_step_ms": float(ms_step - t_dom * 1e3)}
        if paths:
            roof["layer_paths"] = {p_: paths.count(p_) for p_ in sorted(set(paths))}
        tb, trep, lim = measured_traffic(args.workload)
        roof["traffic"] = tb
        roof["traffic_source"] = trep
        if lim is not None and not cols:
            roof["measured_limiter"] = lim
    useful = useful_products(tr, paths, m, Bl, nnzW, layer1) if not cols else None

    # ---- sustained-work variant ---------------------------------------------------------
    sustained = None
    if args.sustained and w["y0"] == "binary" and not cols:
        del model
        sustained = run_sustained(sk, ctx, stream, R, args, pk, b0, Bl, Bg)

    # ---- CPU baseline on rank 0 at N=1: the reference on the full workload -------------
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            cores = cpu_cores()
            times, per_layer = cpu_reference_run(w, Bg, 1, 0, cores)
            cpu = {"value": edges_per_inference(w, Bg) / statistics.mean(times),
                   "unit": "edges/s", "cores": cores, "kind": "reference",
                   "sample": "one step of the " + cpu_sample_desc(w, cores, per_layer),
                   "ms_per_step": statistics.mean(times) * 1e3, "cpu": cpu_model()}
        except Exception as e:  # the reference library is test infrastructure
            cpu = {"value": None, "unit": "edges/s", "cores": cpu_cores(), "kind": "reference",
                   "sample": f"unavailable: {type(e).__name__}: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if (cols or strong) else "weak",
            "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded SplitMix64; BASELINE shapes/distributions)",
            "config": {"workload": w["desc"], "neurons": m, "layers": L,
                       "global_batch": job_batch, "per_gpu_batch": Bl,
                       "edges_per_inference": edges,
                       "parallelism": (f"column-sharded W x{world}, per-layer exchange of the "
                                       f"sparse activations ({args.exchange})" if cols else
                                       f"batch-row x{world} ({'strong' if strong else 'weak'}: "
                                       f"{Bl} samples/GPU), replicated W, no data-path "
                                       f"collective"),
                       "l2": "inputs larger than L2 (W %.2f GB + Y0 %.0f MB vs 126 MB L2)"
                             % (sum(nnzW) * 8 / 1e9, nnz0 * 8 / 1e6)},
            "nnz_trace": ([int(x) for x in trace[:6]] + (["..."] if len(trace) > 6 else [])
                          + [int(trace[-1])]) if trace is not None else None,
            "useful_products_per_s": (useful * (job_batch / Bl) / (ms_step / 1e3)
                                      if useful is not None else None),
            "useful_products_note": ("edges/s counts every nominal MAC nnz(W)·B·L; the network "
                                     "as specified dies after 1-2 layers (SURVEY F5), so this "
                                     "counts the multiply-adds the forward needs (layer 1 exact, "
                                     "later layers nnz(Y_k)·nnz(W_k)/N); see `sustained` for a "
                                     "workload where every layer works"),
            "roofline": roof,
            "sustained": sustained,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "edges/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h[0]), "ms_per_step": e2e_step_ms,
                    "h2d_ms_per_step_alone": h2d_ms,
                    "input_upload": (f"steady-state pipeline, {E2E_DEPTH} inputs in flight: "
                                     "every step issues one pattern upload (copy stream, "
                                     "sk_csr_from_pattern16_async: row_ptr + 16-bit column "
                                     "indices, widened on the device) for the step "
                                     f"{E2E_DEPTH} ahead, then runs its own forward and reads "
                                     "the categories back; K timed steps = K uploads + K "
                                     "forwards + K read-backs, all waited for inside the "
                                     "timed region" if w["y0"] == "binary" else
                                     "synchronous per step (sk_relu_forward_host)")},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N>1 batch-row sharding: split the one global batch (strong, "
                         "BASELINE cfg4) or give every GPU its own full batch (weak)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sustained", dest="sustained", action="store_false",
                    help="skip the sustained-work (saturated cfg3) object")
    ap.add_argument("--shard", default="rows", choices=["rows", "cols"],
                    help="N>1 decomposition: batch-row sharding with replicated W (default, no "
                         "data-path collective) or column sharding of W_k with a per-layer "
                         "exchange of the sparse activations (BASELINE cfg5's layout)")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="--shard cols: per-layer exchange of the sparse row blocks by peer-memory "
                         "stores (one kernel per rank, CUDA IPC over NVLink) or padded NCCL "
                         "all-gathers")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
