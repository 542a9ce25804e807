#!/usr/bin/env python
"""Benchmark of the sparse ReLU DNN inference path (Y_{k+1} = ReLU(Y_k W_k + b_k)).

Default workload: BASELINE.json configs[3] ("cfg4"), the configuration the
metric is quoted on at 1/2/4/8 GPUs: 480 layers, N = 65536 neurons, W_k with
exactly 32 nonzeros per row (value 1/16), bias -0.35, ReLU clipped at 32,
Y0 binary with round(0.4% * N) = 262 active neurons per sample, 60000 samples
per GPU (batch-row sharding, replicated weights, no collective on the data
path: weak scaling -- rank r owns samples [60000 r, 60000 (r+1)) of the
global batch).  One step = one full 480-layer inference of the resident batch.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4|cfg3|cfg1]
    python bench.py --impl reference ...   # the reference's CPU path, rank 0 only

Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
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
                      "bias -0.35, ReLU clip 32, Y0 binary 0.4%/sample, 60000 samples/GPU"),
    "cfg3": dict(m=16384, L=120, B=60000, kW=32, value=1.0 / 16, bias=-0.3, clip=32.0,
                 y0="binary", density=0.015,
                 desc="BASELINE configs[2]: 120-layer sparse DNN, N=16384, 32 nnz/row (1/16), "
                      "bias -0.3, ReLU clip 32, Y0 binary 1.5%/sample, 60000 samples/GPU"),
    # Not a BASELINE config: the cfg3 network driven into its saturated regime
    # (Y0 50% ones -> every activation clips at 32 from layer 1 on), so every
    # layer carries full work.  Exercises the density-adaptive hand-off to the
    # dense engine; reported separately, never as the headline.
    "cfg3_saturated": dict(m=16384, L=120, B=60000, kW=32, value=1.0 / 16, bias=-0.3,
                           clip=32.0, y0="binary", density=0.5,
                           desc="sustained-work variant of BASELINE configs[2] (NOT a BASELINE "
                                "config): cfg3 network, Y0 binary 50%/sample -> activations "
                                "saturate (dense) from layer 1, 60000 samples/GPU"),
    "cfg5": dict(m=262144, L=120, B=60000, kW=32, value=1.0 / 16, bias=-0.45, clip=32.0,
                 y0="binary", density=0.001,
                 desc="BASELINE configs[4]: 120-layer sparse DNN, N=262144, 32 nnz/row (1/16), "
                      "bias -0.45, ReLU clip 32, Y0 binary 0.1%/sample, 60000 samples/GPU"),
    "cfg1": dict(m=1024, L=4, B=256, kW=16, value=float("nan"), bias=-0.05, clip=0.0,
                 y0="dense", density=1.0,
                 desc="BASELINE configs[0]: 4-layer sparse DNN, N=1024, 16 nnz/row U[-1,1), "
                      "bias -0.05, Y0 dense U[0,1), batch 256/GPU"),
}
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


DENSE_ABOVE, SPARSE_BELOW = 1.0 / 32, 1.0 / 128  # library defaults (sk_ctx_set_density_switch)


def layer_engines(trace, m, batch):
    """Replays the density-adaptive rule of relu_forward_sparse on an nnz trace:
    which engine ran each layer ("sparse" / "dense")."""
    full = m * batch
    hi, lo = max(1, int(DENSE_ABOVE * full)), int(SPARSE_BELOW * full)
    out, dense = [], False
    for k in range(len(trace) - 1):
        if not dense and trace[k] > hi:
            dense = True
        out.append("dense" if dense else "sparse")
        if dense and trace[k + 1] < lo:
            dense = False
        elif not dense and trace[k + 1] > hi:
            dense = True
    return out


def sparse_layer_bytes(nnz_in, nnz_out, batch, m, nnzW):
    """8 nnz(Y_k) + 8 nnz(Y_k+1) + 8(B+1) + 4(N+1) + 8 nnz(W) + 4N."""
    return 8 * nnz_in + 8 * nnz_out + 8 * (batch + 1) + 4 * (m + 1) + 8 * nnzW + 4 * m


def dense_layer_bytes(batch, m, nnzW):
    """8 B N + 4(N+1) + 8 nnz(W) + 4N."""
    return 8 * batch * m + 4 * (m + 1) + 8 * nnzW + 4 * m


def measured_traffic(workload):
    """Per-launch DRAM traffic of the dominant kernel from the committed ncu
    capture (profiles/r01/traffic.json) and the unit that binds it there, or None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r01", "traffic.json")))
        return t[workload]["bytes"], t[workload]["report"], t[workload].get("limiter")
    except Exception:
        return None, None, None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# ---------------------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation (oracle/_ref)

def cpu_reference_run(w, batch, layers_sampled, steps, warmup, workers, W_host=None):
    """Times the reference's CPU path on `batch` samples over `layers_sampled`
    layers: per layer the reference's mxm(CsrMatrix W_ref, CsrMatrix Y_ref)
    (proj/src/matrix.cpp:541-547, 452-521) followed by the layer epilogue the
    reference lacks (oracle/sk_oracle.c sko_sparse_epilogue); the dense-input
    config uses the reference's relu_forward (proj/src/dnn.cpp:111-121)."""
    from oracle.oracle import Port, Ref
    R, P = Ref.get(), Port.get()
    m = w["m"]
    b = np.full(m, w["bias"], np.float32)
    if W_host is None:
        W_host = [P.gen_layer_fixed(m, w["kW"], P.layer_seed(SEED, k), w["value"])
                  for k in range(layers_sampled)]
    times = []
    if w["y0"] == "dense":
        y0 = P.gen_input_dense(m, batch, SEED)
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            R.relu_forward(W_host[:layers_sampled], [b] * layers_sampled, y0, workers=workers)
            if it >= warmup:
                times.append(time.perf_counter() - t0)
        return times, [], W_host
    Y0 = P.gen_input_binary(m, batch, kY_of(w), SEED)
    hW = [R.handle(x) for x in W_host[:layers_sampled]]
    per_layer = []
    try:
        for it in range(warmup + steps):
            lt = []
            t0 = time.perf_counter()
            Y = Y0
            for k in range(layers_sampled):
                tl = time.perf_counter()
                hY = R.handle(Y)
                Z = R.take(R.mxm_csr_csr_h(hW[k], hY, workers=workers))
                R.free(hY)
                Y = P.sparse_epilogue(Z, b, w["clip"])
                lt.append(time.perf_counter() - tl)
            if it >= warmup:
                times.append(time.perf_counter() - t0)
                per_layer.append(lt)
    finally:
        for h in hW:
            R.free(h)
    return times, per_layer, W_host


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


def cpu_sample_plan(w):
    """Bounded CPU sample: a slice of the batch over every layer when that
    fits a few seconds per step, else the first 16 layers (then the empty-layer
    cost is extrapolated and the sample string says so)."""
    if w["y0"] == "dense":
        return w["B"], w["L"]
    return 600, min(w["L"], 16)


def extrapolate(w, per_layer_steps, layers_sampled):
    """Per-inference CPU time from a sampled prefix of layers: sampled layers as
    measured, the remaining layers at the median cost of the last sampled half."""
    tot = []
    for lt in per_layer_steps:
        tail = lt[layers_sampled // 2:] or lt
        tot.append(sum(lt) + (w["L"] - layers_sampled) * statistics.median(tail))
    return tot


def run_reference(args, w):
    rank, _, world = env_rank()
    if rank != 0:
        return
    batch, layers = cpu_sample_plan(w)
    cores = cpu_cores()
    times, per_layer, _ = cpu_reference_run(w, batch, layers, args.steps, args.warmup, cores)
    if per_layer and layers < w["L"]:
        times = extrapolate(w, per_layer, layers)
    t = statistics.mean(times)
    edges = edges_per_inference(w, batch)
    value = edges / t
    sample = (f"{batch} of {w['B']} samples/GPU, layers 1-{layers} of {w['L']} timed"
              + (f", remaining {w['L'] - layers} layers at the median cost of layers "
                 f"{layers // 2 + 1}-{layers}" if layers < w["L"] else "")
              + f"; reference mxm(CsrMatrix,CsrMatrix) workers={cores} + C epilogue"
              if w["y0"] != "dense" else f"full workload, reference relu_forward workers={cores}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": w["desc"], "cpu_batch": batch},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": cores,
                         "kind": "reference", "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# our arm

def run_ours(args, w):
    rank, local, world = env_rank()
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or (args.shard == "cols" and "MASTER_ADDR" in os.environ):
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1708_02937_b200 as sk
    sk.set_device(local)
    ctx = sk.default_context()
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)  # the library launches on torch's current stream

    m, L, B = w["m"], w["L"], w["B"]
    cols = args.shard == "cols" and w["y0"] == "binary"
    if cols:
        # column sharding: this rank owns output neurons [r0, r1) of every W_ref and
        # the whole batch; one all-gather of the sparse activations per layer
        from paper_1708_02937_b200 import shard
        dev = torch.device("cuda", local)
        r0, r1 = shard.block_range(m, world, rank)
        blocks, nnzW = [], []
        for k in range(L):
            wf = sk.gen_layer_fixed(m, w["kW"], sk.layer_seed(SEED, k), w["value"])
            nnzW.append(wf.nnz())
            blocks.append(shard.row_block(wf, r0, r1, dev))
            del wf
        bblocks = [np.full(r1 - r0, w["bias"], np.float32)] * L
        Y0 = sk.gen_input_binary(m, B, kY_of(w), SEED)
        # peer: one kernel per rank stores its block into every rank's next-layer
        # buffers over NVLink (CUDA IPC); nccl: padded NCCL all-gathers
        peer = shard.PeerExchange(m, ctx=sk.default_context()) if args.exchange == "peer" else None
        run = lambda y: shard.relu_forward_sparse_colsharded(  # noqa
            blocks, bblocks, y, w["clip"], device=dev, exchange=args.exchange, peer=peer)
        host_rp, host_ci, host_v = (np.array(a) for a in Y0.extract())
        nnz0 = int(host_rp[-1])
    elif w["y0"] == "binary":
        model, Ws = build_model(sk, w)
        nnzW = [x.nnz() for x in Ws]
        Y0 = sk.gen_input_binary(m, B, kY_of(w), SEED, sample_offset=rank * B)
        run = lambda y: sk.relu_forward_sparse(model, y, sk.ForwardOptions(clip=w["clip"]))  # noqa
        host_rp, host_ci, host_v = (np.array(a) for a in Y0.extract())
        nnz0 = int(host_rp[-1])
    else:
        model, Ws = build_model(sk, w)
        nnzW = [x.nnz() for x in Ws]
        Y0 = sk.gen_input_dense(m, B, SEED)
        run = lambda y: (sk.relu_forward(model, y, sk.ForwardOptions(clip=w["clip"])), None)  # noqa
        host_y = Y0.numpy()
        nnz0 = m * B
    torch.cuda.synchronize()
    sampler = ClockSampler(local)  # NVML initialised well before the timed region

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up
    trace = None
    for _ in range(args.warmup):
        out, trace = run(Y0)
        del out
    barrier()

    # ---- timed region: resident inputs ----------------------------------------------
    ctx.set_timing(True)
    launches0 = sk._lib.launches()
    if rank == 0:  # where a launch list (ncu -s) of the timed region starts
        print(f"bench: {launches0} library launches before the timed region", file=sys.stderr)
    with sampler as clocks:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            out, trace = run(Y0)
            del out
        e1.record(stream)
        barrier()
    launches = sk._lib.launches() - launches0
    ktimes = ctx.kernel_times_ms()
    ms = e0.elapsed_time(e1)
    t_local = torch.tensor([ms], device="cuda")
    if dist is not None:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_max = float(t_local.item())
    ms_step = ms_max / args.steps
    edges = edges_per_inference(w, B)
    job_edges = edges if cols else world * edges  # cols: all ranks share one batch
    value = job_edges / (ms_step / 1e3)

    ctx.set_timing(False)
    # ---- e2e: host buffers in, result read back, through the public API ---------------
    if w["y0"] == "binary":
        # Y0 is binary: only its pattern crosses the host link (sk_csr_from_pattern)
        assert np.all(host_v == 1.0), "pattern upload needs a binary Y0"
        for a in (host_rp, host_ci):
            sk._lib.load().sk_host_register(a.ctypes.data, a.nbytes)
        h2d = host_rp.nbytes + host_ci.nbytes
        copy_stream = torch.cuda.Stream()

        def upload():
            # on a copy stream: overlaps the forward already queued on the compute stream
            return sk.CsrMatrix.from_pattern_async(m, B, host_rp, host_ci, 1.0,
                                                   stream=copy_stream.cuda_stream)

        pending = []
        left = [0]  # steps still to run after this one (no upload beyond the last)

        def e2e_step():
            # double-buffered input: step s+1's upload is issued before step s's
            # forward, so the host link and the GPU work overlap; every step's
            # copy still happens inside the timed region
            y = pending.pop() if pending else upload()
            if left[0] > 0:
                pending.append(upload())
                left[0] -= 1
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
    if w["y0"] == "binary":
        left[0] = max(1, args.warmup) - 1
    for _ in range(max(1, args.warmup)):
        e2e_step()
    if w["y0"] == "binary":
        left[0] = args.steps - 1  # the timed region uploads its own inputs
    barrier()
    t0 = time.perf_counter()
    e0.record(stream)
    d2h = 0
    for _ in range(args.steps):
        d2h = e2e_step()
    e1.record(stream)
    barrier()
    e2e_wall = (time.perf_counter() - t0) * 1e3
    e2e_ms = max(e0.elapsed_time(e1), e2e_wall)
    t_e2e = torch.tensor([e2e_ms], device="cuda")
    if dist is not None:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_step_ms = float(t_e2e.item()) / args.steps
    e2e_value = job_edges / (e2e_step_ms / 1e3)

    # ---- roofline of the dominant kernel ---------------------------------------------
    pk, pk_kind = peaks()
    tr = [int(x) for x in trace] if trace is not None else [nnz0] * (L + 1)
    roof = None
    if cols and len(ktimes):
        # per layer: this rank's block SpGEMM + epilogue (k_spgemm_rows); bytes =
        # SURVEY §8(d) with the block's rows and weights, the full input Y_k
        mg = r1 - r0
        nnzb = [x.nnz() for x in blocks]
        byts = sum(sparse_layer_bytes(tr[k], tr[k + 1] * mg // m, B, mg, nnzb[k])
                   for k in range(L) if tr[k] > 0)
        t_launch = float(np.sum(ktimes)) / args.steps / 1e3
        achieved = byts / t_launch / 1e9 if t_launch > 0 else 0.0
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": None,
                "kernel": "k_spgemm_rows (per layer, this rank's output-neuron block)",
                "algorithmic_bytes": byts, "launch_ms": t_launch * 1e3,
                "launches_per_inference": len(ktimes) / args.steps,
                "kernel_share_of_step": float(t_launch * 1e3 / ms_step), "peak_kind": pk_kind}
    elif w["y0"] == "binary" and len(ktimes):
        # Per inference: layer 1 on the order-free fixed-point path (k_exact_layer,
        # its partial sums provably exact) when the statistics allow it, then the
        # thin layers on expand-sort-compress, the windowed engine or the dense
        # engine (ctx.layer_paths).  The timed launches are k_exact_layer and one
        # per engine segment, in that order.  Algorithmic bytes per layer follow
        # SURVEY §8(d) for the representation it ran in.
        paths = ctx.layer_paths(L)
        per_step = len(ktimes) // args.steps if len(ktimes) % args.steps == 0 else 0
        path_count = {p_: paths.count(p_) for p_ in sorted(set(paths))}
        if paths[0] == "exact" and per_step >= 1:
            t1 = float(np.mean(ktimes[0::per_step])) / 1e3
            b1 = sparse_layer_bytes(tr[0], tr[1], B, m, nnzW[0])
            achieved = b1 / t1 / 1e9
            roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved / pk["hbm_gbs"], "traffic": None,
                    "kernel": "k_exact_layer (layer 1: order-free fixed-point windowed SpGEMM + "
                              "bias/ReLU/clip + prune; its partial sums provably exact)",
                    "algorithmic_bytes": b1, "launch_ms": t1 * 1e3, "launches_per_inference": 1,
                    "kernel_share_of_step": float(t1 * 1e3 / ms_step), "peak_kind": pk_kind,
                    "layer_paths": path_count,
                    "rest_of_step_ms": float(ms_step - t1 * 1e3)}
        else:
            eng = layer_engines(tr, m, B)
            byts = sum((sparse_layer_bytes(tr[k], tr[k + 1], B, m, nnzW[k]) if tr[k] > 0 else 0)
                       if eng[k] == "sparse" else dense_layer_bytes(B, m, nnzW[k])
                       for k in range(L))
            t_launch = float(np.sum(ktimes)) / args.steps / 1e3  # timed kernels per inference
            achieved = byts / t_launch / 1e9
            roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved / pk["hbm_gbs"], "traffic": None,
                    "kernel": "k_sparse_engine (persistent: per layer windowed SpGEMM + "
                              "bias/ReLU/clip + prune + compaction) / k_dense_engine",
                    "algorithmic_bytes": byts, "launch_ms": t_launch * 1e3,
                    "launches_per_inference": len(ktimes) / args.steps,
                    "kernel_share_of_step": float(t_launch * 1e3 / ms_step),
                    "peak_kind": pk_kind, "layer_paths": path_count}
    elif len(ktimes):
        # One launch of k_dense_engine per inference (all layers, grid barriers
        # between them): algorithmic bytes = SURVEY §8(d) dense-Y bytes per layer.
        byts = sum(dense_layer_bytes(B, m, nnzW[k]) for k in range(L))
        t_launch = float(np.mean(ktimes)) / 1e3
        achieved = byts / t_launch / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": None,
                "kernel": "k_dense_engine (persistent: per layer fused SpMM + bias/ReLU)",
                "algorithmic_bytes": byts, "launch_ms": t_launch * 1e3,
                "kernel_share_of_step": float(t_launch * 1e3 / ms_step),
                "peak_kind": pk_kind}

    # ---- CPU baseline on rank 0 at N=1 --------------------------------------------------
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            batch, layers = cpu_sample_plan(w)
            cores = cpu_cores()
            times, per_layer, _ = cpu_reference_run(w, batch, layers, 1, 0, cores)
            if per_layer and layers < L:
                times = extrapolate(w, per_layer, layers)
            cpu_v = edges_per_inference(w, batch) / statistics.mean(times)
            cpu = {"value": cpu_v, "unit": "edges/s", "cores": cores, "kind": "reference",
                   "sample": f"{batch} samples, {layers}/{L} layers timed"
                             + (" (rest extrapolated from the empty-layer median)"
                                if layers < L else "")
                             + "; reference CPU path (oracle/_ref)",
                   "cpu": cpu_model()}
        except Exception as e:  # the reference library is test infrastructure
            cpu = {"value": None, "unit": "edges/s", "cores": cpu_cores(), "kind": "reference",
                   "sample": f"unavailable: {type(e).__name__}: {e}"}

    if roof is not None:
        tb, trep, lim = measured_traffic(args.workload)
        roof["traffic"] = tb
        roof["traffic_source"] = trep
        if lim is not None and not cols:
            roof["measured_limiter"] = lim
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if cols else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded SplitMix64; BASELINE shapes/distributions)",
            "config": {"workload": w["desc"], "neurons": m, "layers": L,
                       "per_gpu_batch": B if not cols else B, "global_batch": B if cols else B * world,
                       "edges_per_inference_per_gpu": edges if not cols else edges // world,
                       "parallelism": (f"column-sharded W x{world}, per-layer exchange of the "
                                       f"sparse activations ({args.exchange})" if cols else
                                       f"batch-row x{world}, replicated W, no data-path collective"),
                       "l2": "inputs larger than L2 (W %.2f GB + Y0 %.0f MB vs 126 MB L2)"
                             % (sum(nnzW) * 8 / 1e9, nnz0 * 8 / 1e6)},
            "nnz_trace": ([int(x) for x in trace[:6]] + (["..."] if len(trace) > 6 else [])
                          + [int(trace[-1])]) if trace is not None else None,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "edges/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_step_ms,
                    "input_upload": ("double-buffered: step s+1's pattern upload (copy stream, "
                                     "sk_csr_from_pattern_async) overlaps step s's forward; "
                                     "every step's upload and result read inside the timed "
                                     "region" if w["y0"] == "binary" else
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="rows", choices=["rows", "cols"],
                    help="N>1 decomposition: batch-row sharding with replicated W (default, no "
                         "data-path collective) or column sharding of W_k with a per-layer "
                         "NCCL all-gather of the sparse activations (BASELINE cfg5's layout)")
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
