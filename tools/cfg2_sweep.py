"""BASELINE configs[1]: single-layer density sweep, sparse vs dense leg.

Y0 dense U[0,1) 4096 x 1024 (neuron-major), W 4096 x 4096 Bernoulli(d) with
U[-1,1) values, bias -0.05, ReLU.  Sparse leg: layer_step (K1, fused SpMM +
bias + ReLU, bitwise vs the reference).  Dense leg: dense_layer_step (K4,
pack + tcgen05 3xTF32 GEMM + bias + ReLU).  *_ms are the library's kernels
(CUDA events around each launch on its stream); *_call_ms the whole API call
(adds the host bias upload); medians of --reps after --warmup.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--densities", default="0.5,0.1,0.01,0.001,0.0001")
    a = ap.parse_args()
    import torch
    ctx = sk.default_context()
    stream = torch.cuda.Stream()  # a real handle: 0 would mean the library's own stream
    ctx.set_stream(stream.cuda_stream)
    m, n, seed = 4096, 1024, 42
    y = sk.gen_input_dense(m, n, seed)
    b = np.full(m, -0.05, np.float32)
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))

    def timed(fn):
        """(call ms, kernel ms): CUDA events around the whole API call (includes
        the host bias upload the reference signature implies) and the library's
        own kernel timing (sum of its timed launches per call)."""
        for _ in range(a.warmup):
            fn()
        ts, ks = [], []
        ctx.set_timing(True)
        ctx.kernel_times_ms()
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
            ks.append(float(np.sum(ctx.kernel_times_ms())))
        ctx.set_timing(False)
        return float(np.median(ts)), float(np.median(ks))

    for d in [float(x) for x in a.densities.split(",")]:
        W = sk.gen_layer_density(m, d, sk.layer_seed(seed, 0))
        Wm = sk.Matrix(W)
        nnz = W.nnz()
        t_sp_call, t_sp = timed(lambda: sk.layer_step(Wm, b, y))
        Wd = sk.to_dense(W, 0.0)
        t_de_call, t_de = timed(lambda: sk.dense_layer_step(Wd, b, y))
        edges = nnz * n
        sp_bytes = 8 * n * m + 4 * (m + 1) + 8 * nnz + 4 * m
        de_flops = 2.0 * m * m * n
        print(json.dumps({
            "density": d, "nnz": nnz,
            "sparse_call_ms": t_sp_call, "dense_call_ms": t_de_call,
            "sparse_ms": t_sp, "sparse_edges_per_s": edges / (t_sp / 1e3),
            "sparse_gbs_algorithmic": sp_bytes / (t_sp / 1e3) / 1e9,
            "sparse_frac_hbm": sp_bytes / (t_sp / 1e3) / 1e9 / peaks["hbm_gbs"],
            "sparse_fma_macs_per_s": edges / (t_sp / 1e3),
            "dense_ms": t_de, "dense_tflops_fp32_equiv": de_flops / (t_de / 1e3) / 1e12,
            "dense_tflops_tf32_issued": 3 * de_flops / (t_de / 1e3) / 1e12,
            "dense_over_sparse": t_de / t_sp}), flush=True)


if __name__ == "__main__":
    main()
