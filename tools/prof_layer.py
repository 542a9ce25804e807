"""Profiling driver: the cfg3/cfg4 construction with few layers, so one
k_sparse_engine launch is dominated by layer 1 (the only layer with work in
the as-specified BASELINE configs).  Used under ncu; prints nothing useful
on its own beyond timings."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_02937_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg4", choices=["cfg3", "cfg4", "cfg5"])
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--batch", type=int, default=60000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--skip", type=int, default=0,
                help="run the first SKIP layers once, then profile the rest on their output")
a = ap.parse_args()
m, dens, bias = {"cfg3": (16384, 0.015, -0.3), "cfg4": (65536, 0.004, -0.35),
                  "cfg5": (262144, 0.001, -0.45)}[a.workload]
Ws = [sk.gen_layer_fixed(m, 32, sk.layer_seed(42, k), 1.0 / 16) for k in range(a.layers)]
model = sk.DnnModel(Ws, [np.full(m, bias, np.float32)] * a.layers)
Y0 = sk.gen_input_binary(m, a.batch, int(round(dens * m)), 42)
if a.skip:
    pre = sk.DnnModel(Ws[:a.skip], [np.full(m, bias, np.float32)] * a.skip)
    Y0, _ = sk.relu_forward_sparse(pre, Y0, sk.ForwardOptions(clip=32.0))
    model = sk.DnnModel(Ws[a.skip:], [np.full(m, bias, np.float32)] * (a.layers - a.skip))
ctx = sk.default_context()
ctx.set_timing(True)
for r in range(a.reps):
    t = time.perf_counter()
    out, trace = sk.relu_forward_sparse(model, Y0, sk.ForwardOptions(clip=32.0))
    kt = ctx.kernel_times_ms()
    st = ctx.layer_stamps_ns(a.layers - a.skip + 1).astype(np.float64)
    per = np.round(np.diff(st) / 1e3, 1).tolist()
    print(f"rep {r}: wall {1e3 * (time.perf_counter() - t):.2f} ms kernels {[round(float(x), 3) for x in kt]} ms "
          f"trace {[int(x) for x in trace][:8]} layer_us {per[:8]}", flush=True)
