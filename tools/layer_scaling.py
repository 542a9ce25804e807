"""Forward time against the number of layers for the cfg3/cfg4 construction:
the slope is the per-layer cost of the layers after the activations empty out."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_02937_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg4", choices=["cfg3", "cfg4", "cfg5"])
ap.add_argument("--layers", default="2,3,10,100,480")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--timing", type=int, default=0, help="ctx.set_timing during the runs")
a = ap.parse_args()
m, dens, bias = {"cfg3": (16384, 0.015, -0.3), "cfg4": (65536, 0.004, -0.35),
                  "cfg5": (262144, 0.001, -0.45)}[a.workload]
Ls = [int(x) for x in a.layers.split(",")]
Ws = [sk.gen_layer_fixed(m, 32, sk.layer_seed(42, k), 1.0 / 16) for k in range(max(Ls))]
Y0 = sk.gen_input_binary(m, 60000, int(round(dens * m)), 42)
ctx = sk.default_context()
stream = torch.cuda.Stream()  # a real handle: 0 would mean the library's own stream
ctx.set_stream(stream.cuda_stream)
ctx.set_timing(bool(a.timing))
for L in Ls:
    model = sk.DnnModel(Ws[:L], [np.full(m, bias, np.float32)] * L)
    for _ in range(2):
        out, tr = sk.relu_forward_sparse(model, Y0, sk.ForwardOptions(clip=32.0))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.reps):
        out, tr = sk.relu_forward_sparse(model, Y0, sk.ForwardOptions(clip=32.0))
    e1.record(stream)
    torch.cuda.synchronize()
    kt = ctx.kernel_times_ms() if a.timing else None
    print(f"L={L:4d}  {e0.elapsed_time(e1) / a.reps:.3f} ms/forward  trace[:4]={list(tr)[:4]}  "
          f"kernels={kt}", flush=True)
    if a.timing:
        st = np.asarray(ctx.layer_stamps_ns(L + 1), np.int64)
        print("  layer stamps (us from stamp 0):", ((st[:6] - st[0]) / 1e3).round(1).tolist(),
              "last:", (st[-1] - st[0]) / 1e3, flush=True)
