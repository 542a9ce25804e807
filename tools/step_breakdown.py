"""Where the cfg4 step goes beyond layer 1: the forward timed (CUDA events on the
library's stream, warm) for the first L layers of the bench's network, L in
1, 2, 3, 480.  python tools/step_breakdown.py [cfg4]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    w = bench.WORKLOADS[name]
    ctx = sk.default_context()
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    Ws = [sk.gen_layer_fixed(w["m"], w["kW"], sk.layer_seed(bench.SEED, k), w["value"])
          for k in range(3)]
    B = int(os.environ.get("SB_BATCH", w["B"]))  # e.g. 7500: one GPU's share at N = 8
    Y0 = sk.gen_input_binary(w["m"], B, bench.kY_of(w), bench.SEED)
    opt = sk.ForwardOptions(clip=w["clip"])
    b = np.full(w["m"], w["bias"], np.float32)
    res = {}
    for L in (1, 2, 3, w["L"]):
        layers = [Ws[min(k, 2)] for k in range(L)]
        model = sk.DnnModel(layers, [b] * L)
        for _ in range(3):
            sk.relu_forward_sparse(model, Y0, opt)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(10):
            sk.relu_forward_sparse(model, Y0, opt)
        e1.record(s)
        torch.cuda.synchronize()
        res[L] = round(e0.elapsed_time(e1) / 10, 4)
        ctx.set_timing(True)
        ctx.kernel_times_tagged()
        sk.relu_forward_sparse(model, Y0, opt)
        kt, tags = ctx.kernel_times_tagged()
        ctx.set_timing(False)
        res[f"{L}_kernels"] = {t: round(float(x), 4) for x, t in zip(kt, tags)}
    print(json.dumps({name: res, "batch": B}))


if __name__ == "__main__":
    main()
