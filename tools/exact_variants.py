"""Layer-1 kernel time of the bench workloads under each exact-layer kernel
(sk_tuning.exact_kernel: 1 generic, 2 specialised, 3 push, 4 flat), tagged
CUDA-event timing.  python tools/exact_variants.py [cfg4 cfg3 cfg5]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    ctx = sk.default_context()
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    for name in (sys.argv[1:] or ["cfg4", "cfg3", "cfg5"]):
        w = bench.WORKLOADS[name]
        W0 = sk.gen_layer_fixed(w["m"], w["kW"], sk.layer_seed(bench.SEED, 0), w["value"])
        model = sk.DnnModel([W0], [np.full(w["m"], w["bias"], np.float32)])
        Y0 = sk.gen_input_binary(w["m"], w["B"], bench.kY_of(w), bench.SEED)
        opt = sk.ForwardOptions(clip=w["clip"])
        res = {}
        for kern in (2, 4, 1, 3):
            ctx.set_tuning(exact_kernel=kern)
            for _ in range(2):
                sk.relu_forward_sparse(model, Y0, opt)
            ctx.set_timing(True)
            ctx.kernel_times_tagged()
            for _ in range(5):
                sk.relu_forward_sparse(model, Y0, opt)
            kt, tags = ctx.kernel_times_tagged()
            ctx.set_timing(False)
            res[ctx.last_exact()["kernel"]] = round(float(np.sum(kt)) / 5, 4)
        ctx.set_tuning(exact_kernel=0)
        print(json.dumps({name: res}), flush=True)


if __name__ == "__main__":
    main()
