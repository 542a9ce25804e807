"""Runs the bench's layer 1 (cfg3/4/5) a few times under one exact-layer tuning:
the driver for ncu captures of a single exact-layer kernel.
python tools/prof_exact.py cfg4 exact_kernel=5 exact_group=32"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    name = sys.argv[1]
    tune = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
    ctx = sk.default_context()
    w = bench.WORKLOADS[name]
    W0 = sk.gen_layer_fixed(w["m"], w["kW"], sk.layer_seed(bench.SEED, 0), w["value"])
    Y0 = sk.gen_input_binary(w["m"], w["B"], bench.kY_of(w), bench.SEED)
    L = int(os.environ.get("PE_LAYERS", "1"))
    Ws = [W0] + [sk.gen_layer_fixed(w["m"], w["kW"], sk.layer_seed(bench.SEED, k), w["value"]) for k in range(1, L)]
    model = sk.DnnModel(Ws, [np.full(w["m"], w["bias"], np.float32)] * L)
    ctx.set_tuning(**tune)
    for _ in range(3):
        out, _ = sk.relu_forward_sparse(model, Y0, sk.ForwardOptions(clip=w["clip"]))
    print(name, tune, ctx.last_exact(), out.nnz())


if __name__ == "__main__":
    main()
