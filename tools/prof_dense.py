"""Diagnostic: the dense-activation engine on a saturated cfg3-shaped layer
(N=16384, 32 in-edges/row of 1/16, Y dense 32.0), for ncu captures and quick
timings.  python tools/prof_dense.py [batch] [layers] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 15000
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    m = 16384
    ctx = sk.default_context()
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    Ws = [sk.gen_layer_fixed(m, 32, sk.layer_seed(42, k), 1.0 / 16) for k in range(L)]
    model = sk.DnnModel(Ws, [np.full(m, -0.3, np.float32)] * L)
    y = sk.DenseMatrix(m, B, 32.0)
    opt = sk.ForwardOptions(clip=32.0)
    out = sk.relu_forward(model, y, opt)
    ctx.set_timing(True)
    ctx.kernel_times_tagged()
    for _ in range(reps):
        out = sk.relu_forward(model, y, opt)
    ctx.synchronize()
    kt, tags = ctx.kernel_times_tagged()
    per = float(np.sum(kt)) / reps / L
    macs = m * 32 * B
    print(f"B={B} L={L}: {per:.3f} ms/layer, {macs / per / 1e9:.3f} TMAC/s, "
          f"L2->SM at 4 B/MAC {4 * macs / per / 1e9:.1f} GB/s; kernels {sorted(set(tags))}")
    del out


if __name__ == "__main__":
    main()
