"""Timeline of the bench's end-to-end loop (cfg4): per step the pattern upload on
the copy stream and the forward on the compute stream, as CUDA events (ms from
the first event).  python tools/e2e_timeline.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    w = bench.WORKLOADS["cfg4"]
    m = w["m"]
    ctx = sk.default_context()
    cs = torch.cuda.Stream()
    ctx.set_stream(cs.cuda_stream)
    up = torch.cuda.Stream()
    Ws = [sk.gen_layer_fixed(m, w["kW"], sk.layer_seed(bench.SEED, k), w["value"]) for k in range(3)]
    model = sk.DnnModel([Ws[min(k, 2)] for k in range(w["L"])], [np.full(m, w["bias"], np.float32)] * w["L"])
    Y0 = sk.gen_input_binary(m, w["B"], bench.kY_of(w), bench.SEED)
    rp, ci, _ = Y0.extract()
    ci16 = ci.astype(np.uint16)
    for a in (rp, ci16):
        sk._lib.load().sk_host_register(a.ctypes.data, a.nbytes)
    opt = sk.ForwardOptions(clip=w["clip"])
    ev = []

    def mark(stream, tag):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        ev.append((tag, e))

    def upload():
        mark(up, "up0")
        y = sk.CsrMatrix.from_pattern16_async(m, Y0.cols(), rp, ci16, 1.0, stream=up.cuda_stream)
        mark(up, "up1")
        return y

    pending = [upload()]
    for s in range(steps):
        y = pending.pop()
        if s + 1 < steps:
            pending.append(upload())
        mark(cs, f"f0.{s}")
        out, tr = sk.relu_forward_sparse(model, y, opt)
        sk.categories(out)
        mark(cs, f"f1.{s}")
    torch.cuda.synchronize()
    t0 = ev[0][1]
    for tag, e in ev:
        print(f"{tag:8s} {t0.elapsed_time(e):9.3f}")


if __name__ == "__main__":
    main()
