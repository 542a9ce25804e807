"""Where the GPU idles in the bench's resident-input step (cfg4): per call, the
Python wall time of relu_forward_sparse (+ releasing its result) against the
device time of the same calls (CUDA events), and, with SK_HOST_PROF=1, the C
side's split (printed every 20 calls; the first 20 include the warm-up).
python tools/host_gap.py [cfg4] [batch] [tuning key=value ...]"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    w = dict(bench.WORKLOADS[name])
    B = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else w["B"]
    tune = {k: int(v) for k, v in (a.split("=") for a in sys.argv[3:])}
    ctx = sk.default_context()
    ctx.set_tuning(**tune)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    model, Ws = bench.build_model(sk, w)
    del Ws
    Y0 = sk.gen_input_binary(w["m"], B, bench.kY_of(w), bench.SEED)
    opt = sk.ForwardOptions(clip=w["clip"])
    for _ in range(20):  # warm-up: the first SK_HOST_PROF line
        out, _ = sk.relu_forward_sparse(model, Y0, opt)
        del out
    torch.cuda.synchronize()
    wall, dev = [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(20):
        e0.record(s)
        t0 = time.perf_counter()
        out, _ = sk.relu_forward_sparse(model, Y0, opt)
        del out
        t1 = time.perf_counter()
        e1.record(s)
        torch.cuda.synchronize()
        wall.append((t1 - t0) * 1e6)
        dev.append(e0.elapsed_time(e1) * 1e3)
    # back to back, as the bench times them
    torch.cuda.synchronize()
    e0.record(s)
    t0 = time.perf_counter()
    for _ in range(20):
        out, _ = sk.relu_forward_sparse(model, Y0, opt)
        del out
    e1.record(s)
    torch.cuda.synchronize()
    b2b_dev = e0.elapsed_time(e1) * 1e3 / 20
    b2b_wall = (time.perf_counter() - t0) * 1e6 / 20
    # the Python layer alone: option struct + trace array + wrapper, no library call
    t0 = time.perf_counter()
    for _ in range(1000):
        sk.ForwardOptions(clip=w["clip"])._c()
    opt_us = (time.perf_counter() - t0) * 1e3
    ctx.set_timing(True)
    ctx.kernel_times_tagged()
    out, _ = sk.relu_forward_sparse(model, Y0, opt)
    del out
    kt, tags = ctx.kernel_times_tagged()
    ctx.set_timing(False)
    print(json.dumps({"workload": name, "batch": B, "tuning": tune, "layout": ctx.last_exact()["layout"],
                      "wall_us_median": round(statistics.median(wall), 1),
                      "dev_us_median": round(statistics.median(dev), 1),
                      "b2b_dev_us": round(b2b_dev, 1), "b2b_wall_us": round(b2b_wall, 1),
                      "options_us": round(opt_us, 2),
                      "kernels_us": {t: round(float(x) * 1e3, 1) for x, t in zip(kt, tags)}}))


if __name__ == "__main__":
    main()
