"""Timeline of one bench step (relu_forward_sparse on a bench workload) with
torch.profiler/CUPTI: every kernel, memcpy and memset with its duration, plus
host wall time per call.  Diagnostic only (numbers under a profiler are never
bench values)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    w = bench.WORKLOADS[wl]
    ctx = sk.default_context()
    stream = torch.cuda.Stream()  # a real handle: 0 would mean the library's own stream
    ctx.set_stream(stream.cuda_stream)
    model, _ = bench.build_model(sk, w)
    Y0 = sk.gen_input_binary(w["m"], w["B"], bench.kY_of(w), bench.SEED)
    opts = sk.ForwardOptions(clip=w["clip"])
    for _ in range(3):
        sk.relu_forward_sparse(model, Y0, opts)
    torch.cuda.synchronize()
    walls = []
    for _ in range(5):
        t0 = time.perf_counter()
        sk.relu_forward_sparse(model, Y0, opts)
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
    print("wall ms per call", [round(x, 3) for x in walls])
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            sk.relu_forward_sparse(model, Y0, opts)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start if evs else 0
    for e in evs:
        print(f"{(e.time_range.start - t0) / 1e3:9.3f} ms  {e.time_range.elapsed_us() / 1e3:8.3f} ms  {e.name[:90]}")


if __name__ == "__main__":
    main()
