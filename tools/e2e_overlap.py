"""What slows the forward when the next step's upload runs beside it (cfg4):
device time of the forward (+ categories) and of K7 alone with (a) nothing on the
copy stream, (b) a plain pinned 31.7 MB cudaMemcpyAsync, (c) the library's
pattern16 upload (copy + widen + fill kernels), (d) the same from a helper thread.
python tools/e2e_overlap.py [workload]"""
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    w = bench.WORKLOADS[name]
    m = w["m"]
    ctx = sk.default_context()
    cs = torch.cuda.Stream()
    ctx.set_stream(cs.cuda_stream)
    up = torch.cuda.Stream()
    model, Ws = bench.build_model(sk, w)
    del Ws
    Y0 = sk.gen_input_binary(m, w["B"], bench.kY_of(w), bench.SEED)
    rp, ci, _ = Y0.extract()
    ci16 = ci.astype(np.uint16)
    for a in (rp, ci16):
        sk._lib.load().sk_host_register(a.ctypes.data, a.nbytes)
    opt = sk.ForwardOptions(clip=w["clip"])
    pin = torch.empty(ci16.nbytes, dtype=torch.uint8).pin_memory()
    dev = torch.empty(ci16.nbytes, dtype=torch.uint8, device="cuda")

    def lib_upload():
        return sk.CsrMatrix.from_pattern16_async(m, Y0.cols(), rp, ci16, 1.0, stream=up.cuda_stream)

    def plain_copy():
        with torch.cuda.stream(up):
            dev.copy_(pin, non_blocking=True)
        return None

    def threaded():
        box = []
        t = threading.Thread(target=lambda: box.append(lib_upload()))
        t.start()
        return (t, box)

    res = {}
    for mode, side in (("none", None), ("plain_copy", plain_copy), ("lib_upload", lib_upload),
                       ("lib_upload_thread", threaded)):
        for _ in range(3):
            out, _ = sk.relu_forward_sparse(model, Y0, opt)
            del out
        torch.cuda.synchronize()
        fw, host_side, k7 = [], [], []
        for _ in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ctx.set_timing(True)
            ctx.kernel_times_tagged()
            t0 = time.perf_counter()
            keep = side() if side else None
            t1 = time.perf_counter()
            e0.record(cs)
            out, _ = sk.relu_forward_sparse(model, Y0, opt)
            sk.categories(out)
            e1.record(cs)
            torch.cuda.synchronize()
            if isinstance(keep, tuple):
                keep[0].join()
            kt, tags = ctx.kernel_times_tagged()
            ctx.set_timing(False)
            fw.append(e0.elapsed_time(e1) * 1e3)
            host_side.append((t1 - t0) * 1e6)
            k7.append(sum(float(x) for x, t in zip(kt, tags) if t == "k_exact_stream") * 1e3)
            del out, keep
        res[mode] = {"forward_us": round(statistics.median(fw), 1),
                     "side_call_host_us": round(statistics.median(host_side), 1),
                     "k7_us": round(statistics.median(k7), 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
