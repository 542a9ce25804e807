"""Host-side cost of the calls in the bench's end-to-end step (cfg4 shapes):
wall time of each call from Python, median of 20."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    w = bench.WORKLOADS["cfg4"]
    m = w["m"]
    ctx = sk.default_context()
    cs = torch.cuda.Stream()
    ctx.set_stream(cs.cuda_stream)
    up = torch.cuda.Stream()
    Y0 = sk.gen_input_binary(m, w["B"], bench.kY_of(w), bench.SEED)
    rp, ci, _ = Y0.extract()
    ci16 = ci.astype(np.uint16)
    for a in (rp, ci16, ci):
        sk._lib.load().sk_host_register(a.ctypes.data, a.nbytes)
    res = {}
    for name, fn in (("pattern16_async", lambda: sk.CsrMatrix.from_pattern16_async(
                         m, Y0.cols(), rp, ci16, 1.0, stream=up.cuda_stream)),
                     ("pattern_async", lambda: sk.CsrMatrix.from_pattern_async(
                         m, Y0.cols(), rp, ci, 1.0, stream=up.cuda_stream)),
                     ("categories", lambda: sk.categories(Y0))):
        ts = []
        for _ in range(20):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x = fn()
            ts.append((time.perf_counter() - t0) * 1e6)
            torch.cuda.synchronize()
            del x
        res[name] = round(statistics.median(ts), 1)
    print(res)


if __name__ == "__main__":
    main()
