"""K7's view of Y under each layout (sk_tuning.exact_layout: 2 in place, 1 padded copy,
3 padded copy with bank-ordered pass slices): layer-1 forward time (CUDA events on the
library's stream), K7 time (tagged), and the outputs compared across layouts, at the bench
bias and at a bias with many survivors.  python tools/bank_layout.py [cfg4 cfg3 cfg5]"""
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
    reps = 10
    for name in (sys.argv[1:] or ["cfg4", "cfg3", "cfg5"]):
        w = bench.WORKLOADS[name]
        W0 = sk.gen_layer_fixed(w["m"], w["kW"], sk.layer_seed(bench.SEED, 0), w["value"])
        B = int(os.environ.get("SB_BATCH", w["B"]))
        Y0 = sk.gen_input_binary(w["m"], B, bench.kY_of(w), bench.SEED)
        opt = sk.ForwardOptions(clip=w["clip"])
        for bias in (w["bias"], -0.12):
            model = sk.DnnModel([W0], [np.full(w["m"], bias, np.float32)])
            res, ref = {}, None
            for lay in (2, 1, 3):
                ctx.set_tuning(exact_kernel=5, exact_layout=lay)
                with torch.cuda.stream(s):
                    for _ in range(3):
                        out = sk.relu_forward_sparse(model, Y0, opt)
                    got = out[0].extract()
                    ctx.set_timing(True)
                    ctx.kernel_times_tagged()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    for _ in range(reps):
                        sk.relu_forward_sparse(model, Y0, opt)
                    e1.record(s)
                    e1.synchronize()
                    kt, tags = ctx.kernel_times_tagged()
                    ctx.set_timing(False)
                info = ctx.last_exact()
                if ref is None:
                    ref = got
                same = all(np.array_equal(np.asarray(a), np.asarray(b)) for a, b in zip(ref, got))
                res[f"layout{lay}"] = {"ran": info["layout"], "fields": info["fields"],
                                      "fwd_ms": round(e0.elapsed_time(e1) / reps, 4),
                                      "k7_ms": round(float(np.sum(kt)) / reps, 4),
                                      "nnz": int(len(got[1])), "same_as_first": bool(same)}
            ctx.set_tuning(exact_kernel=0, exact_layout=0)
            print(json.dumps({name: {"bias": bias, **res}}), flush=True)


if __name__ == "__main__":
    main()
