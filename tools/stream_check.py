"""K7 (k_exact_stream) against the specialised windowed kernel on the bench's
layer 1: bitwise comparison of the outputs and tagged kernel times, per pass
width (exact_group = windows per pass) and staging size (exact_records).
python tools/stream_check.py [cfg4 cfg3 cfg5]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402


def run(ctx, model, Y0, opt, reps=5):
    for _ in range(2):
        out, _ = sk.relu_forward_sparse(model, Y0, opt)
    ctx.set_timing(True)
    ctx.kernel_times_tagged()
    for _ in range(reps):
        sk.relu_forward_sparse(model, Y0, opt)
    kt, tags = ctx.kernel_times_tagged()
    ctx.set_timing(False)
    ex = [t for t, g in zip(kt, tags) if g in ("k_exact_layer", "k_exact_stream")]
    return out, round(float(np.sum(ex)) / reps, 4), ctx.last_exact()


GROUPS = [int(x) for x in os.environ.get("SC_GROUPS", "0,1,2,4,8,16").split(",")]
RECS = [int(x) for x in os.environ.get("SC_RECS", "0").split(",")]
FIELDS = [int(x) for x in os.environ.get("SC_FIELDS", "0,8").split(",")]
KERNEL = int(os.environ.get("SC_KERNEL", "5"))


def main():
    ctx = sk.default_context()
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    for name in (sys.argv[1:] or ["cfg4", "cfg3", "cfg5"]):
        w = bench.WORKLOADS[name]
        W0 = sk.gen_layer_fixed(w["m"], w["kW"], sk.layer_seed(bench.SEED, 0), w["value"])
        Y0 = sk.gen_input_binary(w["m"], w["B"], bench.kY_of(w), bench.SEED)
        opt = sk.ForwardOptions(clip=w["clip"])
        for bias in (w["bias"], -0.1):
            model = sk.DnnModel([W0], [np.full(w["m"], bias, np.float32)])
            ctx.set_tuning(exact_kernel=2)
            ref, t_ref, _ = run(ctx, model, Y0, opt)
            rr = ref.extract()
            res = {"specialised": t_ref, "nnz": int(ref.nnz())}
            for grp in GROUPS:
                for fb in FIELDS:
                    ctx.set_tuning(exact_kernel=KERNEL, exact_group=grp, exact_fields=fb)
                    out, t, info = run(ctx, model, Y0, opt)
                    oo = out.extract()
                    same = all(np.array_equal(a.view(np.uint32), b.view(np.uint32))
                               for a, b in zip(oo, rr))
                    res[f"g{grp}f{fb}"] = [t, info["kernel"], info["group"], info["fields"],
                                          "OK" if same else "DIFF", info["wraps"]]
            ctx.set_tuning(exact_kernel=0, exact_group=0, exact_fields=0)
            print(json.dumps({name: {str(bias): res}}), flush=True)


if __name__ == "__main__":
    main()
