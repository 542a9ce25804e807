"""Strong-scaling preview on one GPU: the cfg4 forward on one rank's shard of the
60000-sample batch for N = 1, 2, 4, 8 (7500 samples at N = 8), so the per-rank step
time and the implied efficiency T(1) / (N T(N)) can be read before a multi-GPU run.
python tools/shard_scaling.py [workload]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402
from paper_1708_02937_b200 import shard  # noqa: E402


def main():
    w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
    ctx = sk.default_context()
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    model, _ = bench.build_model(sk, w)
    opt = sk.ForwardOptions(clip=w["clip"])
    res = {}
    for N in (1, 2, 4, 8):
        b0, Bl = shard.batch_shard(w["B"], N, 0)
        Y0 = sk.gen_input_binary(w["m"], Bl, bench.kY_of(w), bench.SEED, sample_offset=b0)
        for _ in range(3):
            sk.relu_forward_sparse(model, Y0, opt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.set_timing(True)
        ctx.kernel_times_tagged()
        e0.record(s)
        reps = 10
        for _ in range(reps):
            sk.relu_forward_sparse(model, Y0, opt)
        e1.record(s)
        torch.cuda.synchronize()
        kt, tags = ctx.kernel_times_tagged()
        ctx.set_timing(False)
        ms = e0.elapsed_time(e1) / reps
        res[N] = {"samples": Bl, "ms_per_step": ms,
                  "kernels_ms": {t: float(sum(x for x, g in zip(kt, tags) if g == t)) / reps
                                 for t in sorted(set(tags))}}
    t1 = res[1]["ms_per_step"]
    for N in res:
        res[N]["efficiency_if_ranks_match"] = t1 / (N * res[N]["ms_per_step"])
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
