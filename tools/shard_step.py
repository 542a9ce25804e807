"""One rank's cfg4 step at N ranks (default 8 -> 7500 samples), inside an NVTX
range "timed" (for ncu --nvtx --nvtx-include timed/ launch lists), plus a
host-side wall-clock split of the forward. python tools/shard_step.py [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402
from paper_1708_02937_b200 import shard  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    w = bench.WORKLOADS["cfg4"]
    ctx = sk.default_context()
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    model, _ = bench.build_model(sk, w)
    opt = sk.ForwardOptions(clip=w["clip"])
    b0, Bl = shard.batch_shard(w["B"], N, 0)
    Y0 = sk.gen_input_binary(w["m"], Bl, bench.kY_of(w), bench.SEED, sample_offset=b0)
    for _ in range(3):
        sk.relu_forward_sparse(model, Y0, opt)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("timed")
    t0 = time.perf_counter()
    for _ in range(2):
        sk.relu_forward_sparse(model, Y0, opt)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print(f"N={N} samples={Bl}: {(time.perf_counter() - t0) / 2 * 1e3:.3f} ms per forward (wall)")


if __name__ == "__main__":
    main()
