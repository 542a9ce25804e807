"""Phase timing of one column-sharded forward (torchrun, any world size):
local layer, device->torch copy, all-gather, handle rebuild.  Diagnostic only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402
from paper_1708_02937_b200 import shard  # noqa: E402
from paper_1708_02937_b200 import semikern as skm  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    w = bench.WORKLOADS[wl]
    rank, local, world = bench.env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    m, L, B = w["m"], 3, w["B"]
    r0, r1 = shard.block_range(m, world, rank)
    blocks = []
    for k in range(L):
        wf = sk.gen_layer_fixed(m, w["kW"], sk.layer_seed(bench.SEED, k), w["value"])
        blocks.append(shard.row_block(wf, r0, r1, dev))
        del wf
    b = np.full(r1 - r0, w["bias"], np.float32)
    Y0 = sk.gen_input_binary(m, B, bench.kY_of(w), bench.SEED)
    for it in range(3):
        t = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        local_y = skm.sparse_layer(blocks[0], b, Y0, w["clip"])
        torch.cuda.synchronize()
        t["layer"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        rp, ci, v = shard.csr_to_torch(local_y, dev)
        t["to_torch"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        frp, fci, fv = shard.allgather_csr_rows(rp, ci, v)
        torch.cuda.synchronize()
        t["allgather"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        nnz = int(frp[-1].item())
        frp32 = frp.to(torch.int32)
        torch.cuda.synchronize()
        y = skm.csr_from_device(m, B, nnz, frp32.data_ptr(), fci.data_ptr(), fv.data_ptr(),
                                ctx=Y0.ctx)
        y.ctx.synchronize()
        t["rebuild"] = time.perf_counter() - t0
        if rank == 0:
            print(it, {k: round(x * 1e3, 3) for k, x in t.items()}, "nnz", nnz)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
