"""Multi-GPU execution of the sparse DNN forward pass (one process per GPU,
torch.distributed for the plumbing).

Two decompositions:

* Batch-row sharding (BASELINE cfg4, 1/2/4/8 GPUs): the samples (columns of
  the neuron-major Y) are split into contiguous shards; W is replicated; every
  sample's inference is independent, so the data path has NO collective.  The
  partition is the reference's static row-block rule count*w/nw
  (proj/src/detail/parallel.hpp:29-43).  Only the final category set is
  gathered.

* Column sharding of W_k (BASELINE cfg5, 8 GPUs): GPU g owns the output
  neurons J_g = rows [m g/G, m (g+1)/G) of every W_ref (= a column block of
  W_k), computes those rows of Y_{k+1} from the full Y_k, and one all-gather of
  the sparse row blocks per layer reassembles Y_{k+1} everywhere.  Row blocks
  concatenate into the full neuron-major CSR after a row-pointer offset, and
  every output row is computed exactly as on one GPU, so the result is
  bitwise identical to the single-GPU forward.

The collective helpers work on any torch.distributed backend (NCCL on the
GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def block_range(count: int, world: int, rank: int) -> tuple[int, int]:
    """[begin, end) of block `rank` of `count` items over `world` owners."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return count * rank // world, count * (rank + 1) // world


def batch_shard(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """(first sample, sample count) of this rank's batch-row shard."""
    b, e = block_range(global_batch, world, rank)
    return b, e - b


def _dist():
    import torch.distributed as dist
    return dist


def gather_categories(local_idx, sample_offset: int, device="cpu", group=None) -> np.ndarray:
    """Global sorted category set from every rank's local (shard-relative)
    indices.  Shards are disjoint contiguous sample ranges, so the union is a
    concatenation in rank order of (local + offset)."""
    import torch
    dist = _dist()
    world = dist.get_world_size(group)
    loc = torch.as_tensor(np.asarray(local_idx, np.int64) + int(sample_offset), device=device)
    n = torch.tensor([loc.numel()], dtype=torch.int64, device=device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    mx = max(1, max(int(x.item()) for x in ns))
    buf = torch.full((mx,), -1, dtype=torch.int64, device=device)
    buf[: loc.numel()] = loc
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.cat([p[: int(c.item())] for p, c in zip(parts, ns)])
    return np.sort(out.cpu().numpy())


def allgather_csr_rows(rp, ci, v, group=None):
    """All-gather of CSR row blocks (torch tensors on the collective's device;
    rp int64 rows_g+1 local offsets, ci int32, v float32) into the full CSR
    (rank order = row order).  Variable block sizes are exchanged as counts
    first, then padded to the largest block (NCCL has no all-gather-v)."""
    import torch
    dist = _dist()
    world = dist.get_world_size(group)
    dev = rp.device
    meta = torch.tensor([rp.numel() - 1, ci.numel()], dtype=torch.int64, device=dev)
    metas = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    rows = [int(m[0].item()) for m in metas]
    nnzs = [int(m[1].item()) for m in metas]
    maxr, maxn = max(rows), max(1, max(nnzs))

    def padded(t, n):
        out = torch.zeros(n, dtype=t.dtype, device=dev)
        out[: t.numel()] = t
        return out

    rp_l = [torch.empty(maxr + 1, dtype=torch.int64, device=dev) for _ in range(world)]
    ci_l = [torch.empty(maxn, dtype=ci.dtype, device=dev) for _ in range(world)]
    v_l = [torch.empty(maxn, dtype=v.dtype, device=dev) for _ in range(world)]
    dist.all_gather(rp_l, padded(rp.to(torch.int64), maxr + 1), group=group)
    dist.all_gather(ci_l, padded(ci, maxn), group=group)
    dist.all_gather(v_l, padded(v, maxn), group=group)
    off = 0
    rps, cis, vs = [], [], []
    for g in range(world):
        rps.append(rp_l[g][: rows[g]] + off)
        cis.append(ci_l[g][: nnzs[g]])
        vs.append(v_l[g][: nnzs[g]])
        off += nnzs[g]
    rps.append(torch.tensor([off], dtype=torch.int64, device=dev))
    return torch.cat(rps), torch.cat(cis), torch.cat(vs)


def csr_to_torch(a, device):
    """Copy a device CSR handle into torch tensors on `device` (D2D)."""
    import torch
    from . import semikern as skm
    rows, nnz = a.rows(), a.nnz()
    rp = torch.empty(rows + 1, dtype=torch.int32, device=device)
    ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=device)
    v = torch.empty(max(nnz, 1), dtype=torch.float32, device=device)
    p_rp, p_ci, p_v = skm.csr_device_arrays(a)
    skm.memcpy_d2d(rp.data_ptr(), p_rp, (rows + 1) * 4, ctx=a.ctx)
    if nnz:
        skm.memcpy_d2d(ci.data_ptr(), p_ci, nnz * 4, ctx=a.ctx)
        skm.memcpy_d2d(v.data_ptr(), p_v, nnz * 4, ctx=a.ctx)
    a.ctx.synchronize()
    return rp.to(torch.int64), ci[:nnz], v[:nnz]


def row_block(a, r0: int, r1: int, device):
    """Rows [r0, r1) of a device CSR as a new handle (device-side slice)."""
    import torch
    from . import semikern as skm
    rp, ci, v = csr_to_torch(a, device)
    e0, e1 = int(rp[r0].item()), int(rp[r1].item())
    brp = (rp[r0:r1 + 1] - e0).to(torch.int32).contiguous()
    bci = ci[e0:e1].contiguous() if e1 > e0 else torch.zeros(1, dtype=torch.int32, device=device)
    bv = v[e0:e1].contiguous() if e1 > e0 else torch.zeros(1, dtype=torch.float32, device=device)
    torch.cuda.synchronize(device)
    out = skm.csr_from_device(r1 - r0, a.cols(), e1 - e0, brp.data_ptr(), bci.data_ptr(),
                              bv.data_ptr(), ctx=a.ctx)
    out.ctx.synchronize()
    return out


def relu_forward_sparse_colsharded(w_blocks, b_blocks, y0, clip=0.0, group=None, device=None):
    """Column-sharded sparse forward pass.  `w_blocks[k]` is this rank's block
    of output-neuron rows of W_ref[k] (a CsrMatrix m_g x m), `b_blocks[k]` its
    bias slice, `y0` the full m x n input (replicated).  Returns (Y_L, trace).
    Per layer: local block SpGEMM + epilogue on the GPU (sk_sparse_layer: the
    order-free kernel when the layer's partial sums are provably exact), then
    one all-gather of the sparse row blocks over NCCL; runs of layers with an
    empty input and every bias <= 0 are skipped on every rank at once."""
    import torch
    from . import semikern as skm
    dist = _dist()
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    m, n = y0.rows(), y0.cols()
    L = len(w_blocks)
    # Per layer, is every bias <= 0 on every rank?  Then an empty input stays
    # empty (untouched positions give epilogue(0 + b) = 0): those layers need no
    # work and no exchange.  Every rank holds the same full Y_k, so all ranks
    # take the same decision.
    flags = torch.tensor([1 if np.all(np.asarray(b, np.float32) <= 0.0) else 0 for b in b_blocks],
                         dtype=torch.int32, device=device)
    if dist.is_initialized() and L:
        dist.all_reduce(flags, op=dist.ReduceOp.MIN, group=group)
    nonpos = [bool(x) for x in flags.cpu().tolist()]
    y = y0
    trace = [y.nnz()]
    for k, (w, b) in enumerate(zip(w_blocks, b_blocks)):
        if y.nnz() == 0 and nonpos[k]:
            trace.append(0)
            continue
        local = skm.sparse_layer(w, b, y, clip)
        rp, ci, v = csr_to_torch(local, device)
        frp, fci, fv = allgather_csr_rows(rp, ci, v, group=group)
        nnz = int(frp[-1].item())
        frp32 = frp.to(torch.int32)
        torch.cuda.synchronize(device)
        y = skm.csr_from_device(m, n, nnz, frp32.data_ptr(), fci.data_ptr(), fv.data_ptr(),
                                ctx=y0.ctx)
        y.ctx.synchronize()
        trace.append(nnz)
    if dist.is_initialized():
        dist.barrier(group=group)
    return y, trace
