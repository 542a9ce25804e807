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


def exchange_plan(counts, rank: int):
    """Entry offset of `rank`'s block and the total, from every rank's block
    nnz (rank order = row order)."""
    counts = [int(c) for c in counts]
    return sum(counts[:rank]), sum(counts)


def grown_capacity(total: int, cap: int) -> int:
    """Receive-buffer capacity (entries) after a layer of `total` entries: a
    rank-independent rule, so every rank reallocates (and re-exchanges its IPC
    handles) at the same layer."""
    if total <= cap:
        return cap
    c = max(cap, 1 << 16)
    while c < total:
        c *= 2
    return c


class PeerExchange:
    """Two sets (ping-pong) of next-layer input buffers per rank (row pointers
    m+1, col_idx / values `cap` entries), exported with CUDA IPC and mapped by
    every peer.  A rank's block is published by ONE kernel (sk_csr_publish:
    stores over NVLink into every rank's buffers); readers are ordered after
    every rank's publish by a collective barrier.  Layer k's output goes to set
    k % 2: a rank can only write set s again after every rank passed the barrier
    of the layer that read it."""

    def __init__(self, m: int, group=None, ctx=None):
        from . import semikern as skm
        self.skm, self.m, self.group, self.ctx = skm, m, group, ctx
        dist = _dist()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.cap = 0
        self.sets = [None, None]
        self.layers = 0  # exchanged layers so far (all calls): picks the ping-pong set

    def next_set(self) -> int:
        """The buffer set of the next exchanged layer.  The count runs across
        calls, so consecutive exchanges always alternate: a rank writes a set
        again only after every rank passed the barrier of the exchange that read
        it (no end-of-call barrier needed)."""
        s = self.layers % 2
        self.layers += 1
        return s

    def _free_all(self):
        # every rank unmaps its peers' buffers before any owner frees its own
        for s in self.sets:
            if s is not None:
                for (_, peers) in s.values():
                    for r, p in enumerate(peers):
                        if r != self.rank:
                            self.skm.ipc_close(p)
        if self.world > 1:
            _dist().barrier(group=self.group)
        for s in self.sets:
            if s is not None:
                for (own, _) in s.values():
                    self.skm.ipc_free(own)
        self.sets = [None, None]

    def _alloc_set(self):
        import torch
        dist = _dist()
        out = {}
        for name, nbytes in (("rp", (self.m + 1) * 4), ("ci", self.cap * 4), ("v", self.cap * 4)):
            own, h = self.skm.ipc_alloc(nbytes, ctx=self.ctx)
            hs = [h]
            if self.world > 1:
                hs = [None] * self.world
                dist.all_gather_object(hs, h, group=self.group)
            peers = [own if r == self.rank else self.skm.ipc_open(hs[r], ctx=self.ctx)
                     for r in range(self.world)]
            out[name] = (own, peers)
        torch.cuda.synchronize()
        return out

    def ensure(self, total: int):
        cap = grown_capacity(total, self.cap)
        if cap != self.cap or self.sets[0] is None:
            if self.world > 1:
                _dist().barrier(group=self.group)  # nobody still reads the old buffers
            self._free_all()
            self.cap = cap
            self.sets = [self._alloc_set(), self._alloc_set()]

    def publish(self, blk, k: int, row_off: int, nnz_off: int, write_last: bool):
        s = self.sets[k % 2]
        self.skm.csr_publish(blk, s["rp"][1], s["ci"][1], s["v"][1], row_off, nnz_off,
                             write_last)

    def publish_staged(self, st, k: int, row_off: int, nnz_off: int, write_last: bool):
        """Write a staged layer's block into every rank's set k % 2 with the
        layer's own gather kernel (the exchange fused into the output gather)."""
        s = self.sets[k % 2]
        st.publish(s["rp"][1], s["ci"][1], s["v"][1], row_off, nnz_off, write_last)

    def local(self, k: int):
        s = self.sets[k % 2]
        return s["rp"][0], s["ci"][0], s["v"][0]

    def close(self):
        if self.world > 1:
            _dist().barrier(group=self.group)
        self._free_all()


class ColShardPlan:
    """Per-model state of the column-sharded forward, built once and reused by
    every call: each layer block's bias on the device with its two summaries
    (sk_sparse_layer_dev), and the per-layer "every bias <= 0 on every rank"
    flags agreed with ONE all-reduce."""

    def __init__(self, w_blocks, b_blocks, device=None, group=None):
        import torch
        from . import semikern as skm
        dist = _dist()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.w_blocks = list(w_blocks)
        self.d_bias = [torch.as_tensor(np.ascontiguousarray(b, np.float32), device=device)
                       for b in b_blocks]
        self.summ = [skm.bias_summaries(b) for b in b_blocks]
        flags = torch.tensor([1 if np.all(np.asarray(b, np.float32) <= 0.0) else 0
                              for b in b_blocks], dtype=torch.int32, device=device)
        if dist.is_initialized() and len(b_blocks):
            dist.all_reduce(flags, op=dist.ReduceOp.MIN, group=group)
        self.nonpos = [bool(x) for x in flags.cpu().tolist()]
        torch.cuda.synchronize(device)


def relu_forward_sparse_colsharded(w_blocks, b_blocks, y0, clip=0.0, group=None, device=None,
                                   exchange="peer", peer=None, plan=None, exchange_single=False):
    """Column-sharded sparse forward pass.  `w_blocks[k]` is this rank's block
    of output-neuron rows of W_ref[k] (a CsrMatrix m_g x m), `b_blocks[k]` its
    bias slice, `y0` the full m x n input (replicated).  Returns (Y_L, trace).
    Per layer: local block SpGEMM + epilogue on the GPU (sk_sparse_layer_dev:
    the order-free kernel when the layer's partial sums are provably exact),
    then one exchange of the sparse row blocks; runs of layers with an empty
    input and every bias <= 0 are skipped on every rank at once.  exchange="peer":
    the block counts go through one tiny NCCL all-gather, then ONE kernel per
    rank stores its block into every rank's next-layer buffers over NVLink (CUDA
    IPC, PeerExchange; pass `peer` to reuse its buffers across calls) -- with
    the exact path that kernel IS the layer's output gather (sk_sparse_layer_stage
    / sk_staged_publish: the block never lands in a local buffer first);
    exchange="nccl": padded NCCL all-gathers of the blocks.  With one rank the
    exchange is the identity and is skipped (exchange_single=True runs it anyway,
    for tests).  Pass `plan` (ColShardPlan) to reuse the per-layer device biases
    and flags across calls."""
    import torch
    from . import semikern as skm
    dist = _dist()
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    if plan is None:
        plan = ColShardPlan(w_blocks, b_blocks, device=device, group=group)
    m, n = y0.rows(), y0.cols()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    y = y0
    trace = [y.nnz()]
    own_peer = None
    for k, w in enumerate(plan.w_blocks):
        if y.nnz() == 0 and plan.nonpos[k]:
            trace.append(0)
            continue
        dense_rows, negmin = plan.summ[k]
        if world == 1 and not exchange_single:  # one block: the exchange is the identity
            y = skm.sparse_layer_dev(w, plan.d_bias[k].data_ptr(), dense_rows, negmin, y, clip)
            trace.append(y.nnz())
            continue
        if exchange == "peer":
            # the layer up to its block's count; the block itself is written into
            # every rank's buffers by the layer's own gather (sk_staged_publish)
            st = skm.sparse_layer_stage(w, plan.d_bias[k].data_ptr(), dense_rows, negmin, y, clip)
            cnt = torch.tensor([st.nnz], dtype=torch.int64, device=device)
            cnts = [cnt]
            if world > 1:
                cnts = [torch.zeros_like(cnt) for _ in range(world)]
                dist.all_gather(cnts, cnt, group=group)
            off, nnz = exchange_plan([int(c.item()) for c in cnts], rank)
            if peer is None:
                peer = own_peer = PeerExchange(m, group=group, ctx=y0.ctx)
            peer.ensure(nnz)
            r0, _ = block_range(m, world, rank)
            s = peer.next_set()
            peer.publish_staged(st, s, r0, off, rank == world - 1)
            # the gather runs on the library context's stream: this rank's stores
            # have landed once that stream is drained ...
            y0.ctx.synchronize()
            # ... and every rank's once the collective has completed on the host
            # side (all ranks enter it only after their own publish finished)
            if world > 1:
                flag = torch.zeros(1, device=device)
                dist.all_reduce(flag, group=group)
                flag.item()
            lrp, lci, lv = peer.local(s)
            y = skm.csr_from_device(m, n, nnz, lrp, lci, lv, ctx=y0.ctx)
            y.ctx.synchronize()
        else:
            local = skm.sparse_layer_dev(w, plan.d_bias[k].data_ptr(), dense_rows, negmin, y, clip)
            rp, ci, v = csr_to_torch(local, device)
            frp, fci, fv = allgather_csr_rows(rp, ci, v, group=group)
            nnz = int(frp[-1].item())
            frp32 = frp.to(torch.int32)
            torch.cuda.synchronize(device)
            y = skm.csr_from_device(m, n, nnz, frp32.data_ptr(), fci.data_ptr(), fv.data_ptr(),
                                    ctx=y0.ctx)
            y.ctx.synchronize()
        trace.append(nnz)
    if own_peer is not None:  # y is an owned copy: the exchange buffers can go
        own_peer.close()
    return y, trace
