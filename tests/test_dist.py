"""CPU, world_size 2 over gloo: the multi-GPU host logic of
paper_1708_02937_b200/shard.py -- batch-row shards, category gathering, and the
per-layer all-gather of sparse row blocks used by the column-sharded forward --
with the oracle restatement standing in for the per-GPU layer compute."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1708_02937_b200.shard import (allgather_csr_rows, batch_shard, block_range,
                                         exchange_plan, gather_categories, grown_capacity)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world(fn, world=2):
    port = free_port()
    mp.spawn(_entry, args=(world, port, fn), nprocs=world, join=True)


def _entry(rank, world, port, fn):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        fn(rank, world)
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_block_range_partitions_exactly():
    for count in (0, 1, 7, 60000, 65536):
        for world in (1, 2, 3, 8):
            ranges = [block_range(count, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == count
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 1
    assert batch_shard(60000, 8, 3) == (22500, 7500)


def _csr_block(rank):
    from oracle.oracle import Port
    P = Port.get()
    rows = 5 + 3 * rank
    W = P.gen_layer_fixed(64, 3, 100 + rank)
    rp = torch.tensor(W.row_ptr[: rows + 1].astype(np.int64))
    nnz = int(rp[-1])
    return rp, torch.tensor(W.col_idx[:nnz].astype(np.int32)), torch.tensor(W.values[:nnz])


def _w_allgather(rank, world):
    rp, ci, v = _csr_block(rank)
    frp, fci, fv = allgather_csr_rows(rp, ci, v)
    blocks = [_csr_block(r) for r in range(world)]
    off, exp_rp = 0, []
    for b in blocks:
        exp_rp.append(b[0][:-1] + off)
        off += int(b[0][-1])
    exp_rp.append(torch.tensor([off]))
    assert torch.equal(frp, torch.cat(exp_rp))
    assert torch.equal(fci, torch.cat([b[1] for b in blocks]))
    assert torch.equal(fv.view(torch.int32), torch.cat([b[2] for b in blocks]).view(torch.int32))


def test_allgather_csr_rows_gloo():
    run_world(_w_allgather)


def _w_colsharded(rank, world):
    """Column-sharded forward on the cfg3 construction (reduced): each rank
    computes its block of output neurons with the oracle, blocks are exchanged
    with allgather_csr_rows; the result must equal the single-process run."""
    from oracle.oracle import Csr, Port
    P = Port.get()
    m, n, L = 2048, 48, 3
    clip, bias = 32.0, -0.05
    Ws = [P.gen_layer_fixed(m, 32, P.layer_seed(9, k), 1.0 / 16) for k in range(L)]
    Y0 = P.gen_input_binary(m, n, 160, 9)
    r0, r1 = block_range(m, world, rank)
    y = Y0
    for k in range(L):
        W = Ws[k]
        blk = Csr(r1 - r0, m, (W.row_ptr[r0:r1 + 1] - W.row_ptr[r0]).astype(np.uint32),
                  W.col_idx[W.row_ptr[r0]:W.row_ptr[r1]], W.values[W.row_ptr[r0]:W.row_ptr[r1]])
        loc = P.layer_sparse(blk, np.full(r1 - r0, bias, np.float32), y, clip)
        frp, fci, fv = allgather_csr_rows(torch.tensor(loc.row_ptr.astype(np.int64)),
                                          torch.tensor(loc.col_idx.astype(np.int32)),
                                          torch.tensor(loc.values))
        y = Csr(m, n, frp.numpy().astype(np.uint32), fci.numpy().astype(np.uint32),
                fv.numpy().astype(np.float32))
    ref = Y0
    for k in range(L):
        ref = P.layer_sparse(Ws[k], np.full(m, bias, np.float32), ref, clip)
    assert y.same_as(ref)
    assert ref.nnz > 0


def test_column_sharded_exchange_matches_single_process():
    run_world(_w_colsharded)


def _w_batchshard(rank, world):
    """Batch-row shards: each rank generates exactly its slice of the global
    batch, runs the whole network, and the gathered category set equals the
    single-process one."""
    from oracle.oracle import Port
    P = Port.get()
    m, B, L = 1024, 90, 2
    Ws = [P.gen_layer_fixed(m, 16, P.layer_seed(4, k), 0.25) for k in range(L)]
    start, count = batch_shard(B, world, rank)
    y = P.gen_input_binary(m, count, 40, 4, sample_offset=start)
    for W in Ws:
        y = P.layer_sparse(W, np.full(m, -0.1, np.float32), y, 32.0)
    cats = gather_categories(P.categories_sparse(y), start)
    full = P.gen_input_binary(m, B, 40, 4)
    for W in Ws:
        full = P.layer_sparse(W, np.full(m, -0.1, np.float32), full, 32.0)
    want = P.categories_sparse(full)
    assert np.array_equal(cats, want) and want.size > 0


def test_batch_sharded_categories_match_single_process():
    run_world(_w_batchshard)


def _w_peer_plan(rank, world):
    """The peer-memory exchange's host logic: every rank derives the same
    entry offsets (a partition of the concatenated blocks, rank order) and the
    same receive-buffer capacity from the gathered block counts, layer after
    layer, so all ranks reallocate and re-exchange IPC handles together."""
    rng = np.random.default_rng(7 + rank)
    cap = 0
    for layer in range(6):
        mine = int(rng.integers(0, 50000 * (layer + 1)))
        c = torch.tensor([mine], dtype=torch.int64)
        cs = [torch.zeros_like(c) for _ in range(world)]
        dist.all_gather(cs, c)
        counts = [int(x.item()) for x in cs]
        off, total = exchange_plan(counts, rank)
        assert off == sum(counts[:rank]) and total == sum(counts)
        cap = grown_capacity(total, cap)
        assert cap >= total
        agreed = [None] * world
        dist.all_gather_object(agreed, (off, off + mine, total, cap))
        spans = sorted((a, b) for a, b, _, _ in agreed)
        assert spans[0][0] == 0 and spans[-1][1] == total
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        assert len({(t, k) for _, _, t, k in agreed}) == 1


def test_peer_exchange_plan_agrees_across_ranks():
    run_world(_w_peer_plan)


def test_grown_capacity_rule():
    assert grown_capacity(0, 0) == 0
    assert grown_capacity(10, 0) == 1 << 16
    assert grown_capacity(70000, 1 << 16) == 1 << 17
    assert grown_capacity(100, 1 << 17) == 1 << 17


def _w_strong_plan(rank, world):
    """bench.py's strong-scaling plan for BASELINE cfg4 (one batch of 60000
    samples split over the ranks): the shards tile the global batch exactly, the
    job counts the global batch once, and each rank's generated input shard is
    bitwise the matching slice of the single-process input (reduced width)."""
    import bench
    from oracle.oracle import Port
    plans = [None] * world
    mine = bench.sample_plan(60000, world, rank, cols=False, strong=True)
    dist.all_gather_object(plans, mine)
    spans = sorted((b, b + n) for b, n, _ in plans)
    assert spans[0][0] == 0 and spans[-1][1] == 60000
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    assert {j for _, _, j in plans} == {60000}
    assert bench.sample_plan(60000, world, rank, cols=False, strong=False) == \
        (rank * 60000, 60000, 60000 * world)
    P = Port.get()
    m, kY = 2048, 9
    b0, Bl, _ = mine
    shard_y = P.gen_input_binary(m, Bl, kY, bench.SEED, sample_offset=b0)
    full = P.gen_input_binary(m, 60000, kY, bench.SEED)
    for k in range(0, m, 97):  # sampled rows: the shard is the global row's slice
        row = full.col_idx[full.row_ptr[k]:full.row_ptr[k + 1]]
        want = row[(row >= b0) & (row < b0 + Bl)] - b0
        got = shard_y.col_idx[shard_y.row_ptr[k]:shard_y.row_ptr[k + 1]]
        assert np.array_equal(got, want)


def test_strong_scaling_plan_tiles_the_global_batch():
    run_world(_w_strong_plan)
