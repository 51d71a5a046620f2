"""GPU: the reference's column-wise split (sharding.py:46-146, simulator.py:422-426) through
`ColumnShardedEmbedding` over `CudaShard`s (libfreqcache_b200 caches).

Every rank caches all rows of its column slice and prepares the GLOBAL batch, so its
residency decisions equal the unsharded cache's; the concatenation of the ranks' slow
tiers after a flush equals the unsharded table bitwise (test_acceptance.py:278-307).

* NCCL world 1 (one process): outputs and the trained table against dense torch
  EmbeddingBag + SGD (1e-5), and the slot table against the oracle cache fed the same
  batches.
* Two ranks as two processes on the one GPU. NCCL refuses two ranks on one device, so
  these run over a gloo process group; the module's two collectives (all-gather of ids,
  all-to-all of pooled columns and gradients) are staged through host memory by a test
  subclass. Each rank's slot table must equal the oracle's and the concatenated slow
  tiers must equal the world-1 run bitwise.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

NUM, DIM, STEPS, B, RATIO, LR = 30_000, 16, 6, 3_000, 0.05, 0.1


def workload():
    rng = np.random.default_rng(31)
    p = 1.0 / np.arange(1, NUM + 1) ** 1.1
    trace = rng.permutation(NUM)[rng.choice(NUM, size=(STEPS, B), p=p / p.sum())]
    table = rng.uniform(-0.1, 0.1, (NUM, DIM)).astype(np.float32)
    grads = rng.standard_normal((STEPS, B, DIM)).astype(np.float32)
    return trace, table, grads


def build(rank, world, trace, table, device):
    import paper_2208_05321_b200 as fc
    from paper_2208_05321_b200.distributed import CudaShard
    from paper_2208_05321_b200.store import pinned_empty

    idx = fc.build_reorder(fc.scan_frequencies(trace, NUM))
    lo, hi = fc.partition_columns(DIM, world).ranges[rank]
    rows = pinned_empty((NUM, hi - lo))
    rows[...] = table[idx.id_of][:, lo:hi]
    shard = CudaShard(NUM, hi - lo, fc.fast_capacity(NUM, RATIO), rows, idx, lr=LR, device=device)
    return shard, idx, rows


def oracle_slot_tables(trace):
    import paper_2208_05321_b200 as fc

    idx = fc.build_reorder(fc.scan_frequencies(trace, NUM))
    cap = fc.fast_capacity(NUM, RATIO)
    orc = oracle.OracleCache(idx.rank_of, np.zeros((NUM, 1), np.float32), cap)
    orc.warmup(cap)
    out = []
    for s in range(STEPS):
        orc.prepare(trace[s], s)
        out.append(orc.slot_rank.copy())
    return out


def test_column_sharded_bypassed_prefetch_matches_dense():
    """A prefetched batch that the next forward does not ask for is executed first (FIFO,
    as the cache's own pipeline does); the outputs and the trained table stay those of
    dense training."""
    import torch.distributed as dist

    from paper_2208_05321_b200.distributed import ColumnShardedEmbedding

    trace, table, grads = workload()
    if not dist.is_initialized():
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1)
    try:
        shard, idx, rows = build(0, 1, trace, table, "cuda")
        mod = ColumnShardedEmbedding(shard, DIM, 1, 0, mode="sum", device=torch.device("cuda"))
        dense = table.copy()
        tids = [torch.from_numpy(trace[s]).cuda() for s in range(STEPS)]
        for s in range(STEPS):
            out = mod(tids[s])
            want = oracle.pooled_bag(dense, trace[s], np.arange(B))
            np.testing.assert_allclose(out.detach().cpu().numpy(), want, rtol=1e-5, atol=1e-6)
            if s + 2 < STEPS:
                mod.prefetch(tids[s + 2])  # not the next batch
            out.backward(torch.from_numpy(grads[s]).cuda())
            g = oracle.pooled_bag_backward_rows(grads[s], trace[s], np.arange(B), NUM)
            oracle.sparse_sgd(dense, np.unique(trace[s]), g, LR)
        mod.flush()
        torch.cuda.synchronize()
        got = np.empty_like(table)
        got[idx.id_of] = rows
        np.testing.assert_allclose(got, dense, rtol=1e-5, atol=1e-6)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("prefetch,peer", [(False, False), (True, False), (True, True)])
def test_column_sharded_nccl_world1_matches_dense_and_oracle(prefetch, peer):
    """peer: the pooled columns written by fc_pool_cols_to_peers and the gradients pulled by
    fc_gather_cols_from_peers (PeerColumns) instead of the NCCL all-to-alls."""
    import torch.distributed as dist

    from paper_2208_05321_b200.distributed import ColumnShardedEmbedding

    trace, table, grads = workload()
    if not dist.is_initialized():
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1)
    try:
        shard, idx, rows = build(0, 1, trace, table, "cuda")
        mod = ColumnShardedEmbedding(shard, DIM, 1, 0, mode="sum", device=torch.device("cuda"),
                                     peer_rows=B if peer else 0)
        assert (mod.peer is not None) == peer
        dense = table.copy()  # the oracle restatement of torch EmbeddingBag + SGD (float64 gradients)
        slots = oracle_slot_tables(trace)
        moved = 0
        tids = [torch.from_numpy(trace[s]).cuda() for s in range(STEPS)]
        for s in range(STEPS):
            out = mod(tids[s])
            moved += mod.last_info.misses
            assert np.array_equal(shard.cache.slot_to_rank.cpu().numpy(), slots[s]), s
            want = oracle.pooled_bag(dense, trace[s], np.arange(B))
            np.testing.assert_allclose(out.detach().cpu().numpy(), want, rtol=1e-5, atol=1e-6)
            if prefetch and s + 1 < STEPS:  # next batch's all-gather + prepare_begin overlap this backward
                mod.prefetch(tids[s + 1])
            out.backward(torch.from_numpy(grads[s]).cuda())
            g = oracle.pooled_bag_backward_rows(grads[s], trace[s], np.arange(B), NUM)
            oracle.sparse_sgd(dense, np.unique(trace[s]), g, LR)
        assert moved > 0
        shard.flush()
        torch.cuda.synchronize()
        got = np.empty_like(table)
        got[idx.id_of] = rows
        np.testing.assert_allclose(got, dense, rtol=1e-5, atol=1e-6)
    finally:
        dist.destroy_process_group()


def _staged_module():
    """ColumnShardedEmbedding whose collectives run over a CPU-only (gloo) group: CUDA
    tensors are staged through host memory around each collective."""
    import torch.distributed as dist

    from paper_2208_05321_b200.distributed import ColumnShardedEmbedding

    class Staged(ColumnShardedEmbedding):
        def _allgather(self, out, inp):
            o = torch.empty(out.shape, dtype=out.dtype)
            dist.all_gather_into_tensor(o, inp.cpu(), group=self.group)
            out.copy_(o)

        def _alltoall(self, out, inp, out_splits, in_splits):
            o = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=self.group)
            out.copy_(o)

    return Staged


def _rank_main(rank, world, port, q, prefetch=False, peer=False):
    import torch.distributed as dist

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        trace, table, grads = workload()
        shard, idx, rows = build(rank, world, trace, table, "cuda:0")
        per = B // world  # this rank's slice of every global batch
        # peer: pooled columns / gradient columns through CUDA IPC peer pointers between the
        # two processes (PeerColumns) instead of the staged all-to-all
        mod = _staged_module()(shard, DIM, world, rank, mode="sum", device=torch.device("cuda", 0),
                               peer_rows=per if peer else 0)
        assert (mod.peer is not None) == peer
        slot_tables = []
        outs = []
        tids = [torch.from_numpy(trace[s, rank * per:(rank + 1) * per]).cuda() for s in range(STEPS)]
        for s in range(STEPS):
            out = mod(tids[s])
            slot_tables.append(shard.cache.slot_to_rank.cpu().numpy())
            outs.append(out.detach().cpu().numpy())
            if prefetch and s + 1 < STEPS:
                mod.prefetch(tids[s + 1])
            out.backward(torch.from_numpy(grads[s, rank * per:(rank + 1) * per]).cuda())
        shard.flush()
        torch.cuda.synchronize()
        q.put((rank, rows.copy(), slot_tables, outs))
        dist.destroy_process_group()
    except Exception as e:  # surface the child's failure in the parent
        q.put((rank, repr(e), None, None))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("prefetch,peer", [(False, False), (True, False), (True, True)])
def test_column_sharded_two_ranks_equal_world1_bitwise(prefetch, peer):
    import torch.multiprocessing as mp

    import paper_2208_05321_b200 as fc

    trace, table, grads = workload()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q, prefetch, peer)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (rows, st, outs)) for r, rows, st, outs in (q.get(timeout=300) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r][0], np.ndarray), res[r][0]
    # the unsharded (world-1) cache on the same global batches, through the same kernels
    from paper_2208_05321_b200.embedding import CachedEmbeddingBag

    idx = fc.build_reorder(fc.scan_frequencies(trace, NUM))
    m = CachedEmbeddingBag(NUM, DIM, RATIO, mode="sum", weight=table, idx_map=idx, lr=LR)
    slots = oracle_slot_tables(trace)
    per = B // world
    for s in range(STEPS):
        out = m(torch.from_numpy(trace[s]))
        o = out.detach().cpu().numpy()
        for r in range(world):  # the rank's bags, all columns (the all-to-all stitched them)
            assert np.array_equal(res[r][2][s], o[r * per:(r + 1) * per]), (s, r)
            assert np.array_equal(res[r][1][s], slots[s]), (s, r)  # identical decisions on every rank
        out.backward(torch.from_numpy(grads[s]).cuda())
    m.flush()
    torch.cuda.synchronize()
    cat = np.concatenate([res[r][0] for r in range(world)], axis=1)  # column slices, rank order
    assert np.array_equal(cat, m.slow_rows)  # bitwise


def test_pool_cols_to_peers_addressing():
    """fc_pool_cols_to_peers / fc_gather_cols_from_peers with local buffers standing in for
    three requesters: occurrence i of the global batch (requester r = its segment) lands
    in r's output row i - seg[r], columns [col, col + width) of ld-wide rows, scaled by psw;
    the gather reads the same columns back in global order."""
    import ctypes

    import paper_2208_05321_b200 as fc
    from paper_2208_05321_b200 import _lib

    lib = _lib.load()
    num, width, ld, col = 4000, 8, 24, 12
    idx = fc.IdxMap(np.arange(num), np.arange(num))
    rows = np.random.default_rng(3).standard_normal((num, width)).astype(np.float32)
    st = fc.CacheStack(idx, fc.SlowTierStore(rows.copy()), fc.FastTierStore(np.zeros((900, width), np.float32)),
                       fc.Transmitter())
    ids = np.random.default_rng(4).integers(0, num, 800)
    p = st.prepare(ids, 0)
    seg = np.array([0, 300, 300, 800], dtype=np.int64)  # requester 1 sends nothing
    W = 3
    psw = torch.rand(800, device="cuda")
    outs = [torch.zeros((seg[r + 1] - seg[r] + 2, ld), device="cuda") for r in range(W)]
    dst = torch.tensor([o.data_ptr() for o in outs], dtype=torch.int64, device="cuda")
    zero = torch.zeros(W, dtype=torch.int64, device="cuda")
    seg_d = torch.from_numpy(seg).cuda()
    dc = st.device
    rc = lib.fc_pool_cols_to_peers(dc.h, ctypes.c_void_p(p.d_unique_slots.data_ptr()),
                                   ctypes.c_void_p(p.d_inverse.data_ptr()), 800, ctypes.c_void_p(seg_d.data_ptr()), W,
                                   ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(zero.data_ptr()), ld, col,
                                   ctypes.c_void_p(psw.data_ptr()), dc.stream())
    assert rc == _lib.OK
    torch.cuda.synchronize()
    w = psw.cpu().numpy()
    for r in range(W):
        got = outs[r].cpu().numpy()
        a, b = seg[r], seg[r + 1]
        want = rows[ids[a:b]] * w[a:b, None]
        assert np.array_equal(got[:b - a, col:col + width], want), r
        assert not got[:, :col].any() and not got[:, col + width:].any() and not got[b - a:].any(), r
    # gather the same slice back: global order, [800, width]
    back = torch.empty((800, width), device="cuda")
    rc = lib.fc_gather_cols_from_peers(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(zero.data_ptr()),
                                       ctypes.c_void_p(seg_d.data_ptr()), W, 800, width, ld, col,
                                       ctypes.c_void_p(back.data_ptr()), dc.stream())
    assert rc == _lib.OK
    torch.cuda.synchronize()
    assert np.array_equal(back.cpu().numpy(), rows[ids] * w[:, None])
    # misaligned column slices are refused
    rc = lib.fc_pool_cols_to_peers(dc.h, ctypes.c_void_p(p.d_unique_slots.data_ptr()),
                                   ctypes.c_void_p(p.d_inverse.data_ptr()), 800, ctypes.c_void_p(seg_d.data_ptr()), W,
                                   ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(zero.data_ptr()), ld, 6,
                                   ctypes.c_void_p(0), dc.stream())
    assert rc == _lib.ERR_BAD_ARG


def test_column_peer_falls_back_to_nccl_on_unaligned_slices():
    """A column slice that is not a multiple of 4 floats cannot use the peer kernels: the
    module warns and keeps the NCCL all-to-all path (forward only here: the CUDA backward
    itself needs rows of a multiple of 4 floats)."""
    import warnings

    import paper_2208_05321_b200 as fc
    from paper_2208_05321_b200.distributed import ColumnShardedEmbedding, CudaShard
    from paper_2208_05321_b200.store import pinned_empty

    num, dim = 2_000, 10
    rows = pinned_empty((num, dim))
    rows[...] = np.random.default_rng(0).standard_normal((num, dim)).astype(np.float32)
    shard = CudaShard(num, dim, 500, rows, fc.IdxMap(np.arange(num), np.arange(num)), lr=0.1, device="cuda")
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        mod = ColumnShardedEmbedding(shard, dim, 1, 0, device=torch.device("cuda"), peer_rows=256)
    assert mod.peer is None and mod.peer_error and any("peer-memory exchange" in str(x.message) for x in w)
    ids = torch.arange(0, 200, device="cuda")
    out = mod(ids)
    np.testing.assert_array_equal(out.detach().cpu().numpy(), rows[:200])
