"""Row-sharded exchange planner (fc_route / fc_pool_rows / fc_route_grads) on one GPU,
against numpy; and the RowShardedEmbedding training step through NCCL at world 1
(every exchange kernel on the real path) against a dense torch EmbeddingBag + SGD."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

from paper_2208_05321_b200.distributed import CudaShard, Router, RowShardedEmbedding, shard_rows_for_rank  # noqa: E402
from paper_2208_05321_b200.store import fast_capacity, pinned_empty  # noqa: E402


@pytest.mark.parametrize("world,num_ids,n", [(1, 1000, 3000), (3, 50_001, 40_000), (8, 1_000_003, 200_000)])
def test_route_matches_numpy(world, num_ids, n):
    rng = np.random.default_rng(world)
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.05
    ids = rng.permutation(num_ids)[rng.choice(num_ids, size=n, p=p / p.sum())]
    r = Router(num_ids, world, "cuda")
    local, inv, counts = r.route(torch.from_numpy(ids).cuda())
    uniq = np.unique(ids)
    order = np.lexsort((uniq // world, uniq % world))  # by owner, then owner-local id
    want = uniq[order]
    assert counts == np.bincount(uniq % world, minlength=world).tolist()
    assert np.array_equal(local.cpu().numpy(), want // world)
    pos = np.empty(uniq.max() + 1, np.int64)
    pos[want] = np.arange(want.size)
    assert np.array_equal(inv.cpu().numpy(), pos[ids])
    # pooled forward through the inverse (bags of 3, mean with weights) and its backward
    D = 8
    rows = torch.randn(want.size, D, device="cuda")
    off = torch.arange(0, n, 3, device="cuda")
    w = torch.rand(n, device="cuda")
    out = r.pool(rows, inv, off, off.numel(), False, w, "mean").cpu().numpy()
    ref = oracle.pooled_bag(rows.cpu().numpy(), inv.cpu().numpy(), off.cpu().numpy(), w.cpu().numpy(), "mean")
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-6)
    g = torch.randn(off.numel(), D, device="cuda")
    gu = r.grads(inv, want.size, g, off, off.numel(), False, w, "mean").cpu().numpy()
    ref_g = oracle.pooled_bag_backward_rows(g.cpu().numpy(), inv.cpu().numpy(), off.cpu().numpy(), want.size,
                                            w.cpu().numpy(), "mean")
    np.testing.assert_allclose(gu, ref_g, rtol=1e-4, atol=1e-5)
    with pytest.raises(ValueError, match="out of range"):
        r.route(torch.tensor([1, num_ids], device="cuda"))
    r.route(torch.from_numpy(ids[:10]).cuda())  # state is clean after an error


@pytest.mark.parametrize("ids_on", ["cuda", "host", "cuda_ready", "cuda_depth2"])
def test_row_sharded_module_nccl_world1_matches_dense(ids_on):
    """ids_on: device ids (the side-stream exchange waits for the current stream), pinned
    host ids (copied on the side stream), device ids with a `ready` event; cuda_depth2: two
    batches in flight (batch s+1 prefetched before forward(s) commits s)."""
    import torch.distributed as dist

    if not dist.is_initialized():
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1)
    num_ids, dim, steps, B = 30_000, 16, 6, 4_000
    rng = np.random.default_rng(4)
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.1
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(steps, B), p=p / p.sum())]
    table = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
    idx = shard_rows_for_rank(np.bincount(trace.reshape(-1), minlength=num_ids), 0, 1)
    rows = pinned_empty((num_ids, dim))
    rows[...] = table[idx.id_of]
    shard = CudaShard(num_ids, dim, fast_capacity(num_ids, 0.05), rows, idx, lr=0.1, device="cuda",
                      global_num_ids=num_ids)
    mod = RowShardedEmbedding(shard, 1, 0, mode="sum", device=torch.device("cuda"))
    assert mod.router is not None
    grads = [rng.standard_normal((B, dim)).astype(np.float32) for _ in range(steps)]
    if ids_on == "host":
        ids = [torch.from_numpy(trace[s]).pin_memory() for s in range(steps)]
    else:
        ids = [torch.from_numpy(trace[s]).cuda() for s in range(steps)]
    ready = None
    if ids_on in ("cuda_ready", "cuda_depth2"):
        ready = torch.cuda.Event()
        ready.record()
    depth2 = ids_on == "cuda_depth2"
    if depth2:
        mod.prefetch(ids[0], ready=ready)
    dense = torch.nn.EmbeddingBag(num_ids, dim, mode="sum", sparse=True)
    dense.weight.data = torch.from_numpy(table.copy())
    opt = torch.optim.SGD(dense.parameters(), lr=0.1)
    for s in range(steps):
        if depth2 and s + 1 < steps:
            mod.prefetch(ids[s + 1], ready=ready)
        out = mod(ids[s])
        want = dense(torch.from_numpy(trace[s]), torch.arange(B))
        # fp32 sums of hot rows' gradients in a different order than torch's: 1e-5 of the
        # values' scale (|w| <~ 0.5) as the absolute floor
        np.testing.assert_allclose(out.detach().cpu().numpy(), want.detach().numpy(), rtol=1e-5, atol=5e-6)
        if s + 1 < steps and not depth2:
            mod.prefetch(ids[s + 1], ready=ready)
        out.backward(torch.from_numpy(grads[s]).cuda())
        opt.zero_grad()
        want.backward(torch.from_numpy(grads[s]))
        opt.step()
    mod.flush()
    torch.cuda.synchronize()
    got = np.empty_like(table)
    got[idx.id_of] = rows
    np.testing.assert_allclose(got, dense.weight.detach().numpy(), rtol=1e-5, atol=5e-6)
    dist.destroy_process_group()


@pytest.mark.parametrize("opt", ["sgd", "adagrad"])
def test_owner_direct_apply_equals_grouped(opt):
    """An owner's backward gets one gradient row per distinct id (u == n, no bags):
    k_bwd_direct applies it without the radix grouping. Bitwise equal to the grouped
    path (the same ids as one-element bags), for SGD and Adagrad, after flush."""
    num_ids, dim, n = 20_000, 32, 5_000
    rng = np.random.default_rng(9)
    table = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
    idx = shard_rows_for_rank(np.ones(num_ids, np.int64), 0, 1)
    out = []
    for bags in (False, True):
        rows = pinned_empty((num_ids, dim))
        rows[...] = table[idx.id_of]
        shard = CudaShard(num_ids, dim, fast_capacity(num_ids, 0.5), rows, idx, optimizer=opt, lr=0.05, device="cuda")
        r2 = np.random.default_rng(10)
        for _ in range(3):
            ids = torch.from_numpy(r2.choice(num_ids, n, replace=False)).cuda()
            g = torch.from_numpy(r2.standard_normal((n, dim)).astype(np.float32)).cuda()
            h = shard.prepare(ids)
            assert int(h["ucnt"].numel()) == n
            if bags:
                shard.backward(h, g, torch.arange(n, device="cuda"), n)
            else:
                shard.backward(h, g)
        shard.flush()
        torch.cuda.synchronize()
        out.append((rows.copy(), None if shard.state is None else shard.state.copy()))
    assert np.array_equal(out[0][0], out[1][0])
    if opt == "adagrad":
        assert np.array_equal(out[0][1], out[1][1])


def test_row_sharded_on_cuda_requires_the_router():
    """No torch fallback for the exchange on a GPU: a shard without the global id space is refused."""
    from paper_2208_05321_b200.distributed import RowShardedEmbedding

    class NoSpace:
        device = torch.device("cuda")
        dim = 4

    with pytest.raises(ValueError, match="global_num_ids"):
        RowShardedEmbedding(NoSpace(), 1, 0, device=torch.device("cuda"))


@pytest.mark.parametrize("world,ntables", [(1, 3), (4, 26), (8, 26)])
def test_route_tables_matches_numpy(world, ntables):
    """Table-wise routing (fc_router_create_tables): whole tables per owner, owner-local ids
    = the owner's tables in table order; output grouped by owner then owner-local id."""
    from paper_2208_05321_b200.distributed import TablePlacement

    rng = np.random.default_rng(world * 31 + ntables)
    sizes = rng.integers(1_000, 60_000, ntables)
    pl = TablePlacement.balanced(sizes, world)
    num_ids, n = pl.num_ids, 150_000
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.05
    ids = rng.permutation(num_ids)[rng.choice(num_ids, size=n, p=p / p.sum())]
    r = Router(num_ids, world, "cuda", placement=pl)
    local, inv, counts = r.route(torch.from_numpy(ids).cuda())
    uniq = np.unique(ids)
    t = np.searchsorted(pl.starts, uniq, side="right") - 1
    own, loc = pl.owner[t], pl.lbase[t] + (uniq - pl.starts[t])
    order = np.lexsort((loc, own))
    assert counts == np.bincount(own, minlength=world).tolist()
    assert np.array_equal(local.cpu().numpy(), loc[order])
    o2, l2 = pl.owner_local(torch.from_numpy(uniq))  # the torch mirror agrees with the kernels
    assert np.array_equal(o2.numpy(), own) and np.array_equal(l2.numpy(), loc)
    pos = np.empty(num_ids, np.int64)
    pos[uniq[order]] = np.arange(uniq.size)
    assert np.array_equal(inv.cpu().numpy(), pos[ids])
    # every owner-local id lies inside that owner's rows
    for w in range(world):
        mine = loc[own == w]
        assert mine.size == 0 or mine.max() < pl.local_sizes[w]
    with pytest.raises(ValueError, match="out of range"):
        r.route(torch.tensor([0, num_ids], device="cuda"))


def test_route_tables_rejects_bad_placements():
    import ctypes

    from paper_2208_05321_b200 import _lib
    from paper_2208_05321_b200.errors import check

    lib = _lib.load()
    h = ctypes.c_void_p()

    def create(starts, owner, world=2, num_ids=None):
        s = np.asarray(starts, np.int64)
        o = np.asarray(owner, np.int32)
        return lib.fc_router_create_tables(int(s[-1] if num_ids is None else num_ids), world, int(o.size),
                                           ctypes.c_void_p(s.ctypes.data), ctypes.c_void_p(o.ctypes.data), 0,
                                           ctypes.byref(h))

    for starts, owner, kw in [([0, 10, 10, 20], [0, 1, 0], {}),    # empty table
                              ([1, 10, 20], [0, 1], {}),           # not starting at 0
                              ([0, 10, 20], [0, 2], {}),           # owner out of range
                              ([0, 10, 20], [0, 1], {"num_ids": 30})]:  # does not cover the ids
        with pytest.raises(ValueError):
            check(create(starts, owner, **kw))
    check(create([0, 10, 20], [1, 0]))
    lib.fc_router_destroy(h)
    from paper_2208_05321_b200.distributed import TablePlacement

    with pytest.raises(ValueError, match="placement is for"):
        Router(20, 3, "cuda", placement=TablePlacement([0, 10, 20], [1, 0], 2))


def test_table_sharded_module_nccl_world1_matches_dense():
    """build_table_sharded + RowShardedEmbedding(placement=...) through NCCL at world 1,
    training against a dense EmbeddingBag + SGD."""
    import torch.distributed as dist

    from paper_2208_05321_b200.distributed import TablePlacement, build_table_sharded

    if not dist.is_initialized():
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1)
    sizes, dim, steps, B = [9_000, 4_000, 12_000, 5_000], 16, 5, 3_000
    pl = TablePlacement.balanced(sizes, 1)
    num_ids = pl.num_ids
    rng = np.random.default_rng(8)
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.1
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(steps, B), p=p / p.sum())]
    table = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
    counts = np.bincount(trace.reshape(-1), minlength=num_ids)
    shard = build_table_sharded(dim, 0.05, counts, pl, 0, lambda g: table[g], lr=0.1, device="cuda")
    mod = RowShardedEmbedding(shard, 1, 0, mode="sum", device=torch.device("cuda"), placement=pl)
    dense = torch.nn.EmbeddingBag(num_ids, dim, mode="sum", sparse=True)
    dense.weight.data = torch.from_numpy(table.copy())
    opt = torch.optim.SGD(dense.parameters(), lr=0.1)
    for s in range(steps):
        ids = torch.from_numpy(trace[s]).cuda()
        out = mod(ids)
        want = dense(torch.from_numpy(trace[s]), torch.arange(B))
        np.testing.assert_allclose(out.detach().cpu().numpy(), want.detach().numpy(), rtol=1e-5, atol=5e-6)
        g = np.random.default_rng(s).standard_normal((B, dim)).astype(np.float32)
        out.backward(torch.from_numpy(g).cuda())
        opt.zero_grad()
        want.backward(torch.from_numpy(g))
        opt.step()
    mod.flush()
    torch.cuda.synchronize()
    got = np.empty_like(table)
    got[pl.global_ids(0)[shard.idx_map.id_of]] = shard.rows
    np.testing.assert_allclose(got, dense.weight.detach().numpy(), rtol=1e-5, atol=5e-6)
    dist.destroy_process_group()
