"""GPU: the row-wise and table-wise exchange at world 2, as two processes on the one GPU.

NCCL refuses two ranks on one device, so the ranks join a gloo process group and the
module's all-to-alls (`distributed._a2a`) are staged through host memory; everything
else -- fc_route / fc_router_create_tables routing, the owners' caches, fc_pool_rows,
fc_route_grads, the fused backward -- runs the CUDA kernels with real cross-rank
traffic (ids owned by the other rank, gradient rows from both requesters). Each rank's
pooled output must equal a dense torch EmbeddingBag on the global batch, and after a
flush the two owners' slow tiers must together equal the dense table trained with SGD
on the global batches (1e-5; fp32 sums in a different order)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

NUM, DIM, STEPS, B, LR = 30_000, 16, 5, 4_000, 0.1
TABLES = [9_000, 1_000, 12_000, 3_000, 5_000]  # sums to NUM


def workload():
    rng = np.random.default_rng(21)
    p = 1.0 / np.arange(1, NUM + 1) ** 1.1
    trace = rng.permutation(NUM)[rng.choice(NUM, size=(STEPS, B), p=p / p.sum())]
    table = rng.uniform(-0.1, 0.1, (NUM, DIM)).astype(np.float32)
    grads = rng.standard_normal((STEPS, B, DIM)).astype(np.float32)
    return trace, table, grads


BAGS = 1_500  # per rank per step (mean mode: bags of 0-3 ids)


def workload_bags():
    """Per step and rank: (ids, offsets, bag gradients) with bag lengths 0..3."""
    rng = np.random.default_rng(33)
    p = 1.0 / np.arange(1, NUM + 1) ** 1.1
    perm = rng.permutation(NUM)
    steps = []
    for _ in range(STEPS):
        per = []
        for _r in range(2):
            lens = rng.integers(0, 4, BAGS)
            ids = perm[rng.choice(NUM, size=int(lens.sum()), p=p / p.sum())]
            off = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
            per.append((ids, off, rng.standard_normal((BAGS, DIM)).astype(np.float32)))
        steps.append(per)
    return steps


def _rank_main(rank, world, port, kind, prefetch, q, mode="sum"):
    import torch.distributed as dist

    import paper_2208_05321_b200.distributed as D
    from paper_2208_05321_b200.store import fast_capacity, pinned_empty

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)

        def staged_a2a(out, inp, out_splits, in_splits, group=None):  # CUDA tensors through host memory
            o = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=group)
            out.copy_(o)
            return out

        D._a2a = staged_a2a
        trace, table, grads = workload()
        bags = workload_bags() if mode == "mean" else None
        if bags is None:
            counts = np.bincount(trace.reshape(-1), minlength=NUM)
        else:
            counts = np.bincount(np.concatenate([b[r][0] for b in bags for r in range(world)]), minlength=NUM)
        placement = None
        if kind == "row":
            idx = D.shard_rows_for_rank(counts, rank, world)
            gids = np.arange(rank, NUM, world)
        else:
            placement = D.TablePlacement.balanced(TABLES, world)
            idx = D.shard_tables_for_rank(counts, placement, rank)
            gids = placement.global_ids(rank)
        n_local = int(gids.size)
        rows = pinned_empty((n_local, DIM))
        rows[...] = table[gids[idx.id_of]]
        cap = fast_capacity(n_local, 0.05 if mode == "sum" else 0.15)  # mean bags: more unique ids per batch
        shard = D.CudaShard(n_local, DIM, cap, rows, idx, lr=LR, device="cuda:0", global_num_ids=NUM)
        mod = D.RowShardedEmbedding(shard, world, rank, mode=mode, device=torch.device("cuda", 0),
                                    placement=placement)
        per = B // world
        if bags is None:
            tids = [torch.from_numpy(trace[s, rank * per:(rank + 1) * per]).cuda() for s in range(STEPS)]
            toff = [None] * STEPS
            tg = [torch.from_numpy(grads[s, rank * per:(rank + 1) * per]).cuda() for s in range(STEPS)]
        else:
            tids = [torch.from_numpy(b[rank][0]).cuda() for b in bags]
            toff = [torch.from_numpy(b[rank][1]).cuda() for b in bags]
            tg = [torch.from_numpy(b[rank][2]).cuda() for b in bags]
        outs = []
        for s in range(STEPS):
            out = mod(tids[s], toff[s])
            outs.append(out.detach().cpu().numpy())
            if prefetch and s + 1 < STEPS:
                mod.prefetch(tids[s + 1])
            out.backward(tg[s])
        mod.flush()
        torch.cuda.synchronize()
        got = np.empty((n_local, DIM), np.float32)
        got[:] = rows
        q.put((rank, gids[idx.id_of], got, outs))
        dist.destroy_process_group()
    except Exception:  # surface the child's failure in the parent
        import traceback

        q.put((rank, traceback.format_exc(), None, None))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("kind", ["row", "table"])
@pytest.mark.parametrize("prefetch", [False, True])
def test_two_ranks_match_dense(kind, prefetch):
    import torch.multiprocessing as mp

    trace, table, grads = workload()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, kind, prefetch, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: (g, rows, outs) for r, g, rows, outs in (q.get(timeout=600) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r][1], np.ndarray), res[r][0]
    dense = torch.nn.EmbeddingBag(NUM, DIM, mode="sum", sparse=True)
    dense.weight.data = torch.from_numpy(table.copy())
    opt = torch.optim.SGD(dense.parameters(), lr=LR)
    per = B // world
    for s in range(STEPS):
        want = dense(torch.from_numpy(trace[s]), torch.arange(B))
        for r in range(world):
            np.testing.assert_allclose(res[r][2][s], want.detach().numpy()[r * per:(r + 1) * per], rtol=1e-5,
                                       atol=5e-6)
        opt.zero_grad()
        want.backward(torch.from_numpy(grads[s]))
        opt.step()
    got = np.full_like(table, np.nan)
    for r in range(world):
        got[res[r][0]] = res[r][1]
    assert not np.isnan(got).any()  # the two owners hold every row exactly once
    np.testing.assert_allclose(got, dense.weight.detach().numpy(), rtol=1e-5, atol=5e-6)


def test_two_ranks_mean_bags_match_dense():
    """Row-wise, mean pooling over bags of 0-3 ids (empty bags included), prefetching."""
    import torch.multiprocessing as mp

    _, table, _ = workload()
    bags = workload_bags()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, "row", True, q, "mean")) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: (g, rows, outs) for r, g, rows, outs in (q.get(timeout=600) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r][1], np.ndarray), res[r][0]
    dense = torch.nn.EmbeddingBag(NUM, DIM, mode="mean", sparse=True)
    dense.weight.data = torch.from_numpy(table.copy())
    opt = torch.optim.SGD(dense.parameters(), lr=LR)
    for s, step in enumerate(bags):
        ids = np.concatenate([step[r][0] for r in range(world)])
        off = np.concatenate([step[0][1], step[1][1] + step[0][0].size])
        want = dense(torch.from_numpy(ids), torch.from_numpy(off))
        for r in range(world):
            np.testing.assert_allclose(res[r][2][s], want.detach().numpy()[r * BAGS:(r + 1) * BAGS], rtol=1e-5,
                                       atol=5e-6)
        opt.zero_grad()
        want.backward(torch.from_numpy(np.concatenate([step[r][2] for r in range(world)])))
        opt.step()
    got = np.full_like(table, np.nan)
    for r in range(world):
        got[res[r][0]] = res[r][1]
    assert not np.isnan(got).any()
    np.testing.assert_allclose(got, dense.weight.detach().numpy(), rtol=1e-5, atol=5e-6)
