"""CPU (gloo, world_size 2): the multi-GPU exchange logic of
paper_2208_05321_b200.distributed — id routing / all-gather, pooled-output and
gradient all-to-alls, column concatenation — with each rank's compute done by the
numpy oracle cache. Outputs and trained tables must equal a single dense table."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2208_05321_b200.distributed import (ColumnShardedEmbedding, RowShardedEmbedding, TablePlacement,
                                               shard_rows_for_rank)
from paper_2208_05321_b200.sharding import partition_columns

NUM, DIM, BAGS, STEPS, LR = 400, 10, 24, 5, 0.1
TABLES = [100, 50, 150, 60, 40]  # table-wise split: five tables over the 400 ids


class OracleShard:
    """Per-rank compute for the tests: an OracleCache over the rank's rows."""

    def __init__(self, rank_of, rows_rank_order, capacity, lr):
        self.c = oracle.OracleCache(rank_of, rows_rank_order, capacity)
        self.c.warmup(capacity)
        self.lr = lr
        self.device = torch.device("cpu")

    def prepare(self, ids):
        p = self.c.prepare(ids.numpy())
        return {"p": p, "n": int(ids.numel()), "slots": self.c.occurrence_slots(p)}

    # prefetch: the oracle executes the prepare at commit time (sequential semantics), FIFO
    def prepare_begin(self, ids):
        self._pending = getattr(self, "_pending", []) + [ids]

    def prepare_commit(self):
        ids = self._pending.pop(0)
        return self.prepare(ids)

    def pool(self, h, offsets=None, n_bags=None, include_last_offset=False, psw=None, mode="sum"):
        off = np.arange(h["n"]) if offsets is None else offsets.numpy()
        w = None if psw is None else psw.numpy()
        return torch.from_numpy(oracle.pooled_bag(self.c.fast, h["slots"], off, w, mode, include_last_offset))

    def backward(self, h, grad, offsets=None, n_bags=None, include_last_offset=False, psw=None, mode="sum"):
        off = np.arange(h["n"]) if offsets is None else offsets.numpy()
        w = None if psw is None else psw.numpy()
        g = oracle.pooled_bag_backward_rows(grad.numpy(), h["slots"], off, self.c.capacity, w, mode,
                                            include_last_offset)
        touched = np.unique(h["slots"])
        oracle.sparse_sgd(self.c.fast, touched, g, self.lr)
        self.c.dirty[touched] = True

    def table(self):
        self.c.flush()
        return self.c.slow


def batches_for(rank, world, mode):
    rng = np.random.default_rng(100)
    p = 1.0 / np.arange(1, NUM + 1) ** 1.1
    perm = rng.permutation(NUM)
    out = []
    for _ in range(STEPS):
        per_rank = []
        for _r in range(world):
            lens = rng.integers(0, 4, BAGS) if mode == "mean" else np.ones(BAGS, dtype=np.int64)
            ids = perm[rng.choice(NUM, size=int(lens.sum()), p=p / p.sum())]
            off = np.concatenate([[0], np.cumsum(lens)[:-1]])
            gout = rng.normal(0, 1, (BAGS, DIM)).astype(np.float32)
            per_rank.append((ids, off, gout))
        out.append(per_rank)
    return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, mode, q, prefetch=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        table = oracle.init_rows(NUM, DIM, 5)
        data = batches_for(rank, world, mode)
        counts = np.bincount(np.concatenate([d[r][0] for d in data for r in range(world)]), minlength=NUM)
        if kind == "row":
            idx = shard_rows_for_rank(counts, rank, world)
            local_rows = table[rank::world][idx.id_of].copy()
            shard = OracleShard(idx.rank_of, local_rows, max(1, idx.num_ids // 2), LR)
            mod = RowShardedEmbedding(shard, world, rank, mode=mode)
        elif kind == "table":
            pl = TablePlacement.balanced(TABLES, world)
            gids = pl.global_ids(rank)
            rank_of, id_of = oracle.rank_permutation(counts[gids])
            shard = OracleShard(rank_of, table[gids][id_of].copy(), max(1, gids.size // 2), LR)
            mod = RowShardedEmbedding(shard, world, rank, mode=mode, placement=pl)
        else:
            rank_of, id_of = oracle.rank_permutation(counts)
            a, b = partition_columns(DIM, world).ranges[rank]
            shard = OracleShard(rank_of, np.ascontiguousarray(table[:, a:b])[id_of], NUM // 2, LR)
            mod = ColumnShardedEmbedding(shard, DIM, world, rank, mode=mode)
        dense = table.copy()
        out = None
        tids = [torch.from_numpy(d[rank][0]) for d in data]
        if prefetch == "depth2":
            mod.prefetch(tids[0])
        for si, step in enumerate(data):
            for r in range(world):  # dense reference of every rank's batch
                ids, off, gout = step[r]
                if r == rank:
                    want = oracle.pooled_bag(dense, ids, off, None, mode)
            ids, off, gout = step[rank]
            t_ids = tids[si] if prefetch in (True, "depth2") else torch.from_numpy(ids)
            if prefetch == "depth2" and si + 1 < len(data):
                mod.prefetch(tids[si + 1])  # two batches in flight: batch si+1 begun before si is committed
            out = mod(t_ids, torch.from_numpy(off) if mode == "mean" else None)
            np.testing.assert_allclose(out.detach().numpy(), want, rtol=1e-5, atol=1e-6)
            if prefetch == "bypass" and si + 2 < len(data):
                # a batch that the next forward does not ask for: that forward executes it
                # first (FIFO), then prepares its own ids; outputs must not change
                mod.prefetch(tids[si + 2])
            elif prefetch is True and si + 1 < len(data):
                mod.prefetch(tids[si + 1])  # next batch's exchange + prepare start, before this backward
            out.backward(torch.from_numpy(gout))
            # dense SGD with every rank's batch (each rank owns its own bags' gradients)
            grad = np.zeros((NUM, DIM))
            for r in range(world):
                i2, o2, g2 = step[r]
                grad += oracle.pooled_bag_backward_rows(g2, i2, o2, NUM, None, mode)
            touched = np.flatnonzero(np.abs(grad).sum(1) > 0)
            oracle.sparse_sgd(dense, touched, grad, LR)
        got = shard.table()
        if kind == "row":
            want_rows = dense[rank::world][idx.id_of]
        elif kind == "table":
            want_rows = dense[gids][id_of]
        else:
            want_rows = np.ascontiguousarray(dense[:, a:b])[id_of]
        np.testing.assert_allclose(got, want_rows, rtol=1e-5, atol=1e-6)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,prefetch", [("row", False), ("row", True), ("row", "bypass"), ("row", "depth2"),
                                            ("table", False), ("table", True), ("column", "depth2"), ("column", False),
                                            ("column", True), ("column", "bypass")])
@pytest.mark.parametrize("mode", ["sum", "mean"])
def test_two_rank_gloo_matches_dense(kind, mode, prefetch):
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, mode, q, prefetch)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
