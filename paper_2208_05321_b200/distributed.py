"""Multi-GPU cached embedding: one process per GPU, NCCL over NVLink/NVSwitch.

Two shardings, both with one device cache per rank:

* `ColumnShardedEmbedding` — the reference's semantics (sharding.py:1-10, 62-118):
  every rank holds all rows of a contiguous column slice (`partition_columns`) and
  runs its own cache over the GLOBAL batch, so residency decisions are identical on
  every rank and the concatenation over ranks equals the unsharded lookup bitwise.
  Exchanges: all-gather of the batch ids, then all-to-all of pooled activations
  [bags_global, D/N] -> [bags_local, D] (sharding.py:121-146 accounts exactly these
  bytes); the backward is the mirror all-to-all of gradients.
* `RowShardedEmbedding` — the scaling variant: rows are owned by rank id % N, each
  rank caches only its shard (its own frequency reorder over its id substream), ids
  travel to their owner by all-to-all and rows come back the same way. Index work
  is partitioned as well as row traffic, so lookups/s scale with N.

The per-rank compute is a `shard` object (`CudaShard` below wraps a DeviceCache and
libfreqcache_b200); the exchange logic is backend-agnostic torch.distributed code,
which the CPU tests run over gloo with an oracle shard.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .device import DeviceCache, _raw_stream
from .freq_stats import IdxMap
from .sharding import partition_columns
from .store import fast_capacity, pinned_empty


class CudaShard:
    """One rank's slice of the table behind a device cache."""

    def __init__(self, num_rows: int, dim: int, capacity: int, rows_rank_order: np.ndarray, idx_map: IdxMap,
                 optimizer: str = "sgd", lr: float = 0.01, eps: float = 1e-10, buffer_bytes: int = 64 * 2**20,
                 warmup: bool = True, device=None, engine: str = "async", global_num_ids: int | None = None):
        self.global_num_ids = global_num_ids  # whole-table id space (row-sharded exchange)
        sw = dim if optimizer == "adagrad" else 0
        self.cache = DeviceCache(num_rows, capacity, dim, state_width=sw, buffer_bytes=buffer_bytes, device=device)
        self.cache.set_idx_map(idx_map.rank_of)
        self.rows = rows_rank_order
        self.state = None
        if sw:
            self.state = pinned_empty((num_rows, sw))
            self.state.fill(0.0)
        self.cache.attach_slow(self.rows, self.state)
        self.cache.set_engine(engine)
        self.idx_map = idx_map
        self.dim, self.optimizer, self.lr, self.eps = dim, optimizer, lr, eps
        self.device = self.cache.device
        if warmup:
            self.cache.warmup(capacity)

    def prepare(self, ids):
        info, uids, ucnt, uranks, uslots, inverse, _ = self.cache.prepare(ids)
        return {"info": info, "uslots": uslots, "inverse": inverse, "ucnt": ucnt, "n": int(inverse.numel())}

    # prefetch pipeline (DeviceCache.prepare_begin / prepare_commit)
    def prepare_begin(self, ids, consumer=None):
        self.cache.prepare_begin(ids, consumer=consumer)

    def prepare_commit(self):
        info, uids, ucnt, uranks, uslots, inverse, _ = self.cache.prepare_commit()
        return {"info": info, "uslots": uslots, "inverse": inverse, "ucnt": ucnt, "n": int(inverse.numel())}

    def pool(self, h, offsets=None, n_bags=None, include_last_offset=False, psw=None, mode="sum"):
        return self.cache.pooled(h["uslots"], h["inverse"], h["n"], offsets, n_bags, include_last_offset, psw, mode)

    def backward(self, h, grad, offsets=None, n_bags=None, include_last_offset=False, psw=None, mode="sum"):
        if h["n"] == 0:
            return
        nb = h["n"] if offsets is None else n_bags
        self.cache.backward_update(h["uslots"], h["inverse"], h["ucnt"], offsets, nb, include_last_offset, psw, mode,
                                   grad.contiguous(), self.optimizer, self.lr, self.eps)

    def flush(self) -> int:
        return self.cache.flush()


class TablePlacement:
    """Table-wise sharding (the other split `north_star` names besides column-wise): table t
    is the global id range [starts[t], starts[t+1]) and belongs whole to rank owner[t]; an
    owner's local rows are its tables in table order (fc_router_create_tables)."""

    def __init__(self, starts, owner, world: int):
        self.starts = np.asarray(starts, dtype=np.int64)
        self.owner = np.asarray(owner, dtype=np.int32)
        self.world = int(world)
        sizes = np.diff(self.starts)
        if self.starts[0] != 0 or (sizes <= 0).any() or self.owner.size != sizes.size:
            raise ValueError("table starts must be strictly increasing from 0, one owner per table")
        if (self.owner < 0).any() or (self.owner >= self.world).any():
            raise ValueError(f"table owners must be ranks in [0, {self.world})")
        self.lbase = np.zeros(sizes.size, dtype=np.int64)
        load = np.zeros(self.world, dtype=np.int64)
        for t, (o, sz) in enumerate(zip(self.owner, sizes)):
            self.lbase[t] = load[o]
            load[o] += sz
        self.local_sizes = load
        self.num_ids = int(self.starts[-1])

    @classmethod
    def balanced(cls, table_sizes, world: int) -> "TablePlacement":
        """The reference's placement, plan_tables_greedy (sharding.py:158-172)."""
        from .sharding import plan_tables_greedy

        return cls.from_plan(plan_tables_greedy(table_sizes, world))

    @classmethod
    def from_plan(cls, plan) -> "TablePlacement":
        """Tables laid out contiguously in table order; owners from a TableShardPlan."""
        starts = np.concatenate([[0], np.cumsum(plan.table_sizes)])
        return cls(starts, plan.assignment, plan.num_shards)

    def owner_local(self, ids):
        """(owner, owner-local id) of global ids (a torch tensor), as the router computes them."""
        starts = torch.as_tensor(self.starts, device=ids.device)
        t = torch.searchsorted(starts, ids.long(), right=True) - 1
        owner = torch.as_tensor(self.owner, device=ids.device).long()[t]
        local = torch.as_tensor(self.lbase, device=ids.device)[t] + (ids.long() - starts[t])
        return owner, local

    def global_ids(self, rank: int) -> np.ndarray:
        """Global ids of rank's local rows, in local order."""
        parts = [np.arange(self.starts[t], self.starts[t + 1]) for t in range(self.owner.size) if self.owner[t] == rank]
        return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)


class Router:
    """libfreqcache_b200's row-sharded exchange planner (fc_route / fc_pool_rows /
    fc_route_grads): dedup + group-by-owner of a requester's ids with the same bitmap
    machinery as prepare, the pooled forward over the rows the owners send back, and
    its backward reduced to one deterministic gradient row per routed id."""

    def __init__(self, num_ids: int, world: int, device, placement=None):
        import ctypes

        from . import _lib
        from .errors import check

        self._ct, self._check = ctypes, check
        self.lib = _lib.load()
        self.device = torch.device(device)
        self.world = int(world)
        h = ctypes.c_void_p()
        if placement is None:  # row-wise: owner id % world
            check(self.lib.fc_router_create(int(num_ids), self.world, self.device.index or 0, ctypes.byref(h)))
        else:  # table-wise: whole tables per owner (TablePlacement)
            if placement.world != self.world or placement.num_ids != int(num_ids):
                raise ValueError(f"placement is for {placement.world} ranks over {placement.num_ids} ids, the router "
                                 f"for {self.world} over {int(num_ids)}")
            starts = np.ascontiguousarray(placement.starts, dtype=np.int64)
            owner = np.ascontiguousarray(placement.owner, dtype=np.int32)
            check(self.lib.fc_router_create_tables(int(num_ids), self.world, int(owner.size),
                                                   ctypes.c_void_p(starts.ctypes.data),
                                                   ctypes.c_void_p(owner.ctypes.data), self.device.index or 0,
                                                   ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.fc_router_destroy(self.h)
            self.h = self._ct.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self):
        return self._ct.c_void_p(_raw_stream(self.device.index))

    def route(self, ids):
        """-> (owner-local unique ids grouped by owner, inverse, per-owner counts)"""
        ct = self._ct
        n = int(ids.numel())
        local = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        inv = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        counts = (ct.c_int64 * self.world)()
        u = ct.c_int64()
        self._check(self.lib.fc_route(self.h, ct.c_void_p(ids.data_ptr()), ids.element_size(), n,
                                      ct.c_void_p(local.data_ptr()), ct.c_void_p(inv.data_ptr()), counts,
                                      ct.byref(u), self._stream()))
        return local[:u.value], inv[:n], list(counts)

    def pool(self, rows, inv, offsets, n_bags, include_last_offset, psw, mode):
        ct = self._ct
        out = torch.empty((n_bags, rows.shape[1]), dtype=torch.float32, device=self.device)
        self._check(self.lib.fc_pool_rows(
            ct.c_void_p(rows.data_ptr()), int(rows.shape[1]), ct.c_void_p(inv.data_ptr()), int(inv.numel()),
            ct.c_void_p(0 if offsets is None else offsets.data_ptr()), 0 if offsets is None else offsets.element_size(),
            int(n_bags), int(bool(include_last_offset)), ct.c_void_p(0 if psw is None else psw.data_ptr()),
            {"sum": 0, "mean": 1}[mode], ct.c_void_p(out.data_ptr()), self._stream()))
        return out

    def grads(self, inv, u, grad_out, offsets, n_bags, include_last_offset, psw, mode, out=None):
        ct = self._ct
        gu = torch.empty((u, grad_out.shape[1]), dtype=torch.float32, device=self.device) if out is None else out
        g = grad_out.contiguous()
        self._check(self.lib.fc_route_grads(
            self.h, ct.c_void_p(inv.data_ptr()), int(u), int(inv.numel()),
            ct.c_void_p(0 if offsets is None else offsets.data_ptr()), 0 if offsets is None else offsets.element_size(),
            int(n_bags), int(bool(include_last_offset)), ct.c_void_p(0 if psw is None else psw.data_ptr()),
            {"sum": 0, "mean": 1}[mode], ct.c_void_p(g.data_ptr()), int(g.shape[1]), ct.c_void_p(gu.data_ptr()),
            self._stream()))
        return gu


# ----------------------------------------------------------------------------- helpers
def _upload(vals, device):
    """A small host list as an int64 device tensor without a host sync (a pageable
    torch.tensor(..., device=cuda) blocks until the stream drains)."""
    t = torch.tensor(vals, dtype=torch.int64)
    if device.type != "cuda":
        return t
    return t.pin_memory().to(device, non_blocking=True)


def _agreed_peer(make, world, group, device):
    """Build a peer-memory exchange on every rank, or on none: a rank whose setup fails (an
    IPC mapping refused, buffers that do not fit) reports it, all ranks agree with a MIN
    all-reduce, and the modules then keep their NCCL path."""
    peer, ok = None, 1
    try:
        peer = make()
    except (RuntimeError, ValueError) as e:
        ok = 0
        import warnings

        warnings.warn(f"peer-memory exchange not set up: {e}")
    if world > 1:
        t = torch.tensor([ok], dtype=torch.int32, device=device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        ok = int(t.item())
    if not ok and peer is not None:
        peer.close()
        peer = None
    return peer


def _peer_barrier(flag, group=None):
    """Stream-ordered barrier after peer-memory writes: a one-element NCCL all-reduce on the
    current stream (every rank's earlier kernels finish before it completes anywhere). A
    CPU-only group (gloo: the single-GPU multi-process tests) waits on the host instead."""
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(flag, group=group)
    else:
        torch.cuda.current_stream(flag.device.index).synchronize()
        dist.barrier(group=group)


def _a2a(out, inp, out_splits, in_splits, group=None):
    dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)
    return out


def bag_grads(grad_out, n, offsets, n_bags, include_last_offset, psw, mode):
    """Per-occurrence gradient rows grad_out[bag(j)] * coef_j (coef = psw_j, / L for mean)."""
    if offsets is None:
        g = grad_out
        if psw is not None:
            g = g * psw.reshape(-1, 1)
        return g
    off = offsets.long()
    ends = torch.cat([off[1:], off.new_tensor([n])]) if not include_last_offset else off[1:]
    starts = off if not include_last_offset else off[:-1]
    lens = ends - starts
    bag_of = torch.repeat_interleave(torch.arange(n_bags, device=grad_out.device), lens)
    pos = torch.arange(bag_of.numel(), device=grad_out.device) - torch.repeat_interleave(
        torch.cumsum(lens, 0) - lens, lens) + torch.repeat_interleave(starts, lens)
    coef = torch.ones(bag_of.numel(), device=grad_out.device, dtype=grad_out.dtype)
    if mode == "mean":
        coef = coef / lens[bag_of].to(coef.dtype)
    if psw is not None:
        coef = coef * psw[pos]
    g = torch.zeros((n, grad_out.shape[1]), device=grad_out.device, dtype=grad_out.dtype)
    g[pos] = grad_out[bag_of] * coef.unsqueeze(1)
    return g


def pool_rows(rows, offsets, n_bags, include_last_offset, psw, mode):
    """EmbeddingBag pooling of per-occurrence rows already gathered in batch order."""
    n = rows.shape[0]
    if offsets is None:
        return rows if psw is None else rows * psw.reshape(-1, 1)
    r = rows if psw is None else rows * psw.reshape(-1, 1)
    off = offsets.long()
    out = torch.nn.functional.embedding_bag(torch.arange(n, device=rows.device), r, off, mode="sum",
                                            include_last_offset=include_last_offset)
    if mode == "mean":
        out = out / _lens(off, n, include_last_offset).clamp(min=1).unsqueeze(1).to(rows.dtype)
    return out


def _lens(offsets, n, include_last_offset):
    off = offsets.long()
    if include_last_offset:
        return off[1:] - off[:-1]
    return torch.cat([off[1:], off.new_tensor([n])]) - off


class PeerRows:
    """The row-sharded forward's return exchange fused into the owner's gather: every rank
    exposes one receive buffer [max_rows, D] to all peers (CUDA IPC handles exchanged once
    with all_gather_object), and an owner's `fc_pool_to_peers` kernel writes each
    requested row straight into its requester's buffer over NVLink, at the position the
    requester's routing expects. A one-element all-reduce on the stream then orders the
    writes before any requester reads. Replaces "gather into a local buffer + NCCL
    all-to-all of the rows"."""

    def __init__(self, shard, world: int, rank: int, max_rows: int, group, device):
        import ctypes

        from . import _lib
        from .errors import check

        self._ct, self._check, self.lib = ctypes, check, _lib.load()
        self.world, self.rank, self.group, self.device = world, rank, group, torch.device(device)
        self.max_rows, self.dim = int(max_rows), int(shard.dim)
        self._opened = []
        # rbuf: rows owners write to me (forward); gbuf: my per-id gradients owners read (backward)
        self.rbuf = torch.empty((self.max_rows, self.dim), dtype=torch.float32, device=self.device)
        self.gbuf = torch.empty((self.max_rows, self.dim), dtype=torch.float32, device=self.device)
        self.dst = self._share(self.rbuf)
        self.gsrc = self._share(self.gbuf)
        self._raise_if_failed()
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)

    def _share(self, buf):
        """Every rank's pointer to its peers' copy of `buf` (CUDA IPC), as a device array.
        A rank that cannot export its handle still joins the exchange (sending None), so
        every rank raises together instead of leaving the others in the collective."""
        from . import _lib

        ct = self._ct
        hd = (ct.c_ubyte * _lib.IPC_HANDLE_BYTES)()
        mine = bytes(hd) if self.lib.fc_ipc_handle(ct.c_void_p(buf.data_ptr()), hd) == _lib.OK else None
        handles = [mine]
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, mine, group=self.group)
        if any(h is None for h in handles):
            raise RuntimeError("a rank could not export a CUDA IPC handle for the peer exchange")
        ptrs = []
        for r in range(self.world):
            if r == self.rank:
                ptrs.append(buf.data_ptr())
                continue
            p = ct.c_void_p()
            hb = (ct.c_ubyte * _lib.IPC_HANDLE_BYTES).from_buffer_copy(handles[r])
            if self.lib.fc_ipc_open(hb, self.device.index or 0, ct.byref(p)) != _lib.OK:
                self._failed = True  # raised after every exchange, so no rank leaves a collective early
                ptrs.append(0)
                continue
            self._opened.append(p)
            ptrs.append(p.value)
        return torch.tensor(ptrs, dtype=torch.int64, device=self.device)

    def _raise_if_failed(self):
        if getattr(self, "_failed", False):
            self.close()
            raise RuntimeError("could not map a peer's buffer (CUDA IPC)")

    def close(self):
        for p in getattr(self, "_opened", []):
            self.lib.fc_ipc_close(p)
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def pool_to_peers(self, shard, h, x):
        ct = self._ct
        seg, off = self._segments(x)
        stream = ct.c_void_p(torch.cuda.current_stream(self.device.index).cuda_stream)
        self._check(self.lib.fc_pool_to_peers(shard.cache.h, ct.c_void_p(h["uslots"].data_ptr()),
                                              ct.c_void_p(h["inverse"].data_ptr()), int(h["n"]),
                                              ct.c_void_p(seg.data_ptr()), self.world, ct.c_void_p(self.dst.data_ptr()),
                                              ct.c_void_p(off.data_ptr()), stream))
        if self.world > 1:  # every owner's writes land before anyone reads (one rank: stream order suffices)
            _peer_barrier(self.flag, self.group)
        return self.rbuf[:x["u"]]

    def segments(self, x):
        """Device arrays for the peer kernels, built once per exchange (uploaded without
        a host sync): seg = prefix sums of what I receive from each requester; off[r] =
        where my segment starts in requester r's routing order (after the ids r sends to
        owners < me)."""
        m, me, W = x["mat"], self.rank, self.world
        # every requester's buffer must hold what it routes: as an owner this rank writes into
        # (forward) and reads from (backward) every peer's buffer, so the bound is checked on the
        # full count matrix (identical on every rank: all raise together) before any peer kernel
        need = max(int(sum(row)) for row in m)
        if need > self.max_rows:
            raise RuntimeError(f"PeerRows buffers hold {self.max_rows} rows, a rank routes {need}")
        x["seg"] = _upload([0] + np.cumsum(x["rc"]).tolist(), self.device)
        x["off"] = _upload([sum(m[r][:me]) for r in range(W)], self.device)

    def _segments(self, x):
        if "seg" not in x:
            self.segments(x)
        return x["seg"], x["off"]

    def grads_from_peers(self, router, x, grad_out, offsets, n_bags, include_last_offset, psw, mode):
        """Requester: per-routed-id gradients into the shared gbuf; barrier; owner: pull the
        rows of its received ids from every requester's gbuf over peer memory."""
        ct = self._ct
        router.grads(x["inv"], x["u"], grad_out, offsets, n_bags, include_last_offset, psw, mode,
                     out=self.gbuf[:x["u"]])
        if self.world > 1:  # every requester's gradients are in place
            _peer_barrier(self.flag, self.group)
        seg, off = self._segments(x)
        n = int(sum(x["rc"]))
        g_recv = torch.empty((n, self.dim), dtype=torch.float32, device=self.device)
        stream = ct.c_void_p(torch.cuda.current_stream(self.device.index).cuda_stream)
        self._check(self.lib.fc_gather_from_peers(ct.c_void_p(self.gsrc.data_ptr()), ct.c_void_p(off.data_ptr()),
                                                  ct.c_void_p(seg.data_ptr()), self.world, n, self.dim,
                                                  ct.c_void_p(g_recv.data_ptr()), stream))
        return g_recv


class PeerColumns(PeerRows):
    """The column-wise exchange fused into the kernels over peer memory (bag size 1): every
    rank exposes two output buffers [max_rows, D] (alternating per step, so a forward's
    output stays valid through the next forward) and one gradient buffer [max_rows, D].
    Forward: `fc_pool_cols_to_peers` writes this rank's column slice of every global
    occurrence straight into its requester's output (replacing the pooled-columns NCCL
    all-to-all); a one-element all-reduce orders the writes before anyone reads. Backward:
    each requester copies its upstream gradient into its shared buffer, a barrier, then
    `fc_gather_cols_from_peers` pulls this rank's columns of every requester's rows."""

    def __init__(self, dim: int, width: int, col: int, world: int, rank: int, max_rows: int, group, device):
        import ctypes

        from . import _lib
        from .errors import check

        self._ct, self._check, self.lib = ctypes, check, _lib.load()
        self.world, self.rank, self.group, self.device = world, rank, group, torch.device(device)
        self.max_rows, self.dim, self.width, self.col = int(max_rows), int(dim), int(width), int(col)
        if self.dim % 4 or self.width % 4 or self.col % 4:
            raise ValueError("peer column exchange needs column slices in multiples of 4 floats")
        self._opened = []
        self.obufs = [torch.empty((self.max_rows, self.dim), dtype=torch.float32, device=self.device)
                      for _ in range(2)]
        self.gbuf = torch.empty((self.max_rows, self.dim), dtype=torch.float32, device=self.device)
        self.dsts = [self._share(b) for b in self.obufs]
        self.gsrc = self._share(self.gbuf)
        self._raise_if_failed()
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.zero_off = torch.zeros(world, dtype=torch.int64, device=self.device)
        self._step = 0

    def pool_cols(self, shard, h, counts, psw):
        """Forward: returns this rank's [n_local, D] output (a view of a shared buffer)."""
        ct = self._ct
        if max(counts) > self.max_rows:
            raise RuntimeError(f"PeerColumns buffers hold {self.max_rows} rows, a rank sends {max(counts)}")
        seg = _upload([0] + np.cumsum(counts).tolist(), self.device)
        dst = self.dsts[self._step & 1]
        buf = self.obufs[self._step & 1]
        self._step += 1
        self._check(self.lib.fc_pool_cols_to_peers(
            shard.cache.h, ct.c_void_p(h["uslots"].data_ptr()), ct.c_void_p(h["inverse"].data_ptr()), int(h["n"]),
            ct.c_void_p(seg.data_ptr()), self.world, ct.c_void_p(dst.data_ptr()), ct.c_void_p(self.zero_off.data_ptr()),
            self.dim, self.col, ct.c_void_p(0 if psw is None else psw.data_ptr()),
            ct.c_void_p(_raw_stream(self.device.index))))
        if self.world > 1:  # every rank's column writes land before anyone reads its output
            _peer_barrier(self.flag, self.group)
        return buf[:counts[self.rank]], seg

    def grads_cols(self, grad_out, seg, n_global):
        """Backward: this rank's columns of every requester's gradient rows, [n_global, width]."""
        ct = self._ct
        if self.world == 1:  # one rank holds every column of every row: the gradient is its own
            return grad_out
        self.gbuf[:grad_out.shape[0]].copy_(grad_out)
        _peer_barrier(self.flag, self.group)  # every requester's gradient rows are in place
        out = torch.empty((n_global, self.width), dtype=torch.float32, device=self.device)
        self._check(self.lib.fc_gather_cols_from_peers(
            ct.c_void_p(self.gsrc.data_ptr()), ct.c_void_p(self.zero_off.data_ptr()), ct.c_void_p(seg.data_ptr()),
            self.world, int(n_global), self.width, self.dim, self.col, ct.c_void_p(out.data_ptr()),
            ct.c_void_p(_raw_stream(self.device.index))))
        return out


# ----------------------------------------------------------------------------- row-wise (scaling)
class _RowShardFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, anchor, mod, ids, offsets, n_bags, psw):
        out, saved = mod._forward(ids, offsets, n_bags, psw, getattr(mod, "_src", None))
        ctx.mod, ctx.saved = mod, saved
        return out

    @staticmethod
    def backward(ctx, grad_out):
        ctx.mod._backward(ctx.saved, grad_out)
        return None, None, None, None, None, None


class RowShardedEmbedding(torch.nn.Module):
    """Rows owned by rank `id % world`; each rank sends its batch's UNIQUE ids to their
    owners (all-to-all), owners prepare + gather, rows come back (all-to-all) and are
    expanded through the inverse. The backward reduces the per-occurrence gradients to
    one row per unique id before the mirror all-to-all, so both exchanges carry
    unique rows only (a Zipf batch repeats each id ~3x at the Criteo shape).

    `prefetch(next_ids)` (call after forward(t), before backward(t), on every rank)
    runs the next batch's id exchange and starts the owner's prepare through the
    cache's prefetch pipeline; the next forward with the same ids commits it."""

    def __init__(self, shard, world: int, rank: int, mode: str = "sum", include_last_offset: bool = False,
                 group=None, device=None, peer_rows: int = 0, placement: TablePlacement | None = None):
        super().__init__()
        self.shard, self.world, self.rank = shard, world, rank
        if placement is not None and placement.world != world:
            raise ValueError(f"table placement is for {placement.world} ranks, the module has {world}")
        self.placement = placement  # None: row-wise (owner id % world); else table-wise
        self.mode, self.include_last_offset, self.group = mode, include_last_offset, group
        self.device = device if device is not None else getattr(shard, "device", torch.device("cpu"))
        self._anchor = torch.nn.Parameter(torch.empty(0, device=self.device))
        self.last_recv = 0
        self._pfq = []  # exchanges of prefetched batches, oldest first (at most two)
        # on a GPU the exchange planning, expansion and gradient reduction run in
        # libfreqcache_b200 (Router) -- there is no torch fallback there; the torch restatement
        # of the same steps below serves CPU process groups only (the gloo tests' oracle shards)
        self.router = None
        self.peer = None
        if self.device.type == "cuda":
            num_ids = getattr(shard, "global_num_ids", None)
            if num_ids is None:
                raise ValueError("RowShardedEmbedding on CUDA needs shard.global_num_ids (the whole table's id "
                                 "space) for the libfreqcache_b200 router")
            self.router = Router(num_ids, world, self.device, placement)
            if peer_rows:  # fused return exchange over NVLink peer memory (PeerRows); all ranks or none
                self.peer = _agreed_peer(lambda: PeerRows(shard, world, rank, int(peer_rows), group, self.device),
                                         world, group, self.device)

    @staticmethod
    def owner_of(ids, world):
        return ids % world, ids // world

    def _exchange_ids(self, ids):
        """Unique ids of this rank's batch to their owners; returns the routing."""
        W = self.world
        if self.router is not None:  # grouped by owner already: no permutation to undo
            send_ids, inv, sc = self.router.route(ids)  # (waits for the routing kernels only)
            order = None
            if W == 1:  # one rank owns everything: the exchanges are identities
                m = [list(sc)]
                x = {"inv": inv, "order": None, "sc": sc, "rc": list(sc), "recv_ids": send_ids,
                     "u": int(send_ids.numel()), "mat": m}
                if self.peer is not None:
                    self.peer.segments(x)
                return x
            if self.peer is not None:  # the full W x W count matrix: splits + peer-write offsets
                mine = _upload(sc, ids.device)
                mat = torch.empty(W * W, dtype=torch.int64, device=ids.device)
                dist.all_gather_into_tensor(mat, mine, group=self.group)
                m = mat.view(W, W).tolist()  # m[r][o] = ids rank r sends to owner o
                rc = [m[r][self.rank] for r in range(W)]
                recv_ids = torch.empty(sum(rc), dtype=send_ids.dtype, device=send_ids.device)
                _a2a(recv_ids, send_ids.contiguous(), rc, sc, self.group)
                x = {"inv": inv, "order": None, "sc": sc, "rc": rc, "recv_ids": recv_ids,
                     "u": int(send_ids.numel()), "mat": m}
                self.peer.segments(x)
                return x
            send_counts = _upload(sc, ids.device)
        else:
            uniq, inv = torch.unique(ids.long(), sorted=True, return_inverse=True)
            owner, local = self.owner_of(uniq, W) if self.placement is None else self.placement.owner_local(uniq)
            order = torch.argsort(owner, stable=True)
            send_ids = local[order]
            send_counts = torch.bincount(owner, minlength=W)
            sc = send_counts.tolist()
        recv_counts = torch.empty_like(send_counts)
        _a2a(recv_counts, send_counts, None, None, self.group)
        rc = recv_counts.tolist()
        recv_ids = torch.empty(sum(rc), dtype=send_ids.dtype, device=send_ids.device)
        _a2a(recv_ids, send_ids.contiguous(), rc, sc, self.group)
        return {"inv": inv, "order": order, "sc": sc, "rc": rc, "recv_ids": recv_ids, "u": int(send_ids.numel())}

    def prefetch(self, ids, ready=None):
        """Next batch's id exchange + the owner's prepare_begin. On a GPU they run on a
        high-priority side stream, so the routing's host sync waits for the routing
        kernels only, not for this batch's queued forward/backward. Host `ids` are
        copied there; device `ids` are read after the work queued on the current stream,
        or after `ready` (a torch.cuda.Event) when given."""
        if len(self._pfq) >= 2:
            raise RuntimeError("two prefetched batches are outstanding: run a forward first")
        if self.device.type != "cuda":
            dev_ids = ids.reshape(-1).to(self.device)
            x = self._exchange_ids(dev_ids)
            if hasattr(self.shard, "prepare_begin") and x["recv_ids"].numel() > 0:
                self.shard.prepare_begin(x["recv_ids"])
                x["begun"] = True
            x["src"], x["ids"] = ids, dev_ids
            self._pfq.append(x)
            return
        main = torch.cuda.current_stream(self.device.index)
        if getattr(self, "_xstream", None) is None:
            self._xstream = torch.cuda.Stream(self.device, priority=-100)
        xs = self._xstream
        with torch.cuda.stream(xs):
            if ids.is_cuda:
                if ready is None:
                    xs.wait_stream(main)
                else:
                    xs.wait_event(ready)
            dev_ids = ids.reshape(-1).to(self.device, non_blocking=True)
            x = self._exchange_ids(dev_ids)
            if hasattr(self.shard, "prepare_begin") and x["recv_ids"].numel() > 0:
                # its index stream waits for xs; the prepare's buffers are used on main
                self.shard.prepare_begin(x["recv_ids"], consumer=main)
                x["begun"] = True
            ev = torch.cuda.Event()
            ev.record(xs)
        for k in ("inv", "recv_ids", "seg", "off"):  # allocated on xs, consumed on main
            if isinstance(x.get(k), torch.Tensor):
                x[k].record_stream(main)
        dev_ids.record_stream(main)
        x["ev"], x["src"], x["ids"] = ev, ids, dev_ids
        self._pfq.append(x)

    def _forward(self, ids, offsets, n_bags, psw, src=None):
        x, h = None, None
        while self._pfq:  # prefetched batches are executed oldest first (FIFO) up to this one
            px = self._pfq.pop(0)
            pids = px["ids"]
            if px.get("ev") is not None:  # the side stream's exchange is ordered before anything below
                torch.cuda.current_stream(self.device.index).wait_event(px["ev"])
            hp = self.shard.prepare_commit() if px.get("begun") else None
            if px["src"] is src or pids is ids or (pids.numel() == ids.numel() and bool(torch.equal(pids, ids))):
                x, h = px, hp
                break
        if x is None:
            x = self._exchange_ids(ids)
        if h is None:
            h = self.shard.prepare(x["recv_ids"])
        self.last_recv = int(x["recv_ids"].numel())
        if self.peer is not None:  # owners write the rows straight into the requesters' buffers
            back = self.peer.pool_to_peers(self.shard, h, x)
        else:
            rows = self.shard.pool(h)  # [n_recv, D] one row per received (unique per requester) id
            if self.world == 1:
                back = rows
            else:
                back = torch.empty((x["u"], rows.shape[1]), dtype=rows.dtype, device=rows.device)
                _a2a(back, rows.contiguous(), x["sc"], x["rc"], self.group)
        if self.router is not None:  # back is in routing order: pool straight through the inverse
            out = self.router.pool(back, x["inv"], offsets, n_bags, self.include_last_offset, psw, self.mode)
        else:
            uniq_rows = torch.empty_like(back)
            uniq_rows[x["order"]] = back
            out = pool_rows(uniq_rows[x["inv"]], offsets, n_bags, self.include_last_offset, psw, self.mode)
        return out, (h, x, int(ids.numel()), offsets, n_bags, psw)

    def _backward(self, saved, grad_out):
        h, x, n, offsets, n_bags, psw = saved
        if self.peer is not None:  # gradients travel back over peer memory as well
            g_recv = self.peer.grads_from_peers(self.router, x, grad_out, offsets, n_bags, self.include_last_offset,
                                                psw, self.mode)
            self.shard.backward(h, g_recv)
            return
        if self.router is not None:  # one deterministic gradient row per routed id, in routing order
            g_send = self.router.grads(x["inv"], x["u"], grad_out, offsets, n_bags, self.include_last_offset, psw,
                                       self.mode)
        else:
            g = bag_grads(grad_out, n, offsets, n_bags, self.include_last_offset, psw, self.mode)
            gu = torch.zeros((x["u"], g.shape[1]), dtype=g.dtype, device=g.device)
            gu.index_add_(0, x["inv"], g)  # one gradient row per unique id of this rank
            g_send = gu[x["order"]].contiguous()
        g = g_send
        if self.world == 1:
            g_recv = g_send
        else:
            g_recv = torch.empty((sum(x["rc"]), g.shape[1]), dtype=g.dtype, device=g.device)
            _a2a(g_recv, g_send, x["rc"], x["sc"], self.group)
        self.shard.backward(h, g_recv)

    def forward(self, ids, offsets=None, per_sample_weights=None):
        self._src = ids
        pf = next((p for p in self._pfq if p["src"] is ids), None)
        if pf is not None:
            ids = pf["ids"]  # already on the device (prefetch copied it)
        else:
            ids = ids.reshape(-1).to(self.device, non_blocking=True)
        n_bags = ids.numel() if offsets is None else offsets.numel() - (1 if self.include_last_offset else 0)
        return _RowShardFn.apply(self._anchor, self, ids, offsets, n_bags, per_sample_weights)

    def flush(self) -> int:
        while self._pfq:  # outstanding prefetches are committed first (their batches become resident)
            px = self._pfq.pop(0)
            if px.get("ev") is not None:
                torch.cuda.current_stream(self.device.index).wait_event(px["ev"])
            if px.get("begun"):
                self.shard.prepare_commit()
        return self.shard.flush()


# ----------------------------------------------------------------------------- column-wise (reference semantics)
class _ColShardFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, anchor, mod, ids, offsets, n_bags, psw, src=None):
        out, saved = mod._forward(ids, offsets, n_bags, psw, src)
        ctx.mod, ctx.saved = mod, saved
        return out

    @staticmethod
    def backward(ctx, grad_out):
        ctx.mod._backward(ctx.saved, grad_out)
        return None, None, None, None, None, None, None


class ColumnShardedEmbedding(torch.nn.Module):
    """Rank r caches columns partition_columns(D, world).ranges[r] of every row.

    `prefetch(next_ids)` (call after forward(t), before backward(t), on every rank; or
    before forward(t) for two batches in flight) all-gathers the next batch's ids on a
    high-priority side stream and starts this rank's prepare of the GLOBAL batch through
    the cache's prefetch pipeline (DeviceCache.prepare_begin), so the index phase and the
    miss staging overlap backward(t). The next forward with the same ids commits it.
    Decisions are identical with and without prefetching (the commits are FIFO)."""

    def __init__(self, shard, dim: int, world: int, rank: int, mode: str = "sum", group=None, device=None,
                 peer_rows: int = 0):
        super().__init__()
        self.shard, self.dim, self.world, self.rank = shard, dim, world, rank
        self.plan = partition_columns(dim, world)
        self.widths = self.plan.widths
        self.mode, self.group = mode, group
        self.device = device if device is not None else getattr(shard, "device", torch.device("cpu"))
        self._anchor = torch.nn.Parameter(torch.empty(0, device=self.device))
        self._pfq = []  # prefetched batches, oldest first: dicts (src, ids, counts, ev, begun)
        self._xstream = None
        # peer_rows > 0 (CUDA, bag size 1): the pooled-columns all-to-all and its backward mirror
        # fused into the kernels over NVLink peer memory (PeerColumns); peer_rows bounds the ids
        # one rank sends per batch
        self.peer = None
        self.peer_error = None
        if peer_rows and self.device.type == "cuda":
            a, b = self.plan.ranges[rank]
            self.peer = _agreed_peer(lambda: PeerColumns(dim, b - a, a, world, rank, int(peer_rows), group,
                                                         self.device), world, group, self.device)
            if self.peer is None:
                self.peer_error = "peer exchange unavailable on some rank; NCCL all-to-all used"

    # the two collectives of the column-wise exchange (overridable: the tests drive the module
    # over a CPU-only process group by staging these through host memory)
    def _allgather(self, out, inp):
        dist.all_gather_into_tensor(out, inp, group=self.group)

    def _alltoall(self, out, inp, out_splits, in_splits):
        _a2a(out, inp, out_splits, in_splits, self.group)

    def _gather_var(self, x, counts, maxn):
        """all-gather of per-rank 1-D tensors of different lengths (padded to maxn)."""
        if self.world == 1:
            return x
        if all(c == maxn for c in counts):  # the usual case: every rank has the same batch size
            g = torch.empty(self.world * maxn, dtype=x.dtype, device=x.device)
            self._allgather(g, x)
            return g
        pad = torch.zeros(maxn, dtype=x.dtype, device=x.device)
        pad[:x.numel()] = x
        g = torch.empty(self.world * maxn, dtype=x.dtype, device=x.device)
        self._allgather(g, pad)
        return torch.cat([g[r * maxn:r * maxn + c] for r, c in enumerate(counts)])

    def _gather_ids(self, ids):
        """(global ids in rank order, per-rank counts). One host sync on the count
        all-gather at world > 1, on whatever stream is current."""
        n = ids.numel()
        if self.world == 1:
            return ids, [n]
        cnt = torch.tensor([n], dtype=torch.int64, device=ids.device)
        all_n = torch.empty(self.world, dtype=torch.int64, device=ids.device)
        self._allgather(all_n, cnt)
        counts = all_n.tolist()
        return self._gather_var(ids.contiguous(), counts, max(counts)), counts

    def prefetch(self, ids, ready=None):
        """Next batch's id all-gather + this rank's prepare_begin of the global batch. On a
        GPU both run on a side stream: host ids are copied there; device ids are read after
        the work queued on the current stream, or after `ready` (a torch.cuda.Event)."""
        if len(self._pfq) >= 2:
            raise RuntimeError("two prefetched batches are outstanding: run a forward first")
        can_begin = hasattr(self.shard, "prepare_begin")
        if self.device.type != "cuda":
            dev_ids = ids.reshape(-1).to(self.device)
            g_ids, counts = self._gather_ids(dev_ids)
            if can_begin:
                self.shard.prepare_begin(g_ids)
            self._pfq.append({"src": ids, "ids": dev_ids, "counts": counts, "ev": None, "begun": can_begin})
            return
        main = torch.cuda.current_stream(self.device.index)
        if self._xstream is None:
            self._xstream = torch.cuda.Stream(self.device, priority=-100)
        xs = self._xstream
        with torch.cuda.stream(xs):
            if ids.is_cuda:
                if ready is None:
                    xs.wait_stream(main)
                else:
                    xs.wait_event(ready)
            dev_ids = ids.reshape(-1).to(self.device, non_blocking=True)
            g_ids, counts = self._gather_ids(dev_ids)
            if can_begin:  # its index stream waits for xs; the prepare's buffers are used on main
                self.shard.prepare_begin(g_ids, consumer=main)
            ev = torch.cuda.Event()
            ev.record(xs)
        dev_ids.record_stream(main)
        g_ids.record_stream(main)
        self._pfq.append({"src": ids, "ids": dev_ids, "counts": counts, "ev": ev, "begun": can_begin})

    def _take_prefetched(self, ids, src):
        """Commit prefetched batches oldest first until `ids`' one (FIFO, like the cache's
        own pipeline); returns (prepare handle, counts) or (None, None) when `ids` was not
        prefetched (the bypassed batches are still executed, in order)."""
        while self._pfq:
            pf = self._pfq.pop(0)
            if pf["ev"] is not None:
                torch.cuda.current_stream(self.device.index).wait_event(pf["ev"])
            h = self.shard.prepare_commit() if pf["begun"] else None
            same = pf["src"] is src or pf["ids"] is ids or (
                pf["ids"].numel() == ids.numel() and bool(torch.equal(pf["ids"], ids)))
            if same and h is not None:
                return h, pf["counts"]
        return None, None

    def _forward(self, ids, offsets, n_bags, psw, src=None):
        W = self.world
        h, counts = self._take_prefetched(ids, src) if self._pfq else (None, None)
        if h is None:
            g_ids, counts = self._gather_ids(ids)
            h = self.shard.prepare(g_ids)  # identical decisions on every rank
        g_off, g_psw = None, None
        if offsets is not None:  # every rank has n_bags bags; shift offsets by the ids before it
            g_off = offsets[:n_bags].contiguous()
            if W > 1:
                g_off = torch.empty(W * n_bags, dtype=offsets.dtype, device=offsets.device)
                self._allgather(g_off, offsets[:n_bags].contiguous())
                base = torch.tensor(np.concatenate([[0], np.cumsum(counts)[:-1]]), dtype=offsets.dtype,
                                    device=offsets.device)
                g_off += base.repeat_interleave(n_bags)
        if psw is not None:
            g_psw = self._gather_var(psw.contiguous(), counts, max(counts))
        self.last_info = h.get("info") if isinstance(h, dict) else None
        if self.peer is not None and offsets is None:  # bag size 1: the all-to-all fused into the gather
            out, seg = self.peer.pool_cols(self.shard, h, counts, g_psw)
            return out, (h, None, n_bags, g_psw, seg, int(sum(counts)))
        pooled = self.shard.pool(h, g_off, W * n_bags, False, g_psw, self.mode)  # [W*n_bags, w_r]
        if W == 1:
            return pooled, (h, g_off, n_bags, g_psw, None, None)
        w_r = self.widths[self.rank]
        recv = torch.empty(sum(n_bags * w for w in self.widths), dtype=pooled.dtype, device=pooled.device)
        self._alltoall(recv, pooled.reshape(-1).contiguous(), [n_bags * w for w in self.widths], [n_bags * w_r] * W)
        parts = torch.split(recv, [n_bags * w for w in self.widths])
        out = torch.cat([p.reshape(n_bags, w) for p, w in zip(parts, self.widths)], dim=1)
        return out, (h, g_off, n_bags, g_psw, None, None)

    def _backward(self, saved, grad_out):
        h, g_off, n_bags, g_psw, seg, n_global = saved
        W, w_r = self.world, self.widths[self.rank]
        if seg is not None:  # fused peer-memory path: this rank's columns of every requester's rows
            recv = self.peer.grads_cols(grad_out.contiguous(), seg, n_global)
            self.shard.backward(h, recv, None, n_global, False, g_psw, self.mode)
            return
        if W == 1:
            recv = grad_out.contiguous()
        else:
            send = torch.cat([grad_out[:, a:b].reshape(-1) for a, b in self.plan.ranges]).contiguous()
            recv = torch.empty(W * n_bags * w_r, dtype=grad_out.dtype, device=grad_out.device)
            self._alltoall(recv, send, [n_bags * w_r] * W, [n_bags * w for w in self.widths])
        self.shard.backward(h, recv.reshape(W * n_bags, w_r), g_off, W * n_bags, False, g_psw, self.mode)

    def forward(self, ids, offsets=None, per_sample_weights=None):
        src = ids
        pf = next((p for p in self._pfq if p["src"] is ids), None)
        ids = pf["ids"] if pf is not None else ids.reshape(-1).to(self.device, non_blocking=True)
        n_bags = ids.numel() if offsets is None else offsets.numel()
        return _ColShardFn.apply(self._anchor, self, ids, offsets, n_bags, per_sample_weights, src)

    def flush(self) -> int:
        """Commit outstanding prefetches (their batches become resident), then write every
        dirty cached row of this rank's column slice back to its slow tier."""
        while self._pfq:
            pf = self._pfq.pop(0)
            if pf["ev"] is not None:
                torch.cuda.current_stream(self.device.index).wait_event(pf["ev"])
            if pf["begun"]:
                self.shard.prepare_commit()
        return self.shard.flush()


# ----------------------------------------------------------------------------- builders
def shard_rows_for_rank(counts: np.ndarray, rank: int, world: int):
    """Local id space of a row shard (ids with id % world == rank) and its frequency reorder."""
    local_counts = counts[rank::world]
    id_of = np.argsort(-local_counts, kind="stable").astype(np.int64)
    rank_of = np.empty_like(id_of)
    rank_of[id_of] = np.arange(id_of.size, dtype=np.int64)
    return IdxMap(rank_of=rank_of, id_of=id_of)


def shard_tables_for_rank(counts: np.ndarray, placement: TablePlacement, rank: int):
    """Local id space of a table shard (rank's tables in table order) and its frequency reorder."""
    local_counts = counts[placement.global_ids(rank)]
    id_of = np.argsort(-local_counts, kind="stable").astype(np.int64)
    rank_of = np.empty_like(id_of)
    rank_of[id_of] = np.arange(id_of.size, dtype=np.int64)
    return IdxMap(rank_of=rank_of, id_of=id_of)


def build_table_sharded(dim, cache_ratio, counts, placement: TablePlacement, rank, init_rows_fn, **kw):
    """CudaShard for this rank's tables (table-wise split): its own frequency reorder over
    its local rows; `init_rows_fn(global_ids) -> rows` seeds values."""
    idx = shard_tables_for_rank(counts, placement, rank)
    n_local = int(idx.id_of.size)
    rows = pinned_empty((n_local, dim))
    rows[...] = init_rows_fn(placement.global_ids(rank)[idx.id_of])
    kw.setdefault("global_num_ids", placement.num_ids)
    return CudaShard(n_local, dim, fast_capacity(n_local, cache_ratio), rows, idx, **kw)


def build_row_sharded(num_ids, dim, cache_ratio, counts, rank, world, init_rows_fn, **kw):
    """CudaShard for this rank's rows; `init_rows_fn(global_ids) -> rows` seeds values."""
    idx = shard_rows_for_rank(counts, rank, world)
    n_local = idx.num_ids
    rows = pinned_empty((n_local, dim))
    rows[...] = init_rows_fn(rank + world * idx.id_of)
    kw.setdefault("global_num_ids", num_ids)
    return CudaShard(n_local, dim, fast_capacity(n_local, cache_ratio), rows, idx, **kw)
