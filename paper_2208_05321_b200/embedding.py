"""`CachedEmbeddingBag`: the frequency-aware software-cached EmbeddingBag module.

The paper's module (ColossalAI `FreqCacheEmbeddingBag`) built on the
device cache: `forward(indices, offsets[, per_sample_weights])` makes the batch's
rows resident (prepare_cache, cache_manager.py:234-348), then pools them in HBM
with `torch.nn.functional.embedding_bag` semantics (sum / mean; mean with
per-sample weights is sum(w*row)/L, empty bag -> 0). The backward is fused with a
sparse SGD or element-wise Adagrad row update applied directly to the cached rows
(north star item 6) — the table is not a torch Parameter, exactly like a fused
TBE optimizer; Adagrad state rows are cached and written back with their weights.
"""

from __future__ import annotations

import numpy as np
import torch

from .device import DeviceCache
from .freq_stats import IdxMap
from .store import fast_capacity, init_reference_rows, pinned_empty


class _CachedBagFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, anchor, module, prep, offsets, n_bags, psw):
        cache: DeviceCache = module.cache
        out = cache.pooled(prep["uslots"], prep["inverse"], prep["n"], offsets, n_bags, module.include_last_offset,
                           psw, module.mode)
        ctx.module = module
        ctx.prep = prep
        ctx.offsets = offsets
        ctx.n_bags = n_bags
        ctx.psw = psw
        ctx.generation = module._generation
        return out

    @staticmethod
    def backward(ctx, grad_out):
        m = ctx.module
        if m._generation != ctx.generation:
            raise RuntimeError("CachedEmbeddingBag: backward must run before the next forward "
                               "(the cache may have evicted this batch's rows)")
        p = ctx.prep
        if p["u"] > 0:
            m.cache.backward_update(p["uslots"], p["inverse"], p["ucnt"], ctx.offsets, ctx.n_bags,
                                    m.include_last_offset, ctx.psw, m.mode, grad_out.contiguous(), m.optimizer,
                                    m.lr, m.eps)
        return None, None, None, None, None, None


class CachedEmbeddingBag(torch.nn.Module):
    """EmbeddingBag whose table lives in host memory behind a frequency-aware GPU cache.

    Args:
        num_embeddings, embedding_dim: table shape.
        cache_ratio: fraction of rows resident in HBM (capacity = floor(ratio*num), >= 1).
        mode: "sum" or "mean".
        weight: optional host float32 [num_embeddings, dim] initial table (raw-id order);
            default is the reference's seeded uniform(+-0.5/dim) init (store.py:118-131).
        idx_map: frequency reorder (build_reorder(scan_frequencies(trace))); default identity.
        optimizer: "sgd" or "adagrad" (fused into backward), lr, eps.
        warmup: pre-fill the cache with the hottest rows (ranks 0..C-1).
        slow_rows: optional pinned host rows already in rank order (fc_host_alloc / pinned_empty).
        engine: "async" (write-backs ride the copy engine and host threads, off the
            critical path; the table is current after flush()) or "zerocopy".
    """

    def __init__(self, num_embeddings: int, embedding_dim: int, cache_ratio: float = 0.015, *, mode: str = "sum",
                 include_last_offset: bool = False, weight: np.ndarray | None = None, init_seed: int = 0,
                 idx_map: IdxMap | None = None, optimizer: str = "sgd", lr: float = 0.01, eps: float = 1e-10,
                 buffer_bytes: int = 64 * 2**20, write_back: str = "dirty_only", warmup: bool = True, device=None,
                 slow_rows: np.ndarray | None = None, engine: str = "async"):
        super().__init__()
        if mode not in ("sum", "mean"):
            raise ValueError("mode must be 'sum' or 'mean'")
        if optimizer not in ("sgd", "adagrad"):
            raise ValueError("optimizer must be 'sgd' or 'adagrad'")
        self.num_embeddings, self.embedding_dim = int(num_embeddings), int(embedding_dim)
        self.mode, self.include_last_offset = mode, include_last_offset
        self.optimizer, self.lr, self.eps = optimizer, float(lr), float(eps)
        if idx_map is None:
            ar = np.arange(num_embeddings, dtype=np.int64)
            idx_map = IdxMap(rank_of=ar, id_of=ar.copy())
        self.idx_map = idx_map
        self.capacity = fast_capacity(num_embeddings, cache_ratio)
        sw = embedding_dim if optimizer == "adagrad" else 0
        self.cache = DeviceCache(num_embeddings, self.capacity, embedding_dim, state_width=sw, write_back=write_back,
                                 buffer_bytes=buffer_bytes, device=device)
        self.cache.set_idx_map(idx_map.rank_of)
        if slow_rows is not None:  # caller-provided pinned rows, already in rank order
            if slow_rows.shape != (num_embeddings, embedding_dim):
                raise ValueError("slow_rows must be [num_embeddings, embedding_dim] in rank order")
            rows = slow_rows
        else:
            rows = pinned_empty((num_embeddings, embedding_dim))
            if weight is None:
                weight = init_reference_rows(num_embeddings, embedding_dim, init_seed)
            np.take(np.asarray(weight, dtype=np.float32), idx_map.id_of, axis=0, out=rows)  # rank order
        self.slow_rows = rows
        self.slow_state = None
        if sw:
            self.slow_state = pinned_empty((num_embeddings, sw))
            self.slow_state.fill(0.0)
        self.cache.attach_slow(self.slow_rows, self.slow_state)
        self.cache.set_engine(engine)
        self.cache.prefetch_ring = True  # a batch's prepare outputs die with its backward
        if warmup:
            self.cache.warmup(self.capacity)
        self._anchor = torch.nn.Parameter(torch.empty(0, device=self.cache.device), requires_grad=True)
        self._generation = 0
        self.last_info = None

    def prefetch(self, indices, ready=None) -> None:
        """Start the cache work of the NEXT batch now (the paper's future-work prefetch,
        PAPER.md:490): its index phase runs on a side stream and its misses are staged
        host -> HBM on the transfer stream while this batch's backward still runs.
        Call it after forward(batch t) and before backward(t); the next forward with
        the same `indices` object commits it. It may also be called before forward(t)
        (two prefetches outstanding): batch t+1's index phase then starts on the device
        as soon as batch t's has ended. Cache decisions, slot assignment and
        write-backs are bit-identical to not prefetching. Device `indices` are read
        after the work queued on the current stream, or after `ready` (a
        torch.cuda.Event) when given (DeviceCache.prepare_begin)."""
        self.cache.prepare_begin(indices, ready=ready)

    def forward(self, indices, offsets=None, per_sample_weights=None):
        dev = self.cache.device
        n = int(indices.numel())
        if offsets is not None:
            offsets = offsets.to(dev, non_blocking=True).contiguous()
            n_bags = int(offsets.numel()) - (1 if self.include_last_offset else 0)
        else:
            n_bags = n
        if per_sample_weights is not None:
            if per_sample_weights.requires_grad:
                raise NotImplementedError("gradients w.r.t. per_sample_weights are not supported")
            per_sample_weights = per_sample_weights.to(dev, dtype=torch.float32).reshape(-1).contiguous()
        res = None
        while self.cache.prefetch_outstanding:  # prefetched batches are executed first (FIFO commits)
            res = self.cache.prepare_commit()
            if self.cache.committed_matches(indices):
                break
            res = None  # not this batch: it runs after every prefetched one
        if res is None:
            res = self.cache.prepare(indices.to(dev, non_blocking=True).reshape(-1))
        info, uids, ucnt, uranks, uslots, inverse, _ = res
        self._generation += 1
        self.last_info = info
        prep = {"uslots": uslots, "inverse": inverse, "ucnt": ucnt, "u": int(info.unique), "n": n}
        return _CachedBagFn.apply(self._anchor, self, prep, offsets, n_bags, per_sample_weights)

    def flush(self) -> int:
        """Write every dirty cached row (and optimizer state) back to host memory.
        An outstanding prefetch is committed first (its batch becomes resident)."""
        while self.cache.prefetch_outstanding:
            self.cache.prepare_commit()
        return self.cache.flush()

    def weight(self) -> np.ndarray:
        """The full table in raw-id order (after a flush)."""
        torch.cuda.synchronize(self.cache.device)
        return self.slow_rows[self.idx_map.rank_of]

    def optimizer_state(self) -> np.ndarray | None:
        if self.slow_state is None:
            return None
        torch.cuda.synchronize(self.cache.device)
        return self.slow_state[self.idx_map.rank_of]
