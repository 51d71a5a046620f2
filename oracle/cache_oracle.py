"""Numpy restatement of the reference cache path — TEST INFRASTRUCTURE ONLY.

Restates, in its own structure, what `/root/reference/pkg/src/freqcache` computes
on the hot path, so the GPU build can be checked on identical id streams:

* `rank_permutation` / `frequency_counts` — freq_stats.py:97-111, 136-148
* `OracleCache.prepare`   — cache_manager.py:234-348 (Alg. 1)
* `OracleCache.warmup`    — cache_manager.py:351-390
* `OracleCache.flush`     — cache_manager.py:403-415
* `OracleCache.mark_dirty`, `select_evictions`, `gather`, `scatter_update`,
  `apply_unique_update`, `first_divergence` — cache_manager.py:205-216, 393-400,
  418-438, 509-551
* `chunk_messages`        — transmitter.py:97-109, 144-195 (message accounting)
* `fast_capacity`, `init_rows` — store.py:104-131
* `hash_unit`, `row_scalars`, `column_weights` — simulator.py:229-260
* `column_ranges`         — sharding.py:46-59
* `replay_law`            — simulator.py:571-621 (static-frequency policy only)

Plus restatements of semantics the reference does NOT have,
pinned to torch's CPU implementations by tests/golden/make_golden.py:

* `pooled_bag` — `torch.nn.functional.embedding_bag` sum/mean (+ per-sample
  weights for sum); mean with per-sample weights is defined here as
  sum_i(w_i * row_i) / L with an empty bag giving 0 (torch rejects that combo).
* `pooled_bag_backward_rows`, `sparse_sgd`, `sparse_adagrad` — the gradient of the
  pooled output w.r.t. each unique row and torch.optim.SGD / Adagrad updates.

Nothing here is imported by the product package.
"""

from __future__ import annotations

import math
import warnings

import numpy as np

EMPTY = -1
ABSENT = -1
ROW_DTYPE = np.float32


class OracleBatchExceedsCapacity(ValueError):
    pass


class OracleInsufficientEvictable(RuntimeError):
    pass


class OracleInsufficientFreeSlots(RuntimeError):
    pass


class OracleBufferTooSmall(ValueError):
    pass


# --------------------------------------------------------------------------
# static statistics (freq_stats.py)
# --------------------------------------------------------------------------

def frequency_counts(ids, num_ids: int) -> np.ndarray:
    """Dense per-id occurrence counts (freq_stats.py:97-111)."""
    flat = np.asarray(ids).reshape(-1)
    if flat.size and (flat.min() < 0 or flat.max() >= num_ids):
        raise ValueError("id out of range")
    return np.bincount(flat.astype(np.int64), minlength=num_ids).astype(np.int64)


def rank_permutation(counts) -> tuple[np.ndarray, np.ndarray]:
    """(rank_of, id_of): descending count, ties by ascending id (freq_stats.py:136-148).

    Written as a two-key lexsort instead of a stable argsort; the order is the same.
    """
    counts = np.asarray(counts, dtype=np.int64)
    n = counts.size
    if n < 1:
        raise ValueError("num_ids must be >= 1")
    id_of = np.lexsort((np.arange(n, dtype=np.int64), -counts)).astype(np.int64)
    rank_of = np.empty(n, dtype=np.int64)
    rank_of[id_of] = np.arange(n, dtype=np.int64)
    return rank_of, id_of


# --------------------------------------------------------------------------
# stores (store.py)
# --------------------------------------------------------------------------

def fast_capacity(num_ids: int, cache_ratio: float) -> int:
    """floor(ratio * num_ids), clamped to >= 1 with a warning (store.py:104-115)."""
    if not (0.0 < cache_ratio <= 1.0):
        raise ValueError(f"cache_ratio must be in (0, 1], got {cache_ratio}")
    slots = math.floor(cache_ratio * num_ids)
    if slots >= 1:
        return slots
    warnings.warn("capacity rounds to zero slots; clamping to 1", stacklevel=2)
    return 1


def init_rows(num_ids: int, dim: int, seed: int) -> np.ndarray:
    """Seeded uniform(+-0.5/dim) rows in raw-id order (store.py:118-131).

    Filled from one PCG64 stream in 2**24-element pieces, like the reference.
    """
    half = 0.5 / dim
    out = np.empty(num_ids * dim, dtype=ROW_DTYPE)
    gen = np.random.default_rng(seed)
    piece = 1 << 24
    pos = 0
    while pos < out.size:
        end = min(out.size, pos + piece)
        out[pos:end] = gen.uniform(-half, half, end - pos)
        pos = end
    return out.reshape(num_ids, dim)


# --------------------------------------------------------------------------
# transmitter accounting (transmitter.py)
# --------------------------------------------------------------------------

def chunk_messages(rows: int, row_bytes: int, buffer_bytes: int, mode: str = "block") -> int:
    """Messages for `rows` whole rows through a bounded buffer (transmitter.py:97-109).

    Rows never straddle messages, so each message carries floor(buffer/row);
    a row larger than the buffer is an error even when nothing moves
    (transmitter.py:162-164). "rowwise" mode sends one message per row (:167-177).
    """
    if rows < 0 or row_bytes < 1 or buffer_bytes < 1:
        raise ValueError("bad sizes")
    if row_bytes > buffer_bytes:
        raise OracleBufferTooSmall("row does not fit the staging buffer")
    if mode == "rowwise":
        return rows
    per = buffer_bytes // row_bytes
    return -(-rows // per) if rows else 0


# --------------------------------------------------------------------------
# synthetic updates (simulator.py:229-260)
# --------------------------------------------------------------------------

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def hash_unit(values, salt: int) -> np.ndarray:
    """splitmix64 finaliser of (v * golden + salt) -> top 24 bits -> [0,1) float32."""
    with np.errstate(over="ignore"):
        z = np.asarray(values).astype(np.uint64) * _M1 + np.uint64(int(salt) % (1 << 64))
        z = (z ^ (z >> np.uint64(30))) * _M2
        z = (z ^ (z >> np.uint64(27))) * _M3
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / (1 << 24))


def column_weights(dim: int, updates_seed: int) -> np.ndarray:
    return hash_unit(np.arange(dim), updates_seed * 3 + 1) + np.float32(0.5)


def row_scalars(unique_ids, counts, batch_seq: int, updates_seed: int) -> np.ndarray:
    salt = (batch_seq + 1) * 0x9E3779B97F4A7C15 + updates_seed
    base = hash_unit(unique_ids, salt) - np.float32(0.5)
    return base * np.asarray(counts).astype(np.float32)


# --------------------------------------------------------------------------
# column sharding (sharding.py:46-59)
# --------------------------------------------------------------------------

def column_ranges(dim: int, shards: int) -> list[tuple[int, int]]:
    if not (1 <= shards <= dim):
        raise ValueError("bad shard count")
    q, r = divmod(dim, shards)
    bounds = [0]
    for s in range(shards):
        bounds.append(bounds[-1] + q + (s < r))
    return list(zip(bounds[:-1], bounds[1:]))


# --------------------------------------------------------------------------
# the cache (cache_manager.py)
# --------------------------------------------------------------------------

class OracleCache:
    """Host restatement of one CacheStack: slot table, inverse index, dirty bits,
    fast rows, and a rank-indexed slow tier that it mutates in place."""

    def __init__(self, rank_of, slow_rows, capacity: int, *, write_back="dirty_only",
                 evict_mode="occupancy_aware", buffer_bytes=64 * 2**20, mode="block",
                 reference_rows=None):
        self.rank_of = np.asarray(rank_of, dtype=np.int64)
        self.num_ids = int(self.rank_of.size)
        if capacity < 1 or capacity > self.num_ids:
            raise ValueError("bad capacity")
        self.slow = slow_rows
        self.dim = int(slow_rows.shape[1])
        self.capacity = int(capacity)
        self.fast = np.zeros((capacity, self.dim), dtype=ROW_DTYPE)
        self.slot_rank = np.full(capacity, EMPTY, dtype=np.int64)
        self.rank_slot = np.full(self.num_ids, ABSENT, dtype=np.int32)
        self.dirty = np.zeros(capacity, dtype=bool)
        self.free = int(capacity)
        self.write_back = write_back
        self.evict_mode = evict_mode
        self.buffer_bytes = int(buffer_bytes)
        self.mode = mode
        self.reference = reference_rows  # dense, raw-id indexed mirror (store.py:90-101)
        self.events: list[dict] = []

    # -- helpers ---------------------------------------------------------
    def _move_messages(self, rows: int) -> int:
        """Messages of one Transmitter._move (transmitter.py:144-195), raising where it
        raises -- BEFORE any row is copied: a row larger than the buffer is an error for a
        no-op move and for every block-mode move (:162-164, :179 rows_per_message);
        row-wise moves send one message per row and never stage (:167-177)."""
        row_bytes = self.dim * 4
        if (rows == 0 or self.mode == "block") and row_bytes > self.buffer_bytes:
            raise OracleBufferTooSmall(f"row of {row_bytes} B cannot fit in a {self.buffer_bytes} B buffer")
        if rows == 0:
            return 0
        return rows if self.mode == "rowwise" else -(-rows // (self.buffer_bytes // row_bytes))

    def _report(self, direction: str, rows: int) -> dict:
        row_bytes = self.dim * 4
        msgs = self._move_messages(rows)
        return {"direction": direction, "rows": int(rows), "bytes": int(rows * row_bytes), "messages": int(msgs)}

    def _occupied_ranks(self) -> np.ndarray:
        return self.slot_rank[self.slot_rank != EMPTY]

    def _largest_unprotected(self, needed: int, protected) -> np.ndarray:
        """The `needed` largest occupied ranks outside `protected`, descending
        (StaticFreqLfu.victim_ranks, cache_manager.py:67-75)."""
        occ = self._occupied_ranks()
        pool = occ[~np.isin(occ, np.asarray(protected, dtype=np.int64))]
        if needed > pool.size:
            raise OracleInsufficientEvictable(f"need {needed} victims, {pool.size} evictable")
        if needed == 0:
            return np.empty(0, dtype=np.int64)
        return np.sort(pool)[::-1][:needed].copy()

    # -- verbs -----------------------------------------------------------
    def prepare(self, ids, batch_seq: int = 0) -> dict:
        if self.write_back not in ("dirty_only", "always"):
            raise ValueError("bad write_back")
        if self.evict_mode not in ("occupancy_aware", "paper_literal"):
            raise ValueError("bad evict_mode")
        flat = np.asarray(ids).reshape(-1)
        none = np.empty(0, dtype=np.int64)
        if flat.size == 0:
            return {"ids": flat, "unique_ids": none, "unique_ranks": none, "unique_counts": none,
                    "unique_slots": none, "hits": 0, "misses": 0, "evictions": 0, "reports": [],
                    "evicted": none, "admitted": none}
        lo, hi = int(flat.min()), int(flat.max())
        if lo < 0 or hi >= self.num_ids:
            bad = lo if lo < 0 else hi
            raise ValueError(f"id out of range: {bad} not in [0, {self.num_ids})")
        uniq, counts = np.unique(flat, return_counts=True)
        if uniq.size > self.capacity:
            raise OracleBatchExceedsCapacity(f"{uniq.size} unique ids > capacity {self.capacity}")
        ranks = self.rank_of[uniq]
        where = self.rank_slot[ranks].astype(np.int64)
        missing = where == ABSENT
        n_miss = int(missing.sum())
        n_hit = int(uniq.size - n_miss)
        if self.evict_mode == "occupancy_aware":
            needed = max(0, n_miss - self.free)
        else:
            needed = max(0, int(uniq.size) - self.capacity)
        reports = []
        evicted = np.empty(0, dtype=np.int64)
        if needed:
            evicted = self._largest_unprotected(needed, ranks)
            vslots = self.rank_slot[evicted].astype(np.int64)
            wb = vslots if self.write_back == "always" else vslots[self.dirty[vslots]]
            if wb.size:  # _write_back skips the move (and its buffer check) when no victim is dirty (:227-230)
                rep = self._report("to_slow", wb.size)  # raises before any mutation
                self.slow[self.slot_rank[wb]] = self.fast[wb]
                reports.append(rep)
            else:
                reports.append({"direction": "to_slow", "rows": 0, "bytes": 0, "messages": 0})
            self.slot_rank[vslots] = EMPTY
            self.rank_slot[evicted] = ABSENT
            self.dirty[vslots] = False
            self.free += needed
        admitted = np.sort(ranks[missing])
        if n_miss:
            empties = np.nonzero(self.slot_rank == EMPTY)[0]
            if empties.size < n_miss:
                raise OracleInsufficientFreeSlots(f"{n_miss} to admit, {empties.size} free")
            tgt = empties[:n_miss]
            rep = self._report("to_fast", n_miss)  # raises after the evictions above were applied
            self.fast[tgt] = self.slow[admitted]
            reports.append(rep)
            self.slot_rank[tgt] = admitted
            self.rank_slot[admitted] = tgt.astype(np.int32)
            self.dirty[tgt] = False
            self.free -= n_miss
        slots = self.rank_slot[ranks].astype(np.int64)
        self.events.append({"batch_seq": batch_seq, "protected": np.sort(ranks), "evicted": evicted,
                            "admitted": admitted, "hits": n_hit, "misses": n_miss})
        return {"ids": flat, "unique_ids": uniq.astype(np.int64), "unique_ranks": ranks,
                "unique_counts": counts.astype(np.int64), "unique_slots": slots, "hits": n_hit,
                "misses": n_miss, "evictions": int(needed), "reports": reports,
                "evicted": evicted, "admitted": admitted}

    def warmup(self, k: int) -> dict:
        if k < 0 or k > self.capacity:
            raise ValueError(f"warmup k must be in [0, capacity={self.capacity}], got {k}")
        if self.free != self.capacity:
            raise ValueError("warmup requires an empty cache")
        if k == 0:
            return {"direction": "to_fast", "rows": 0, "bytes": 0, "messages": 0}
        r = np.arange(k, dtype=np.int64)
        rep = self._report("to_fast", k)
        self.fast[:k] = self.slow[:k]
        self.slot_rank[:k] = r
        self.rank_slot[:k] = r.astype(np.int32)
        self.dirty[:k] = False
        self.free -= k
        self.events.append({"batch_seq": -1, "protected": np.empty(0, np.int64),
                            "evicted": np.empty(0, np.int64), "admitted": r, "hits": 0, "misses": k})
        return rep

    def mark_dirty(self, slots) -> None:
        s = np.asarray(slots, dtype=np.int64).reshape(-1)
        if s.size and (s.min() < 0 or s.max() >= self.capacity):
            raise IndexError(f"slot out of range [0, {self.capacity})")
        self.dirty[s] = True

    def flush(self) -> dict:
        ds = np.nonzero(self.dirty)[0]
        if ds.size == 0:
            return {"direction": "to_slow", "rows": 0, "bytes": 0, "messages": 0}
        rep = self._report("to_slow", ds.size)
        self.slow[self.slot_rank[ds]] = self.fast[ds]
        self.dirty[ds] = False
        return rep

    def select_evictions(self, needed: int, protected) -> np.ndarray:
        if needed < 0:
            raise ValueError("needed must be >= 0")
        if needed == 0:
            return np.empty(0, dtype=np.int64)
        victims = self._largest_unprotected(needed, np.asarray(protected).reshape(-1))
        return self.rank_slot[victims].astype(np.int64)

    @staticmethod
    def occurrence_slots(prep: dict) -> np.ndarray:
        """Slot per id in batch order (PrepareResult.slots_for_ids, :187-190)."""
        if prep["ids"].size == 0:
            return np.empty(0, dtype=np.int64)
        return prep["unique_slots"][np.searchsorted(prep["unique_ids"], prep["ids"])]

    def gather(self, prep: dict) -> np.ndarray:
        return self.fast[self.occurrence_slots(prep)]

    def gather_unique(self, prep: dict) -> np.ndarray:
        return self.fast[prep["unique_slots"]]

    def scatter_update(self, prep: dict, deltas) -> None:
        d = np.asarray(deltas, dtype=ROW_DTYPE)
        if d.shape != (prep["ids"].size, self.dim):
            raise ValueError("bad deltas shape")
        np.add.at(self.fast, self.occurrence_slots(prep), d)
        self.dirty[prep["unique_slots"]] = True
        if self.reference is not None:
            np.add.at(self.reference, prep["ids"], d)

    def apply_unique_update(self, prep: dict, add) -> None:
        self.fast[prep["unique_slots"]] += add
        self.dirty[prep["unique_slots"]] = True
        if self.reference is not None:
            self.reference[prep["unique_ids"]] += add

    def first_divergence(self, id_of) -> dict | None:
        """Bitwise compare of the slow tier with the dense mirror (:528-551)."""
        want = self.reference[np.asarray(id_of)]
        bad = np.argwhere(self.slow != want)
        if bad.size == 0:
            return None
        r, c = (int(v) for v in bad[0])
        return {"rank": r, "id": int(id_of[r]), "col": c,
                "slow_value": float(self.slow[r, c]), "reference_value": float(want[r, c])}

    def check_invariants(self) -> None:
        occ = self.slot_rank != EMPTY
        r = self.slot_rank[occ]
        assert np.unique(r).size == r.size
        assert self.free == int((~occ).sum())
        assert np.array_equal(self.rank_slot[r], np.nonzero(occ)[0].astype(np.int32))
        assert int((self.rank_slot != ABSENT).sum()) == r.size


def replay_law(events: list, num_ids: int) -> list:
    """Static-frequency eviction law replay (simulator.py:571-621, freq_lfu branch)."""
    resident = np.zeros(num_ids, dtype=bool)
    bad = []
    for i, ev in enumerate(events):
        ev_evicted = np.asarray(ev["evicted"], dtype=np.int64)
        if ev_evicted.size:
            prot = np.asarray(ev["protected"], dtype=np.int64)
            if np.intersect1d(prot, ev_evicted).size:
                bad.append({"event": i, "kind": "protected_evicted"})
            pool = np.nonzero(resident)[0]
            pool = pool[~np.isin(pool, prot)]
            want = np.sort(pool)[pool.size - ev_evicted.size:]
            if not np.array_equal(want, np.sort(ev_evicted)):
                bad.append({"event": i, "kind": "wrong_victims"})
            resident[ev_evicted] = False
        resident[np.asarray(ev["admitted"], dtype=np.int64)] = True
    return bad


# --------------------------------------------------------------------------
# pooled EmbeddingBag and sparse optimisers (not in the reference)
# --------------------------------------------------------------------------

def _bag_layout(offsets, n: int, include_last_offset: bool):
    """(bag_of, pos, lens): for every pooled position, its bag and its index into
    `indices`; bags are [offsets[b], offsets[b+1]) with the last ending at n
    (or at offsets[-1] when include_last_offset)."""
    off = np.asarray(offsets, dtype=np.int64).reshape(-1)
    if include_last_offset:
        starts, ends = off[:-1], off[1:]
    else:
        starts, ends = off, np.append(off[1:], n)
    lens = ends - starts
    total = int(lens.sum())
    bag_of = np.repeat(np.arange(starts.size), lens)
    first = np.cumsum(lens) - lens
    pos = np.arange(total, dtype=np.int64) - np.repeat(first, lens) + np.repeat(starts, lens)
    return bag_of, pos, lens


def pooled_bag(rows, indices, offsets, per_sample_weights=None, mode: str = "sum",
               include_last_offset: bool = False) -> np.ndarray:
    """out[b] = sum_{j in bag b} w_j * rows[indices[j]]  (mode 'sum'), divided by the
    bag length for mode 'mean' (empty bag -> 0). Accumulated in float64."""
    if mode not in ("sum", "mean"):
        raise ValueError("mode must be 'sum' or 'mean'")
    idx = np.asarray(indices, dtype=np.int64).reshape(-1)
    bag_of, pos, lens = _bag_layout(offsets, idx.size, include_last_offset)
    rows64 = np.asarray(rows, dtype=np.float64)
    contrib = rows64[idx[pos]]
    if per_sample_weights is not None:
        contrib = contrib * np.asarray(per_sample_weights, dtype=np.float64).reshape(-1)[pos][:, None]
    out = np.zeros((lens.size, rows64.shape[1]), dtype=np.float64)
    np.add.at(out, bag_of, contrib)
    if mode == "mean":
        out = np.divide(out, lens[:, None].astype(np.float64), out=np.zeros_like(out),
                        where=lens[:, None] > 0)
    return out.astype(np.float32)


def pooled_bag_backward_rows(grad_out, indices, offsets, num_rows: int, per_sample_weights=None,
                             mode: str = "sum", include_last_offset: bool = False) -> np.ndarray:
    """d(loss)/d(rows[r]) for every row r (dense [num_rows, D], float64)."""
    idx = np.asarray(indices, dtype=np.int64).reshape(-1)
    bag_of, pos, lens = _bag_layout(offsets, idx.size, include_last_offset)
    g = np.asarray(grad_out, dtype=np.float64)
    coef = np.ones(pos.size, dtype=np.float64)
    if mode == "mean":
        coef = coef / lens[bag_of]
    if per_sample_weights is not None:
        coef = coef * np.asarray(per_sample_weights, dtype=np.float64).reshape(-1)[pos]
    out = np.zeros((num_rows, g.shape[1]), dtype=np.float64)
    np.add.at(out, idx[pos], g[bag_of] * coef[:, None])
    return out


def sparse_sgd(rows, touched, grad_rows, lr: float) -> None:
    """torch.optim.SGD on the touched rows: w -= lr * g."""
    rows[touched] = (rows[touched].astype(np.float64) - lr * grad_rows[touched]).astype(np.float32)


def sparse_adagrad(rows, state, touched, grad_rows, lr: float, eps: float = 1e-10) -> None:
    """torch.optim.Adagrad (lr_decay=0, wd=0, init acc=0) on the touched rows:
    G += g^2; w -= lr * g / (sqrt(G) + eps)."""
    g = grad_rows[touched]
    s = state[touched].astype(np.float64) + g * g
    state[touched] = s.astype(np.float32)
    rows[touched] = (rows[touched].astype(np.float64) - lr * g / (np.sqrt(s) + eps)).astype(np.float32)
