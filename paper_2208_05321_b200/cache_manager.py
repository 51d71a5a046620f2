"""Fast-tier residency management, one batch at a time — on the GPU.

Drop-in for /root/reference/pkg/src/freqcache/cache_manager.py: same names,
signatures, exception classes and results. `prepare_cache` (Alg. 1) runs as one
stream-ordered sequence of sm_100a kernels in libfreqcache_b200 (dedup, rank and
residency lookup, protected static-LFU victim selection, write-back, admission)
with a single host synchronisation to hand back the counts. State lives in HBM;
the attributes tests reach into (`state.slot_to_rank`, `state.dirty`, ...) are
host copies materialised on access.

Index spaces, as in the reference: raw ids (trace values), ranks (slow-tier rows,
frequency order), slots (fast-tier rows).
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .device import DeviceCache
from .errors import BatchExceedsCapacity, InsufficientEvictable, InsufficientFreeSlots  # noqa: F401
from .freq_stats import IdxMap
from .store import FastTierStore, ReferenceStore, SlowTierStore
from .transmitter import TO_FAST, TO_SLOW, Transmitter, TransferReport

EMPTY = -1
ABSENT = -1
WRITE_BACK_MODES = ("dirty_only", "always")
EVICT_MODES = ("occupancy_aware", "paper_literal")


class StaticFreqLfu:
    """Static-frequency LFU: evict the occupied, unprotected rows with the largest
    ranks (cache_manager.py:55-75). Implemented on device by the descending
    compaction of (resident & ~protected) ranks; this object names the policy."""

    name = "freq_lfu"

    def on_reference(self, ranks, multiplicities, batch_seq: int) -> None:
        pass


def _check_policy(policy) -> StaticFreqLfu:
    if policy is None:
        return StaticFreqLfu()
    if getattr(policy, "name", None) not in ("freq_lfu", "rowwise_transfer"):
        raise NotImplementedError(
            f"policy {getattr(policy, 'name', policy)!r}: only the static-frequency LFU runs on device")
    return policy


@dataclass
class CacheEvent:
    """One prepare/warmup decision (cache_manager.py:78-111)."""

    batch_seq: int
    policy: str
    protected_ranks: np.ndarray
    evicted_ranks: np.ndarray
    admitted_ranks: np.ndarray
    hits: int
    misses: int

    def to_json_dict(self) -> dict:
        return {"batch_seq": self.batch_seq, "policy": self.policy, "protected": self.protected_ranks.tolist(),
                "evicted": self.evicted_ranks.tolist(), "admitted": self.admitted_ranks.tolist(),
                "hits": self.hits, "misses": self.misses}

    @classmethod
    def from_json_dict(cls, doc: dict) -> "CacheEvent":
        return cls(int(doc["batch_seq"]), doc["policy"], np.asarray(doc["protected"], dtype=np.int64),
                   np.asarray(doc["evicted"], dtype=np.int64), np.asarray(doc["admitted"], dtype=np.int64),
                   int(doc["hits"]), int(doc["misses"]))


def write_events_jsonl(events, path) -> None:
    with open(path, "w") as fh:
        for ev in events:
            fh.write(json.dumps(ev.to_json_dict()) + "\n")


def read_events_jsonl(path) -> list:
    with open(path) as fh:
        return [CacheEvent.from_json_dict(json.loads(line)) for line in fh if line.strip()]


class CacheState:
    """The slot table and its inverse index (cache_manager.py:126-170), resident on
    the GPU once bound to a `DeviceCache`. Array attributes are host copies."""

    def __init__(self, capacity: int, num_ids: int):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        if capacity > num_ids:
            raise ValueError(f"capacity {capacity} exceeds num_ids {num_ids}")
        self.capacity = int(capacity)
        self.num_ids = int(num_ids)
        self.device: DeviceCache | None = None

    # -- binding ------------------------------------------------------------
    def bind(self, idx_map: IdxMap, slow: SlowTierStore, fast: FastTierStore, transmitter: Transmitter,
             write_back: str = "dirty_only", evict_mode: str = "occupancy_aware", device=None,
             engine: str = "zerocopy") -> DeviceCache:
        """Create the device cache for this state and move the tiers into place:
        slow rows pinned + mapped, fast rows copied into HBM (FastTierStore.slots
        becomes a CUDA tensor view)."""
        if self.device is not None:
            return self.device
        if idx_map.num_ids != self.num_ids:
            raise ValueError("idx_map does not match the state's id space")
        dev = DeviceCache(self.num_ids, self.capacity, fast.embedding_dim, write_back=write_back,
                          evict_mode=evict_mode, buffer_bytes=_device_buffer(transmitter, fast), device=device)
        dev.set_idx_map(idx_map.rank_of)
        slow.pin()
        dev.attach_slow(slow.rows)
        if engine != "zerocopy":
            dev.set_engine(engine)
        init = fast.slots
        if isinstance(init, np.ndarray):
            if np.any(init):
                dev.fast_rows.copy_(dev.torch.from_numpy(np.ascontiguousarray(init, dtype=np.float32)))
        else:
            dev.fast_rows.copy_(init)
        fast.slots = dev.fast_rows
        fast._dev = dev
        self.device = dev
        return dev

    def _need(self) -> DeviceCache:
        if self.device is None:
            raise RuntimeError("CacheState is not bound to a device cache yet")
        return self.device

    # -- host views -----------------------------------------------------------
    @property
    def slot_to_rank(self) -> np.ndarray:
        if self.device is None:
            return np.full(self.capacity, EMPTY, dtype=np.int64)
        return self.device.slot_to_rank.cpu().numpy().astype(np.int64)

    @property
    def rank_to_slot(self) -> np.ndarray:
        if self.device is None:
            return np.full(self.num_ids, ABSENT, dtype=np.int32)
        return self.device.rank_to_slot.cpu().numpy()

    @property
    def dirty(self) -> np.ndarray:
        if self.device is None:
            return np.zeros(self.capacity, dtype=bool)
        return self.device.dirty.cpu().numpy().astype(bool)

    def clear_dirty(self) -> None:
        """Drop every dirty bit without writing back (fault injection in tests)."""
        self._need().dirty.zero_()

    @property
    def free_count(self) -> int:
        return self.capacity if self.device is None else self.device.free_count

    @property
    def occupied_count(self) -> int:
        return self.capacity - self.free_count

    def occupied_slots(self) -> np.ndarray:
        return np.flatnonzero(self.slot_to_rank != EMPTY)

    def occupied_ranks(self) -> np.ndarray:
        s = self.slot_to_rank
        return s[s != EMPTY]

    def free_slots(self) -> np.ndarray:
        return np.flatnonzero(self.slot_to_rank == EMPTY)

    @property
    def index_bytes(self) -> int:
        """Reference-equivalent index footprint (int64 slot table, int32 inverse, bool dirty)."""
        return int(self.capacity * 8 + self.num_ids * 4 + self.capacity)

    def check_invariants(self) -> None:
        s2r = self.slot_to_rank
        r2s = self.rank_to_slot
        occ = s2r != EMPTY
        ranks = s2r[occ]
        if np.unique(ranks).size != ranks.size:
            raise AssertionError("a rank occupies more than one slot")
        if self.free_count != int(np.count_nonzero(~occ)):
            raise AssertionError("free_count out of sync with slot table")
        if not np.array_equal(r2s[ranks], np.flatnonzero(occ).astype(r2s.dtype)):
            raise AssertionError("rank_to_slot is not the inverse of slot_to_rank")
        if np.count_nonzero(r2s != ABSENT) != ranks.size:
            raise AssertionError("rank_to_slot has entries for non-occupied ranks")


class PrepareResult:
    """Residency outcome for one batch (cache_manager.py:173-194). Device tensors
    (`d_*`, int32) feed the lookup/update kernels; the numpy attributes of the
    reference are materialised lazily."""

    def __init__(self, ids, d_ids=None, d_unique_ids=None, d_unique_counts=None, d_unique_ranks=None,
                 d_unique_slots=None, d_inverse=None, hits=0, misses=0, evictions=0, transfer_reports=None):
        self.ids = ids
        self.d_ids = d_ids
        self.d_unique_ids = d_unique_ids
        self.d_unique_counts = d_unique_counts
        self.d_unique_ranks = d_unique_ranks
        self.d_unique_slots = d_unique_slots
        self.d_inverse = d_inverse
        self.hits = int(hits)
        self.misses = int(misses)
        self.evictions = int(evictions)
        self.transfer_reports = list(transfer_reports or [])
        self._host = {}

    def _np(self, name):
        if name not in self._host:
            t = getattr(self, "d_" + name)
            self._host[name] = np.empty(0, dtype=np.int64) if t is None else t.cpu().numpy().astype(np.int64)
        return self._host[name]

    @property
    def num_unique(self) -> int:
        return 0 if self.d_unique_ids is None else int(self.d_unique_ids.numel())

    @property
    def unique_ids(self) -> np.ndarray:
        return self._np("unique_ids")

    @property
    def unique_ranks(self) -> np.ndarray:
        return self._np("unique_ranks")

    @property
    def unique_counts(self) -> np.ndarray:
        return self._np("unique_counts")

    @property
    def unique_slots(self) -> np.ndarray:
        return self._np("unique_slots")

    @property
    def inverse(self) -> np.ndarray:
        return self._np("inverse")

    def d_slots_for_ids(self):
        """Slot of every id in batch order, on device (int64)."""
        return self.d_unique_slots.long()[self.d_inverse.long()]

    def slots_for_ids(self) -> np.ndarray:
        if self.d_inverse is None:
            return np.empty(0, dtype=np.int64)
        return self.d_slots_for_ids().cpu().numpy()

    def slot_of(self) -> dict:
        return {int(i): int(s) for i, s in zip(self.unique_ids, self.unique_slots)}


def _device_buffer(transmitter: Transmitter, fast: FastTierStore) -> int:
    """The staging-buffer bound the device applies. Row-wise moves never stage a row
    (transmitter.py:167-177), so only the block transmitter can refuse a row; and no
    prepare issues a no-op move (the reference skips empty moves), so the row-wise bound
    never binds."""
    b = int(transmitter.buffer.capacity_bytes)
    return b if transmitter.mode == "block" else max(b, fast.embedding_dim * 4)


def _bound(state: CacheState, idx_map, transmitter, slow, fast, write_back="dirty_only",
           evict_mode="occupancy_aware") -> DeviceCache:
    if state.device is None:
        state.bind(idx_map, slow, fast, transmitter, write_back, evict_mode)
    return state.device


def select_evictions(state: CacheState, needed: int, protected_ranks) -> np.ndarray:
    """Slots of the `needed` largest-rank occupied rows outside `protected_ranks`,
    in descending-rank order (cache_manager.py:205-216)."""
    if needed < 0:
        raise ValueError("needed must be >= 0")
    if needed == 0:
        return np.empty(0, dtype=np.int64)
    prot = np.asarray(protected_ranks, dtype=np.int64).reshape(-1)
    return state._need().select_evictions(int(needed), prot)


def prepare_cache(state: CacheState, idx_map: IdxMap, ids, transmitter: Transmitter, slow: SlowTierStore,
                  fast: FastTierStore, *, policy=None, write_back: str = "dirty_only",
                  evict_mode: str = "occupancy_aware", batch_seq: int = 0, event_log: list | None = None
                  ) -> PrepareResult:
    """Make every id of the batch resident and return its slot assignment
    (cache_manager.py:234-348). Raises before any mutation on invalid input."""
    if write_back not in WRITE_BACK_MODES:
        raise ValueError(f"write_back must be one of {WRITE_BACK_MODES}, got {write_back!r}")
    if evict_mode not in EVICT_MODES:
        raise ValueError(f"evict_mode must be one of {EVICT_MODES}, got {evict_mode!r}")
    policy = _check_policy(policy)
    dev = _bound(state, idx_map, transmitter, slow, fast, write_back, evict_mode)
    while dev.prefetch_outstanding:
        # prefetched batches are executed first (their commits, FIFO); when `ids` is one of
        # them (the very object handed to prefetch, or equal contents) its commit is the
        # result, else `ids` is prepared after all of them. Every commit is logged (event +
        # transfer reports) like the prepare it is.
        obj, seq = dev.prefetched_ids(), dev.prefetched_seq()
        res = dev.prepare_commit()
        if dev.committed_matches(ids):
            return _prepare_result(dev, ids, res, transmitter, fast, policy, batch_seq, event_log,
                                   rows_to_slow=dev.last_writebacks())
        _prepare_result(dev, obj, res, transmitter, fast, policy, seq, event_log, rows_to_slow=dev.last_writebacks())
    dev.set_modes(write_back, evict_mode)
    dev.set_buffer_bytes(_device_buffer(transmitter, fast))  # the reference takes the transmitter per call
    return _prepare_result(dev, ids, dev.prepare(ids, batch_seq), transmitter, fast, policy, batch_seq, event_log)


def prefetch_cache(state: CacheState, idx_map: IdxMap, ids, transmitter: Transmitter, slow: SlowTierStore,
                   fast: FastTierStore, *, write_back: str = "dirty_only", evict_mode: str = "occupancy_aware",
                   batch_seq: int = 0) -> None:
    """Start `ids`' prepare ahead of time (extension; the paper's future-work prefetch,
    PAPER.md:490): the index phase and the host -> HBM staging of its misses overlap
    the previous batch's row work. The next prepare_cache call with the same `ids`
    object commits it; the outcome is bit-identical to a plain prepare_cache then."""
    dev = _bound(state, idx_map, transmitter, slow, fast, write_back, evict_mode)
    dev.set_modes(write_back, evict_mode)
    dev.set_buffer_bytes(_device_buffer(transmitter, fast))
    dev.prepare_begin(ids, batch_seq)


def _prepare_result(dev, ids, res, transmitter, fast, policy, batch_seq, event_log, rows_to_slow=None):
    info, uids, ucnt, uranks, uslots, inverse, d_ids = res
    if rows_to_slow is None:
        rows_to_slow = int(info.rows_to_slow)
    if int(d_ids.numel()) == 0:
        return PrepareResult(ids if not hasattr(ids, "shape") else ids, d_ids=d_ids)
    row_bytes = fast.embedding_dim * 4
    reports = []
    if info.evictions:
        reports.append(transmitter.report(TO_SLOW, rows_to_slow, row_bytes)
                       if rows_to_slow else TransferReport.empty(TO_SLOW))
    if info.misses:
        reports.append(transmitter.report(TO_FAST, int(info.misses), row_bytes))
    prep = PrepareResult(ids, d_ids, uids, ucnt, uranks, uslots, inverse, info.hits, info.misses, info.evictions,
                         reports)
    if event_log is not None:
        evicted, admitted = dev.last_events(int(info.evictions), int(info.misses))
        event_log.append(CacheEvent(batch_seq, policy.name, np.sort(prep.unique_ranks), evicted, admitted,
                                    int(info.hits), int(info.misses)))
    return prep


def warmup(state: CacheState, idx_map: IdxMap, k: int, transmitter: Transmitter, slow: SlowTierStore,
           fast: FastTierStore, *, policy=None, event_log: list | None = None) -> TransferReport:
    """Pre-fill an empty cache with ranks 0..k-1 in slots 0..k-1 (cache_manager.py:351-390)."""
    if k < 0 or k > state.capacity:
        raise ValueError(f"warmup k must be in [0, capacity={state.capacity}], got {k}")
    if state.free_count != state.capacity:
        raise ValueError("warmup requires an empty cache")
    if k == 0:
        return TransferReport.empty(TO_FAST)
    report = transmitter.report(TO_FAST, int(k), fast.embedding_dim * 4)
    dev = _bound(state, idx_map, transmitter, slow, fast)
    dev.set_buffer_bytes(_device_buffer(transmitter, fast))
    dev.warmup(int(k))
    if event_log is not None:
        name = policy.name if policy is not None else "warmup"
        ranks = np.arange(k, dtype=np.int64)
        event_log.append(CacheEvent(-1, name, np.empty(0, np.int64), np.empty(0, np.int64), ranks, 0, int(k)))
    return report


def mark_dirty(state: CacheState, slots) -> None:
    """Flag slots as newer than the slow tier (cache_manager.py:393-400)."""
    slots = np.asarray(slots, dtype=np.int64).reshape(-1)
    if slots.size:
        lo, hi = int(slots.min()), int(slots.max())
        if lo < 0 or hi >= state.capacity:
            raise IndexError(f"slot out of range [0, {state.capacity})")
        state._need().mark_dirty(slots)


def flush(state: CacheState, transmitter: Transmitter, slow: SlowTierStore, fast: FastTierStore) -> TransferReport:
    """Write every dirty slot back; rows stay resident, now clean (cache_manager.py:403-415)."""
    if state.device is None:
        return TransferReport.empty(TO_SLOW)
    dev = state.device
    row_bytes = fast.embedding_dim * 4
    if transmitter.mode == "block" and row_bytes > transmitter.buffer.capacity_bytes and int(dev.dirty.sum().item()):
        transmitter.buffer.rows_per_message(row_bytes)  # raises BufferTooSmall before any mutation (:410-413)
    rows = dev.flush()
    if rows == 0:
        return TransferReport.empty(TO_SLOW)
    return transmitter.report(TO_SLOW, rows, row_bytes)


def gather(fast: FastTierStore, prep: PrepareResult):
    """Rows for the batch in id order, duplicates repeated (cache_manager.py:418-420).
    Returns a CUDA tensor [n, dim]."""
    dev = fast._dev
    if prep.d_inverse is None:
        return dev.torch.empty((0, fast.embedding_dim), dtype=dev.torch.float32, device=dev.device)
    return dev.pooled(prep.d_unique_slots, prep.d_inverse, int(prep.d_inverse.numel()))


def _device_rows(dev: DeviceCache, values, shape):
    torch = dev.torch
    if isinstance(values, torch.Tensor):
        t = values.to(device=dev.device, dtype=torch.float32)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(values, dtype=np.float32))).to(dev.device)
    t = t.reshape(shape) if t.numel() == int(np.prod(shape)) else t
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"deltas must be {tuple(shape)}, got {tuple(t.shape)}")
    return t.contiguous()


def scatter_update(state: CacheState, fast: FastTierStore, prep: PrepareResult, deltas) -> None:
    """Per-occurrence deltas accumulated in batch order (bit-exact with np.add.at) and
    every unique slot dirtied, even for zero deltas (cache_manager.py:423-438)."""
    dev = state._need()
    n = 0 if prep.d_inverse is None else int(prep.d_inverse.numel())
    if not hasattr(deltas, "shape") or tuple(deltas.shape) != (n, fast.embedding_dim):
        raise ValueError(f"deltas must be ({n}, {fast.embedding_dim}), got {getattr(deltas, 'shape', None)}")
    if n == 0:
        return
    d = _device_rows(dev, deltas, (n, fast.embedding_dim))
    dev.scatter_update(prep.d_unique_slots, prep.d_inverse, prep.d_unique_counts, d)


class CacheStack:
    """One worker's cache over (a column slice of) the table (cache_manager.py:441-562):
    stores, device state, transmitter accounting, policy, optional dense mirror."""

    def __init__(self, idx_map: IdxMap, slow: SlowTierStore, fast: FastTierStore, transmitter: Transmitter,
                 reference: ReferenceStore | None = None, policy=None, write_back: str = "dirty_only",
                 evict_mode: str = "occupancy_aware", log_events: bool = False, col_range: tuple | None = None,
                 device=None, engine: str = "zerocopy"):
        if slow.embedding_dim != fast.embedding_dim:
            raise ValueError("slow and fast tier column widths differ")
        if write_back not in WRITE_BACK_MODES:
            raise ValueError(f"write_back must be one of {WRITE_BACK_MODES}, got {write_back!r}")
        if evict_mode not in EVICT_MODES:
            raise ValueError(f"evict_mode must be one of {EVICT_MODES}, got {evict_mode!r}")
        self.idx_map = idx_map
        self.slow = slow
        self.fast = fast
        self.reference = reference
        self.transmitter = transmitter
        self.policy = _check_policy(policy)
        self.write_back = write_back
        self.evict_mode = evict_mode
        self.events: list[CacheEvent] | None = [] if log_events else None
        self.col_range = col_range if col_range is not None else (0, slow.embedding_dim)
        self.state = CacheState(fast.capacity, idx_map.num_ids)
        # engine "zerocopy": the slow tier is current after every prepare (reference semantics);
        # "async": write-backs land later, the slow tier is current after flush()
        self.device = self.state.bind(idx_map, slow, fast, transmitter, write_back, evict_mode, device, engine)
        self._colw = {}

    @property
    def capacity(self) -> int:
        return self.fast.capacity

    def warmup(self, k: int) -> TransferReport:
        return warmup(self.state, self.idx_map, k, self.transmitter, self.slow, self.fast, policy=self.policy,
                      event_log=self.events)

    def prepare(self, ids, batch_seq: int) -> PrepareResult:
        return prepare_cache(self.state, self.idx_map, ids, self.transmitter, self.slow, self.fast,
                             policy=self.policy, write_back=self.write_back, evict_mode=self.evict_mode,
                             batch_seq=batch_seq, event_log=self.events)

    def prefetch(self, ids, batch_seq: int) -> None:
        """Start the prepare of the next batch early (see prefetch_cache); the following
        prepare(ids, ...) with the same ids object commits it."""
        prefetch_cache(self.state, self.idx_map, ids, self.transmitter, self.slow, self.fast,
                       write_back=self.write_back, evict_mode=self.evict_mode, batch_seq=batch_seq)

    def gather(self, prep: PrepareResult):
        return gather(self.fast, prep)

    def gather_unique(self, prep: PrepareResult):
        if prep.d_unique_slots is None:
            return self.device.torch.empty((0, self.fast.embedding_dim), device=self.device.device)
        return self.device.gather_rows(prep.d_unique_slots)

    def scatter_update(self, prep: PrepareResult, deltas) -> None:
        scatter_update(self.state, self.fast, prep, deltas)
        if self.reference is not None and prep.d_inverse is not None:
            host = deltas.detach().cpu().numpy() if hasattr(deltas, "detach") else np.asarray(deltas, np.float32)
            np.add.at(self.reference.rows, np.asarray(prep.ids).reshape(-1), host.astype(np.float32))

    def apply_unique_update(self, prep: PrepareResult, add) -> None:
        """fast[unique_slots] += add; dirty (cache_manager.py:517-523)."""
        if prep.num_unique == 0:
            return
        a = _device_rows(self.device, add, (prep.num_unique, self.fast.embedding_dim))
        self.device.unique_add(prep.d_unique_slots, a)
        if self.reference is not None:
            host = a.cpu().numpy()
            self.reference.rows[prep.unique_ids] += host

    def apply_synthetic_update(self, prep: PrepareResult, batch_seq: int, updates_seed: int, col_w) -> None:
        """The simulator's per-batch update (simulator.py:429-433), fused on device:
        fast[slot] += (update_row_scalars(...)[:, None] * col_w[lo:hi])."""
        if prep.num_unique == 0:
            return
        from .updates import batch_salt, update_row_scalars

        lo, hi = self.col_range
        key = (id(col_w), lo, hi)
        if key not in self._colw:
            w = np.ascontiguousarray(np.asarray(col_w, dtype=np.float32)[lo:hi])
            self._colw[key] = self.device.torch.from_numpy(w).to(self.device.device)
        self.device.synthetic(prep.d_unique_ids, prep.d_unique_counts, prep.d_unique_slots,
                              batch_salt(batch_seq, updates_seed), self._colw[key])
        if self.reference is not None:
            g = update_row_scalars(prep.unique_ids, prep.unique_counts, batch_seq, updates_seed)
            self.reference.rows[prep.unique_ids] += g[:, None] * np.asarray(col_w, np.float32)[lo:hi][None, :]

    def flush(self) -> TransferReport:
        rep = flush(self.state, self.transmitter, self.slow, self.fast)
        return rep

    def first_divergence(self, chunk_rows: int = 1 << 16):
        """Bitwise compare of the slow tier with the dense mirror after a flush (:528-551)."""
        if self.reference is None:
            raise ValueError("stack was built without a reference store")
        self.device.torch.cuda.synchronize(self.device.device)
        id_of = self.idx_map.id_of
        for lo in range(0, id_of.size, chunk_rows):
            hi = min(lo + chunk_rows, id_of.size)
            want = self.reference.rows[id_of[lo:hi]]
            got = self.slow.rows[lo:hi]
            if not np.array_equal(got, want):
                off, col = np.argwhere(got != want)[0]
                rank = int(lo + off)
                return {"rank": rank, "id": int(id_of[rank]), "col": int(self.col_range[0] + col),
                        "slow_value": float(got[off, col]), "reference_value": float(want[off, col])}
        return None

    def memory_report(self) -> dict:
        """The reference's report (cache_manager.py:553-562), same keys and formula (the
        simulator's RunMetrics document embeds it): fast rows + the TransferBuffer's
        capacity + the reference's index arrays. What the device cache really allocates is
        `device_memory()`."""
        rows = self.fast.nbytes
        buf = self.transmitter.buffer.capacity_bytes
        index = self.state.index_bytes
        return {"fast_rows_bytes": int(rows), "buffer_bytes": int(buf), "index_bytes": int(index),
                "peak_fast_tier_bytes": int(rows + buf + index)}

    def device_memory(self) -> dict:
        """Every device allocation of this stack's cache by category (fc_memory_bytes):
        fast rows, id-space arrays, bitmaps, slot-space arrays, the HBM staging buffers
        (bounded by buffer_bytes, grown only when a batch needs more), scratch, the 2 MiB
        page slack, and `device_total_bytes` = what the allocations reserve."""
        return self.device.memory()
