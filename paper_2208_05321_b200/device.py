"""`DeviceCache`: the Python owner of one libfreqcache_b200 handle.

Thin ctypes plumbing: torch supplies device memory for per-call outputs, the
current CUDA stream and zero-copy tensor views of the handle's HBM state; all
cache computation happens in the library's sm_100a kernels.
"""

from __future__ import annotations

import collections
import ctypes
import os

import numpy as np

from . import _lib
from .errors import check


class _CudaArray:
    """`__cuda_array_interface__` wrapper so torch can view handle-owned memory."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self._owner = owner  # keeps the handle (and its memory) alive
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


_RAW_STREAM = None


def _raw_stream(index) -> int:
    """Raw handle of the current CUDA stream of device `index` (None: the current device)."""
    global _RAW_STREAM
    if _RAW_STREAM is None:
        import torch

        _RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None) or (
            lambda i: torch.cuda.current_stream(i).cuda_stream)  # older torch: the public (slower) path
    if index is None:
        import torch

        index = torch.cuda.current_device()
    return _RAW_STREAM(index)


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


class DeviceCache:
    """One device-resident cache (a CacheStack's state + fast tier) on one GPU."""

    def __init__(self, num_ids: int, capacity: int, dim: int, *, state_width: int = 0,
                 write_back: str = "dirty_only", evict_mode: str = "occupancy_aware",
                 buffer_bytes: int = 64 * 2**20, device=None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("freqcache_b200 needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        self.lib = _lib.load()
        self.num_ids, self.capacity, self.dim, self.state_width = int(num_ids), int(capacity), int(dim), int(state_width)
        self.write_back, self.evict_mode = write_back, evict_mode
        self.buffer_bytes = int(buffer_bytes)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(self.lib.fc_create(self.num_ids, self.capacity, self.dim, self.state_width,
                                     _lib.WB[write_back], _lib.EVICT[evict_mode], self.buffer_bytes,
                                     self.device.index, ctypes.byref(h)))
        self.h = h
        v = _lib.Views()
        check(self.lib.fc_get_views(self.h, ctypes.byref(v)))
        dev = self.device

        def view(ptr, shape, typestr):
            return torch.as_tensor(_CudaArray(ptr, shape, typestr, self), device=dev)

        self.fast_rows = view(v.fast_rows, (self.capacity, self.dim), "<f4")
        self.fast_state = view(v.fast_state, (self.capacity, self.state_width), "<f4") if self.state_width else None
        self.slot_to_rank = view(v.slot_to_rank, (self.capacity,), "<i4")
        self.rank_to_slot = view(v.rank_to_slot, (self.num_ids,), "<i4")
        self.dirty = view(v.dirty, (self.capacity,), "|u1")
        self.rank_of = view(v.rank_of, (self.num_ids,), "<i4")
        self._slow = None
        self._slow_state = None
        # prefetch pipeline: outputs in a ring of buffer sets owned by the cache (valid until
        # PF_RING further prefetches; set by CachedEmbeddingBag, whose per-batch results die
        # with the batch's backward) or freshly allocated per call (CacheStack results may
        # be kept by the caller)
        self.prefetch_ring = False
        # prefetch pipeline: run the index phase on the caller's stream (serialised with
        # the forward/backward; only the miss staging overlaps) or on a side stream
        self.index_on_main = os.environ.get("FC_INDEX_ON_MAIN", "0") == "1"

    # ------------------------------------------------------------------ plumbing
    def stream(self):
        # the raw handle of the current stream (torch.cuda.current_stream builds a Stream object
        # and re-parses the device on every call: ~10 us of host time per call on this path)
        return ctypes.c_void_p(_raw_stream(self.device.index))

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.fc_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_modes(self, write_back: str, evict_mode: str) -> None:
        if (write_back, evict_mode) != (self.write_back, self.evict_mode):
            check(self.lib.fc_set_modes(self.h, _lib.WB[write_back], _lib.EVICT[evict_mode]))
            self.write_back, self.evict_mode = write_back, evict_mode

    def set_buffer_bytes(self, buffer_bytes: int) -> None:
        """Staging-buffer size of the transmitter this call uses (BufferTooSmall + accounting)."""
        if int(buffer_bytes) != self.buffer_bytes:
            check(self.lib.fc_set_buffer_bytes(self.h, int(buffer_bytes)))
            self.buffer_bytes = int(buffer_bytes)

    @property
    def free_count(self) -> int:
        return int(self.lib.fc_free_count(self.h))

    def set_engine(self, engine: str) -> None:
        """'zerocopy' (paired SM-issued transfers, slow tier current after every prepare)
        or 'async' (copy-engine write-back + host scatter; current after flush/drain)."""
        check(self.lib.fc_set_engine(self.h, {"zerocopy": 0, "async": 1}[engine]))
        self.engine = engine

    def drain(self) -> None:
        """Wait until every queued write-back has landed in the slow tier."""
        check(self.lib.fc_drain(self.h))

    def drain_stream(self, stream=None) -> None:
        """A stream-ordered drain: later work on `stream` (default: current) runs once every
        queued write-back has landed in the slow tier."""
        s = self.stream() if stream is None else ctypes.c_void_p(stream.cuda_stream)
        if getattr(self.lib, "fc_drain_stream", None) is None:  # an older A/B build (FC_LIB_PATH)
            return
        check(self.lib.fc_drain_stream(self.h, s))

    def profile(self, enable: bool) -> dict:
        """Toggle per-kernel CUDA-event timing; returns (and resets) the totals so far."""
        out = (ctypes.c_double * 12)()
        check(self.lib.fc_profile(self.h, int(bool(enable)), out))
        return {"prepare_ms": out[0], "transfer_ms": out[1], "calls": int(out[2]), "host_link_bytes": out[3],
                "victim_bytes": out[4], "host_wait_ms": out[5], "scatter_ms": out[6], "scatter_jobs": int(out[7]),
                "transfer_launches": int(out[8]), "writeback_rows": int(out[9]), "writeback_d2h_bytes": out[10],
                "scatter_threads": int(out[11])}

    def trace(self, enable: bool) -> None:
        """Timeline tracing of the pipeline (fc_trace)."""
        check(self.lib.fc_trace(self.h, int(bool(enable))))

    def trace_mark(self, tag: int, stream=None) -> None:
        s = self.stream() if stream is None else ctypes.c_void_p(stream.cuda_stream)
        check(self.lib.fc_trace_mark(self.h, int(tag), s))

    def trace_read(self, max_events: int = 100000):
        tags = np.zeros(max_events, np.int32)
        ms = np.zeros(max_events, np.float64)
        n = int(self.lib.fc_trace_read(self.h, tags.ctypes.data_as(ctypes.c_void_p), ms.ctypes.data_as(ctypes.c_void_p),
                                       max_events))
        return tags[:n], ms[:n]

    def to_device_ids(self, ids):
        """Accept numpy / list / torch ids; return a contiguous CUDA int64/int32 tensor."""
        torch = self.torch
        if isinstance(ids, torch.Tensor):
            t = ids.reshape(-1)
            if t.dtype not in (torch.int64, torch.int32):
                t = t.to(torch.int64)
            return t.to(self.device, non_blocking=True).contiguous()
        a = np.asarray(ids).reshape(-1)
        if a.dtype not in (np.int64, np.int32):
            a = a.astype(np.int64)
        return torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    # ------------------------------------------------------------------ setup
    def set_idx_map(self, rank_of: np.ndarray) -> None:
        r = np.ascontiguousarray(np.asarray(rank_of, dtype=np.int64))
        if r.shape != (self.num_ids,):
            raise ValueError(f"rank_of must have {self.num_ids} entries")
        check(self.lib.fc_set_idx_map(self.h, r.ctypes.data_as(ctypes.c_void_p), self.stream()))

    def attach_slow(self, rows: np.ndarray, state_rows: np.ndarray | None = None) -> None:
        if rows.dtype != np.float32 or rows.shape[1] != self.dim or rows.shape[0] != self.num_ids:
            raise ValueError("slow tier must be float32 [num_ids, dim]")
        ld = rows.strides[0] // 4
        sp, sld = None, 0
        if state_rows is not None:
            sp, sld = state_rows.ctypes.data_as(ctypes.c_void_p), state_rows.strides[0] // 4
        check(self.lib.fc_attach_slow_tier(self.h, rows.ctypes.data_as(ctypes.c_void_p), ld, sp, sld))
        self._slow, self._slow_state = rows, state_rows  # keep the host buffers alive

    # ------------------------------------------------------------------ verbs
    def warmup(self, k: int) -> None:
        check(self.lib.fc_warmup(self.h, int(k), self.stream()))

    def prepare(self, ids, batch_seq: int = 0):
        """Run prepare_cache on device. Returns (info, uids, ucnt, uranks, uslots, inverse, d_ids)."""
        torch = self.torch
        d_ids = self.to_device_ids(ids)
        n = int(d_ids.numel())
        k = min(n, self.capacity)
        buf = torch.empty(4 * k + n, dtype=torch.int32, device=self.device)
        uids, ucnt, uranks, uslots = buf[:k], buf[k:2 * k], buf[2 * k:3 * k], buf[3 * k:4 * k]
        inverse = buf[4 * k:]
        info = _lib.PrepareInfo()
        rc = self.lib.fc_prepare(self.h, ctypes.c_void_p(_ptr(d_ids)), d_ids.element_size(), n, int(batch_seq),
                                 ctypes.c_void_p(_ptr(uids)), ctypes.c_void_p(_ptr(ucnt)),
                                 ctypes.c_void_p(_ptr(uranks)), ctypes.c_void_p(_ptr(uslots)),
                                 ctypes.c_void_p(_ptr(inverse)), self.stream(), ctypes.byref(info))
        check(rc)
        u = int(info.unique)
        return info, uids[:u], ucnt[:u], uranks[:u], uslots[:u], inverse, d_ids

    # ------------------------------------------------------------------ prefetch pipeline
    @property
    def prefetch_outstanding(self) -> bool:
        return bool(getattr(self, "_pfq", None))

    @property
    def prefetch_depth(self) -> int:
        """Prefetched prepares begun and not yet committed (0, 1 or 2)."""
        return len(getattr(self, "_pfq", ()))

    def prepare_begin(self, ids, batch_seq: int = 0, index_on_main: bool | None = None, ready=None, consumer=None):
        """Launch the next batch's prepare ahead of time (fc_prepare_begin): the index
        phase runs on this cache's index stream and the admitted rows are staged
        host -> HBM on the library's transfer stream, both overlapping whatever the
        current stream is still running (the previous batch's forward/backward).
        The result is claimed with prepare_commit().

        Host ids are copied on the index stream. Device ids are read there once the
        work queued so far on the current stream is done (they may be its output),
        or, when `ready` (a torch.cuda.Event) is given, once that event has fired --
        pass it for ids that were complete earlier, so the index phase does not wait
        for this batch's queued forward. `consumer` is the stream that will use the
        results after the commit (default: the current stream); the per-batch buffers
        are recorded on it so the allocator cannot hand them out while it still reads
        them (a caller that begins on a side stream passes its main stream here).

        Up to two prepares may be outstanding (commits are FIFO): calling
        prepare_begin(t+1) before prepare_commit(t) lets batch t+1's index phase start
        on the device as soon as batch t's has ended, instead of after the host has
        committed t; its staging is launched by that commit."""
        torch = self.torch
        if self.prefetch_depth >= 2:
            raise RuntimeError("two prefetched prepares are outstanding: commit one first")
        if getattr(self, "index_stream", None) is None:
            # highest priority: the index phase is short but on the pipeline's critical
            # path, and must not queue behind the previous batch's backward blocks
            self.index_stream = torch.cuda.Stream(self.device, priority=-100)
        main = torch.cuda.current_stream(self.device.index)  # orders device ids
        consumer = main if consumer is None else consumer
        if index_on_main is None:
            index_on_main = self.index_on_main
        idx = main if index_on_main else self.index_stream
        if idx is not main and isinstance(ids, torch.Tensor) and ids.is_cuda:
            if ready is None:
                idx.wait_stream(main)
            else:
                idx.wait_event(ready)
        slot = self._ring_slot(ids) if self.prefetch_ring else None
        if slot is not None:
            # a ring of PF_RING buffer sets owned by this cache: no per-step allocation (a
            # cudaMalloc inside a training loop stalls the host for tens of ms). A set is
            # rewritten PF_RING prefetches later, when the pipeline's event order has put
            # its previous batch's backward behind us (see prefetch_ring)
            buf, d_ids = slot
            n = int(ids.numel())
            if ids.is_cuda and ids.device == self.device and ids.is_contiguous():
                # device ids are read in place (the ordering above makes them complete; the
                # caller must not rewrite them before the commit): no copy on the critical
                # path, where it would queue behind the write-back on the copy engines
                d_ids = ids.reshape(-1)
                if idx is not main:
                    d_ids.record_stream(idx)
            else:
                with torch.cuda.stream(idx):
                    d_ids = d_ids[:n]
                    d_ids.copy_(ids.reshape(-1), non_blocking=True)
            k = min(n, self.capacity)
            buf = buf[:4 * k + n]
        else:
            with torch.cuda.stream(idx):
                # allocated on the index stream (no reuse hazard with blocks main still uses),
                # then marked as used by main, which consumes them after the commit
                d_ids = self.to_device_ids(ids)
                n = int(d_ids.numel())
                if n == 0:
                    raise ValueError("prefetch needs a non-empty batch")
                k = min(n, self.capacity)
                buf = torch.empty(4 * k + n, dtype=torch.int32, device=self.device)
            for st_ in {main, consumer}:
                d_ids.record_stream(st_)
                buf.record_stream(st_)
        check(self.lib.fc_prepare_begin(self.h, ctypes.c_void_p(_ptr(d_ids)), d_ids.element_size(), n, int(batch_seq),
                                        ctypes.c_void_p(_ptr(buf[:k])), ctypes.c_void_p(_ptr(buf[k:2 * k])),
                                        ctypes.c_void_p(_ptr(buf[2 * k:3 * k])),
                                        ctypes.c_void_p(_ptr(buf[3 * k:4 * k])), ctypes.c_void_p(_ptr(buf[4 * k:])),
                                        ctypes.c_void_p(idx.cuda_stream)))
        if not hasattr(self, "_pfq"):
            self._pfq = collections.deque()
        self._pfq.append((buf, k, d_ids, ids, int(batch_seq)))

    PF_RING = 3

    def _ring_slot(self, ids):
        """Next buffer set of the prefetch ring, (re)allocated when the batch outgrows it;
        None for inputs the ring does not take (non-tensor or empty ids)."""
        torch = self.torch
        if not isinstance(ids, torch.Tensor) or ids.numel() == 0 or ids.dtype not in (torch.int32, torch.int64):
            return None
        n = int(ids.numel())
        ring = getattr(self, "_ring", None)
        if ring is None or ring["n"] < n or ring["dtype"] != ids.dtype:
            torch.cuda.synchronize(self.device)  # nothing in flight still uses the old ring
            k = min(n, self.capacity)
            ring = {"n": n, "dtype": ids.dtype, "i": 0,
                    "sets": [(torch.empty(4 * k + n, dtype=torch.int32, device=self.device),
                              torch.empty(n, dtype=ids.dtype, device=self.device)) for _ in range(self.PF_RING)]}
            self._ring = ring
        s = ring["sets"][ring["i"] % self.PF_RING]
        ring["i"] += 1
        return s

    def prepare_commit(self):
        """Finish the outstanding prefetch on the current stream (fc_prepare_commit).
        Returns what prepare() returns; info.rows_to_slow is -1 (decided on device)."""
        if not self.prefetch_outstanding:
            raise RuntimeError("no prefetched prepare to commit")
        buf, k, d_ids, obj, _ = self._pfq.popleft()  # the oldest (fc_prepare_commit's order)
        self._last_pf = (obj, d_ids)
        info = _lib.PrepareInfo()
        check(self.lib.fc_prepare_commit(self.h, self.stream(), ctypes.byref(info)))
        u = int(info.unique)
        return info, buf[:u], buf[k:k + u], buf[2 * k:2 * k + u], buf[3 * k:3 * k + u], buf[4 * k:], d_ids

    MEM_FIELDS = ("fast_rows_bytes", "id_space_bytes", "bitmap_bytes", "slot_space_bytes", "staging_bytes",
                  "scratch_bytes", "allocation_slack_bytes", "device_total_bytes", "pinned_staging_bytes",
                  "wb_stage_rows", "admission_stage_rows")

    def memory(self) -> dict:
        """Every device allocation of this cache by category (fc_memory_bytes), plus the
        pinned host staging and the current staging row counts."""
        out = (ctypes.c_int64 * len(self.MEM_FIELDS))()
        check(self.lib.fc_memory_bytes(self.h, out, len(self.MEM_FIELDS)))
        return {k: int(v) for k, v in zip(self.MEM_FIELDS, out)}

    def last_writebacks(self) -> int:
        """Rows written back by the last commit (waits for its kernels)."""
        v = ctypes.c_int64()
        check(self.lib.fc_last_writebacks(self.h, ctypes.byref(v)))
        return int(v.value)

    def prefetched_ids(self):
        """The ids object of the oldest outstanding prepare_begin, the next one to be
        committed (or None)."""
        return self._pfq[0][3] if self.prefetch_outstanding else None

    def prefetched_seq(self):
        """The batch_seq of the oldest outstanding prepare_begin (or None)."""
        return self._pfq[0][4] if self.prefetch_outstanding else None

    def committed_matches(self, ids) -> bool:
        """After prepare_commit: was the committed batch `ids`? Same object, or equal
        contents (compared after the commit, so the index stream's copy is complete)."""
        pf = getattr(self, "_last_pf", None)
        if pf is None:
            return False
        obj, d_ids = pf
        if obj is ids:
            return True
        torch = self.torch
        b = ids if isinstance(ids, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(ids))
        if b.numel() != d_ids.numel():
            return False
        return bool(torch.equal(d_ids.reshape(-1).long(), b.reshape(-1).to(d_ids.device).long()))

    def last_events(self, evictions: int, misses: int):
        ev = np.empty(evictions, dtype=np.int64)
        ad = np.empty(misses, dtype=np.int64)
        check(self.lib.fc_last_events(self.h, ev.ctypes.data_as(ctypes.c_void_p),
                                      ad.ctypes.data_as(ctypes.c_void_p), self.stream()))
        return ev, ad

    def flush(self) -> int:
        rows = ctypes.c_int64()
        check(self.lib.fc_flush(self.h, self.stream(), ctypes.byref(rows)))
        return int(rows.value)

    def mark_dirty(self, slots: np.ndarray) -> None:
        d = self.torch.from_numpy(np.ascontiguousarray(slots, dtype=np.int64)).to(self.device)
        check(self.lib.fc_mark_dirty(self.h, ctypes.c_void_p(_ptr(d)), int(d.numel()), self.stream()))

    def select_evictions(self, needed: int, protected: np.ndarray) -> np.ndarray:
        p = self.torch.from_numpy(np.ascontiguousarray(protected, dtype=np.int64)).to(self.device)
        out = np.empty(max(needed, 0), dtype=np.int64)
        check(self.lib.fc_select_evictions(self.h, int(needed), ctypes.c_void_p(_ptr(p)), int(p.numel()),
                                           out.ctypes.data_as(ctypes.c_void_p), self.stream()))
        return out

    def pooled(self, uslots, inverse, n: int, offsets=None, n_bags: int | None = None, include_last_offset=False,
               per_sample_weights=None, mode: str = "sum", out=None):
        torch = self.torch
        if offsets is None:
            n_bags = n
        elif n_bags is None:
            n_bags = int(offsets.numel()) - (1 if include_last_offset else 0)
        if out is None:
            out = torch.empty((n_bags, self.dim), dtype=torch.float32, device=self.device)
        check(self.lib.fc_pooled_forward(self.h, ctypes.c_void_p(_ptr(uslots)), ctypes.c_void_p(_ptr(inverse)), n,
                                         ctypes.c_void_p(_ptr(offsets)), 0 if offsets is None else offsets.element_size(),
                                         n_bags, int(bool(include_last_offset)),
                                         ctypes.c_void_p(_ptr(per_sample_weights)), _lib.POOL[mode],
                                         ctypes.c_void_p(_ptr(out)), self.stream()))
        return out

    def gather_rows(self, slots):
        out = self.torch.empty((int(slots.numel()), self.dim), dtype=self.torch.float32, device=self.device)
        check(self.lib.fc_gather_rows(self.h, ctypes.c_void_p(_ptr(slots)), int(slots.numel()),
                                      ctypes.c_void_p(_ptr(out)), self.stream()))
        return out

    def unique_add(self, uslots, add) -> None:
        check(self.lib.fc_apply_unique_update(self.h, ctypes.c_void_p(_ptr(uslots)), int(uslots.numel()),
                                              ctypes.c_void_p(_ptr(add)), self.stream()))

    def synthetic(self, uids, ucnt, uslots, salt: int, colw) -> None:
        check(self.lib.fc_apply_synthetic_update(self.h, ctypes.c_void_p(_ptr(uids)), ctypes.c_void_p(_ptr(ucnt)),
                                                 ctypes.c_void_p(_ptr(uslots)), int(uslots.numel()),
                                                 ctypes.c_uint64(int(salt) % (1 << 64)),
                                                 ctypes.c_void_p(_ptr(colw)), self.stream()))

    def scatter_update(self, uslots, inverse, ucnt, deltas) -> None:
        check(self.lib.fc_scatter_update(self.h, ctypes.c_void_p(_ptr(uslots)), ctypes.c_void_p(_ptr(inverse)),
                                         ctypes.c_void_p(_ptr(ucnt)), int(uslots.numel()), int(inverse.numel()),
                                         ctypes.c_void_p(_ptr(deltas)), self.stream()))

    def backward_update(self, uslots, inverse, ucnt, offsets, n_bags, include_last_offset, per_sample_weights,
                        mode, grad_out, optim: str, lr: float, eps: float) -> None:
        check(self.lib.fc_backward_update(
            self.h, ctypes.c_void_p(_ptr(uslots)), ctypes.c_void_p(_ptr(inverse)), ctypes.c_void_p(_ptr(ucnt)),
            int(uslots.numel()), int(inverse.numel()), ctypes.c_void_p(_ptr(offsets)),
            0 if offsets is None else offsets.element_size(), int(n_bags), int(bool(include_last_offset)),
            ctypes.c_void_p(_ptr(per_sample_weights)), _lib.POOL[mode], ctypes.c_void_p(_ptr(grad_out)),
            _lib.OPTIM[optim], float(lr), float(eps), self.stream()))
