"""Exception classes of the cache path (same names and bases as
/root/reference/pkg/src/freqcache/cache_manager.py:35-52 and transmitter.py:28-29)
and the mapping from the C ABI's fc_status codes to them."""

from __future__ import annotations

from . import _lib
from .transmitter import BufferTooSmall


class BatchExceedsCapacity(ValueError):
    """More unique ids in one batch than the fast tier has slots."""


class InsufficientEvictable(RuntimeError):
    """Eviction needs more slots than there are unprotected occupied ones."""


class InsufficientFreeSlots(RuntimeError):
    """Admission ran out of free slots (paper_literal mode once the tier is full)."""


class FreqCacheCudaError(RuntimeError):
    """A CUDA call inside libfreqcache_b200 failed."""


_MAP = {
    _lib.ERR_BATCH_EXCEEDS_CAPACITY: BatchExceedsCapacity,
    _lib.ERR_ID_OUT_OF_RANGE: ValueError,
    _lib.ERR_INSUFFICIENT_EVICTABLE: InsufficientEvictable,
    _lib.ERR_INSUFFICIENT_FREE_SLOTS: InsufficientFreeSlots,
    _lib.ERR_BUFFER_TOO_SMALL: BufferTooSmall,
    _lib.ERR_CUDA: FreqCacheCudaError,
    _lib.ERR_BAD_ARG: ValueError,
    _lib.ERR_SLOT_OUT_OF_RANGE: IndexError,
    _lib.ERR_NOT_EMPTY: ValueError,
    _lib.ERR_NO_SLOW_TIER: RuntimeError,
}


def check(rc: int, what: str = "") -> None:
    if rc == _lib.OK:
        return
    msg = _lib.last_error() or f"fc status {rc}"
    raise _MAP.get(rc, RuntimeError)(msg if not what else f"{msg}")
