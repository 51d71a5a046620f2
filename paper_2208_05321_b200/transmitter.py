"""Transfer accounting and the row-moving verbs between tiers.

Mirrors `freqcache.transmitter` (/root/reference/pkg/src/freqcache/transmitter.py):
the same `ChannelModel`, `TransferReport`, `TransferBuffer`, `chunk_plan` and
`Transmitter` names and arithmetic. On B200 the rows of a prepare/flush are moved
by the device kernels of libfreqcache_b200 (zero-copy over the host link, both
directions in one kernel); this module supplies the reference-identical
rows/bytes/messages accounting (one message per floor(buffer/row_bytes) rows,
transmitter.py:97-109), the modeled time (:51-59) and, next to it, the measured
device time of the step when the caller records it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DEFAULT_BUFFER_BYTES = 64 * 2**20
DEFAULT_LATENCY_S = 10e-6
DEFAULT_BANDWIDTH_BPS = 12 * 2**30
DEFAULT_LOCAL_BANDWIDTH_BPS = 200 * 2**30

TO_FAST = "to_fast"
TO_SLOW = "to_slow"


class BufferTooSmall(ValueError):
    """A single row does not fit in the staging buffer (transmitter.py:28-29)."""


@dataclass(frozen=True)
class ChannelModel:
    """Per-message latency plus cross-tier and within-tier bandwidths (transmitter.py:33-59)."""

    latency_s: float = DEFAULT_LATENCY_S
    bandwidth_Bps: float = DEFAULT_BANDWIDTH_BPS
    local_bandwidth_Bps: float = DEFAULT_LOCAL_BANDWIDTH_BPS

    def __post_init__(self) -> None:
        if min(self.latency_s, self.bandwidth_Bps, self.local_bandwidth_Bps) <= 0:
            raise ValueError("channel parameters must be strictly positive")
        if self.local_bandwidth_Bps < self.bandwidth_Bps:
            raise ValueError("local bandwidth must be >= cross-tier bandwidth")

    def block_time_s(self, messages: int, nbytes: int) -> float:
        return messages * self.latency_s + nbytes / self.bandwidth_Bps + 2 * nbytes / self.local_bandwidth_Bps

    def rowwise_time_s(self, rows: int, nbytes: int) -> float:
        return rows * self.latency_s + nbytes / self.bandwidth_Bps


@dataclass(frozen=True)
class TransferReport:
    direction: str
    rows: int
    bytes: int
    messages: int
    modeled_time_s: float

    @classmethod
    def empty(cls, direction: str) -> "TransferReport":
        return cls(direction=direction, rows=0, bytes=0, messages=0, modeled_time_s=0.0)


class TransferBuffer:
    """The bounded staging budget (transmitter.py:75-94). On B200 the staging of a
    prepare lives in HBM; the capacity still fixes the message granularity."""

    def __init__(self, capacity_bytes: int = DEFAULT_BUFFER_BYTES):
        if capacity_bytes < 1:
            raise ValueError("buffer capacity must be >= 1 byte")
        self.capacity_bytes = int(capacity_bytes)

    def rows_per_message(self, row_bytes: int) -> int:
        if row_bytes > self.capacity_bytes:
            raise BufferTooSmall(f"row of {row_bytes} B cannot fit in a {self.capacity_bytes} B buffer")
        return self.capacity_bytes // row_bytes


def chunk_plan(rows: int, row_bytes: int, buffer_bytes: int) -> int:
    """Messages needed to move `rows` whole rows through the buffer (transmitter.py:97-109)."""
    if rows < 0 or row_bytes < 1 or buffer_bytes < 1:
        raise ValueError("rows must be >= 0, sizes >= 1")
    if row_bytes > buffer_bytes:
        raise BufferTooSmall(f"row of {row_bytes} B cannot fit in a {buffer_bytes} B buffer")
    if rows == 0:
        return 0
    return math.ceil(rows / (buffer_bytes // row_bytes))


def rowwise_baseline_report(rows: int, row_bytes: int, channel: ChannelModel) -> TransferReport:
    """Cost of the one-message-per-row scheme (transmitter.py:112-121)."""
    nbytes = rows * row_bytes
    return TransferReport(TO_FAST, rows, nbytes, rows, channel.rowwise_time_s(rows, nbytes))


class Transmitter:
    """Accounting + explicit row moves between a slow and a fast store.

    ``mode="block"`` counts whole-row chunks through the bounded buffer;
    ``mode="rowwise"`` counts one message per row (transmitter.py:124-142).
    """

    def __init__(self, buffer: TransferBuffer | None = None, channel: ChannelModel | None = None,
                 mode: str = "block"):
        if mode not in ("block", "rowwise"):
            raise ValueError(f"mode must be 'block' or 'rowwise', got {mode!r}")
        self.buffer = buffer if buffer is not None else TransferBuffer()
        self.channel = channel if channel is not None else ChannelModel()
        self.mode = mode

    def report(self, direction: str, rows: int, row_bytes: int) -> TransferReport:
        """The reference's TransferReport for `rows` rows moved in `direction`."""
        if rows == 0:
            self.buffer.rows_per_message(row_bytes)  # a row must fit even for a no-op (:162-164)
            return TransferReport.empty(direction)
        nbytes = rows * row_bytes
        if self.mode == "rowwise":
            return TransferReport(direction, rows, nbytes, rows, self.channel.rowwise_time_s(rows, nbytes))
        msgs = chunk_plan(rows, row_bytes, self.buffer.capacity_bytes)
        return TransferReport(direction, rows, nbytes, msgs, self.channel.block_time_s(msgs, nbytes))

    # -- explicit moves (transmitter.py:197-207); prepare/flush never call these ----
    def move_to_fast(self, slow, fast, ranks, target_slots) -> TransferReport:
        """Copy slow rows (by rank) into fast slots."""
        import torch

        ranks = np.asarray(ranks, dtype=np.int64).reshape(-1)
        slots = np.asarray(target_slots, dtype=np.int64).reshape(-1)
        self._check(ranks, slots, slow.num_rows, fast.capacity)
        rep = self.report(TO_FAST, int(ranks.size), fast.embedding_dim * 4)
        if ranks.size:
            rows = torch.from_numpy(np.ascontiguousarray(slow.rows[ranks]))
            fast.slots[torch.from_numpy(slots).to(fast.slots.device)] = rows.to(fast.slots.device)
        return rep

    def move_to_slow(self, fast, slow, slots, target_ranks) -> TransferReport:
        """Copy fast slots back to slow rows (by rank)."""
        import torch

        slots = np.asarray(slots, dtype=np.int64).reshape(-1)
        ranks = np.asarray(target_ranks, dtype=np.int64).reshape(-1)
        self._check(slots, ranks, fast.capacity, slow.num_rows)
        rep = self.report(TO_SLOW, int(slots.size), fast.embedding_dim * 4)
        if slots.size:
            rows = fast.slots[torch.from_numpy(slots).to(fast.slots.device)].cpu().numpy()
            slow.rows[ranks] = rows
        return rep

    @staticmethod
    def _check(src_idx, dst_idx, src_limit, dst_limit):
        if src_idx.size != dst_idx.size:
            raise ValueError(f"{src_idx.size} source rows but {dst_idx.size} targets")
        for idx, limit, what in ((src_idx, src_limit, "source"), (dst_idx, dst_limit, "target")):
            if idx.size and (int(idx.min()) < 0 or int(idx.max()) >= limit):
                raise IndexError(f"{what} row index out of range [0, {limit})")
