"""Synthetic id streams for benchmarks and parity runs.

`gen_zipf` reproduces the reference generator's streams bit-for-bit
(/root/reference/pkg/src/freqcache/workload.py:73-192: ranks drawn i.i.d. from a
(shifted) power law by inverse CDF, mapped through a seeded permutation of the id
space), so the GPU build and the CPU reference consume identical ids. The
inverse-CDF search can run on the GPU (`device=`) for large traces; it performs
the same exact float64 comparisons, so the ranks are identical.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_CHUNK = 1 << 24


def zipf_pmf(num_ids: int, exponent: float, shift: float = 0.0) -> np.ndarray:
    """p(r) proportional to (r + 1 + shift)^-exponent, computed in log space (workload.py:73-90)."""
    if num_ids < 1:
        raise ValueError("num_ids must be >= 1")
    if exponent <= 0:
        raise ValueError(f"exponent must be > 0, got {exponent}")
    if shift < 0:
        raise ValueError(f"shift must be >= 0, got {shift}")
    lw = -exponent * np.log(np.arange(1, num_ids + 1, dtype=np.float64) + shift)
    lw -= lw.max()
    w = np.exp(lw)
    return w / w.sum()


@dataclass
class Trace:
    num_ids: int
    features: int
    samples: np.ndarray
    provenance: dict = field(default_factory=dict)
    table_sizes: list | None = None

    @property
    def num_samples(self) -> int:
        return int(self.samples.shape[0])


@dataclass
class Batch:
    seq: int
    ids: np.ndarray


def gen_zipf(num_ids: int, exponent: float, num_samples: int, features: int, seed: int, shift: float = 0.0,
             device=None) -> Trace:
    """num_samples x features ids from the skewed law (workload.py:136-192)."""
    if num_samples < 0 or features < 1:
        raise ValueError("num_samples must be >= 0 and features >= 1")
    cdf = np.cumsum(zipf_pmf(num_ids, exponent, shift))
    cdf[-1] = 1.0
    perm_ss, draw_ss = np.random.SeedSequence(seed).spawn(2)
    dtype = np.int32 if num_ids <= np.iinfo(np.int32).max else np.int64
    perm = np.random.default_rng(perm_ss).permutation(num_ids).astype(dtype)
    total = num_samples * features
    out = np.empty(total, dtype=dtype)
    rng = np.random.default_rng(draw_ss)
    if device is not None:
        import torch

        cdf_t = torch.from_numpy(cdf).to(device)
        perm_t = torch.from_numpy(perm).to(device)
    for lo in range(0, total, _CHUNK):
        hi = min(lo + _CHUNK, total)
        u = rng.random(hi - lo)
        if device is None:
            out[lo:hi] = perm[np.searchsorted(cdf, u, side="right")]
        else:
            r = torch.searchsorted(cdf_t, torch.from_numpy(u).to(device), right=True)
            out[lo:hi] = perm_t[r].cpu().numpy()
    return Trace(num_ids, features, out.reshape(num_samples, features),
                 {"generator": "zipf", "exponent": float(exponent), "shift": float(shift),
                  "num_samples": num_samples, "seed": int(seed)})


def gen_uniform(num_ids: int, num_samples: int, features: int, seed: int) -> Trace:
    """num_samples x features ids drawn uniformly (the eviction/transfer stress stream of
    BASELINE configs[4]; the reference has no uniform generator, so this one is simply a
    seeded numpy PCG64 draw, identical for the GPU build and the CPU reference arm)."""
    if num_samples < 0 or features < 1 or num_ids < 1:
        raise ValueError("num_samples must be >= 0, features >= 1, num_ids >= 1")
    dtype = np.int32 if num_ids <= np.iinfo(np.int32).max else np.int64
    rng = np.random.default_rng(np.random.SeedSequence(seed))
    out = rng.integers(0, num_ids, size=num_samples * features, dtype=np.int64).astype(dtype)
    return Trace(num_ids, features, out.reshape(num_samples, features),
                 {"generator": "uniform", "num_samples": num_samples, "seed": int(seed)})


def batches(trace: Trace, batch_size: int):
    """Consecutive windows of batch_size samples, flattened (workload.py:259-270)."""
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    for seq, lo in enumerate(range(0, trace.num_samples, batch_size)):
        yield Batch(seq, trace.samples[lo:lo + batch_size].reshape(-1))
