"""Synthetic id streams for benchmarks and parity runs.

`gen_zipf` reproduces the reference generator's streams bit-for-bit
(/root/reference/pkg/src/freqcache/workload.py:73-192: ranks drawn i.i.d. from a
(shifted) power law by inverse CDF, mapped through a seeded permutation of the id
space), so the GPU build and the CPU reference consume identical ids. The
inverse-CDF search can run on the GPU (`device=`) for large traces; it performs
the same exact float64 comparisons, so the ranks are identical.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import lru_cache

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


# ----------------------------------------------------------------------------- skew presets
# (workload.py:93-133, 195-248) — the calibrated laws the reference simulator's
# `preset=` configs use: a named head share covering a named share of accesses.

def expected_head_coverage(num_ids: int, exponent: float, top_fraction: float, shift: float = 0.0) -> float:
    """Share of accesses on the top ceil(top_fraction * num_ids) ranks under the law."""
    k = math.ceil(top_fraction * num_ids)
    return 0.0 if k <= 0 else float(zipf_pmf(num_ids, exponent, shift)[:k].sum())


def calibrate_exponent(num_ids: int, top_fraction: float, target_coverage: float, shift: float = 0.0,
                       lo: float = 1e-3, hi: float = 64.0, iterations: int = 60) -> float:
    """Bisection on the exponent (head coverage increases with it) until the head share is met."""
    if not (0.0 < target_coverage < 1.0):
        raise ValueError("target_coverage must be in (0, 1)")
    c_lo = expected_head_coverage(num_ids, lo, top_fraction, shift)
    c_hi = expected_head_coverage(num_ids, hi, top_fraction, shift)
    if not (c_lo <= target_coverage <= c_hi):
        raise ValueError(f"target {target_coverage} unreachable in exponent bracket [{lo}, {hi}] "
                         f"(coverage range [{c_lo:.4f}, {c_hi:.4f}])")
    for _ in range(iterations):
        mid = 0.5 * (lo + hi)
        if expected_head_coverage(num_ids, mid, top_fraction, shift) < target_coverage:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


@dataclass(frozen=True)
class SkewPreset:
    features: int
    top_fraction: float
    target_coverage: float
    shift_frac: float


PRESETS = {
    "criteo_like": SkewPreset(features=26, top_fraction=0.0014, target_coverage=0.90, shift_frac=1e-3),
    "avazu_like": SkewPreset(features=13, top_fraction=0.00012, target_coverage=0.90, shift_frac=5.5e-5),
}


@lru_cache(maxsize=64)
def preset_params(name: str, num_ids: int) -> tuple[float, float]:
    """(exponent, shift) of a preset at this id-space size."""
    if name not in PRESETS:
        raise ValueError(f"unknown preset {name!r}, have {sorted(PRESETS)}")
    p = PRESETS[name]
    shift = p.shift_frac * num_ids
    return calibrate_exponent(num_ids, p.top_fraction, p.target_coverage, shift), shift


def gen_preset(name: str, num_ids: int, num_samples: int, seed: int, features: int | None = None,
               device=None) -> Trace:
    exponent, shift = preset_params(name, num_ids)
    tr = gen_zipf(num_ids, exponent, num_samples, PRESETS[name].features if features is None else features, seed,
                  shift=shift, device=device)
    tr.provenance["preset"] = name
    return tr


def batches(trace: Trace, batch_size: int):
    """Consecutive windows of batch_size samples, flattened (workload.py:259-270)."""
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    for seq, lo in enumerate(range(0, trace.num_samples, batch_size)):
        yield Batch(seq, trace.samples[lo:lo + batch_size].reshape(-1))


# ----------------------------------------------------------------------------- CSV ingestion
# (workload.py:276-392) — the trace interchange format, feeding the device path: the loaded
# Trace goes straight to build_reorder_device / CacheStack / simulator.run.

@dataclass
class ColumnRemap:
    """Per-feature categorical remap into one offset global id space (workload.py:276-287)."""

    maps: list
    offsets: np.ndarray
    num_ids: int

    @property
    def table_sizes(self) -> list:
        return [len(m) for m in self.maps]


def save_csv(trace: Trace, path) -> None:
    """Header f0..fN, one sample per line, decimal global ids (workload.py:290-297)."""
    with open(path, "w", newline="") as fh:
        fh.write(",".join(f"f{i}" for i in range(trace.features)) + "\r\n")
        if trace.samples.size:
            np.savetxt(fh, np.asarray(trace.samples, dtype=np.int64), fmt="%d", delimiter=",", newline="\r\n")


def _first_seen_ids(tokens, remap_dict: dict) -> np.ndarray:
    """Column tokens -> local ids in first-seen order, extending `remap_dict` exactly as
    the reference's per-row dict.setdefault does (workload.py:363-366), but vectorised:
    unique tokens, each one's first position, new tokens ranked by it."""
    tok = np.asarray(tokens, dtype=object)
    if tok.size == 0:
        return np.empty(0, dtype=np.int64)
    uniq, first, inv = np.unique(tok.astype(str), return_index=True, return_inverse=True)
    known = np.array([remap_dict.get(u, -1) for u in uniq], dtype=np.int64)
    new = np.flatnonzero(known < 0)
    base = len(remap_dict)
    for k, u in enumerate(new[np.argsort(first[new], kind="stable")]):
        known[u] = base + k
        remap_dict[uniq[u]] = base + k
    return known[inv.reshape(-1)]


def load_csv(path, feature_columns: list | None = None, id_remap=None, num_ids: int | None = None,
             on_error: str = "fail") -> Trace:
    """A categorical CSV as a Trace (workload.py:300-392): every column remapped, per column
    and in first-seen order, into a contiguous id space with per-feature offsets (the same raw
    value in two columns gets two ids); a previous ColumnRemap keeps ids stable across files;
    id_remap="identity" parses global ids directly (save_csv's format; id space = num_ids or
    max + 1). Malformed rows raise with their line number, or are skipped (on_error="skip")."""
    import csv

    if on_error not in ("fail", "skip"):
        raise ValueError("on_error must be 'fail' or 'skip'")
    identity = id_remap == "identity"
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header is None:
            return Trace(num_ids=num_ids or 0, features=1, samples=np.empty((0, 1), dtype=np.int64))
        header = [h.strip() for h in header]
        if feature_columns is None:
            cols = list(range(len(header)))
        else:
            missing = [c for c in feature_columns if c not in header]
            if missing:
                raise ValueError(f"{path}: feature columns not in header: {missing}")
            cols = [header.index(c) for c in feature_columns]
        features = len(cols)
        if identity:
            remap = None
        elif id_remap is None:
            remap = ColumnRemap(maps=[{} for _ in cols], offsets=np.zeros(features, dtype=np.int64), num_ids=0)
        elif isinstance(id_remap, ColumnRemap):
            remap = id_remap
            if len(remap.maps) != features:
                raise ValueError(f"id_remap covers {len(remap.maps)} columns, trace has {features}")
        else:
            raise ValueError(f"id_remap must be None, 'identity', or a ColumnRemap, got {id_remap!r}")
        rows = []
        for lineno, row in enumerate(reader, start=2):
            if not row:
                continue
            if len(row) != len(header):
                if on_error == "skip":
                    continue
                raise ValueError(f"{path}:{lineno}: expected {len(header)} fields, got {len(row)}")
            if identity:
                try:
                    rows.append([int(row[c]) for c in cols])
                except ValueError:
                    if on_error == "skip":
                        continue
                    raise ValueError(f"{path}:{lineno}: malformed id field") from None
            else:
                rows.append([row[c] for c in cols])
    if identity:
        samples = np.asarray(rows, dtype=np.int64).reshape(-1, features)
        space = num_ids if num_ids is not None else (int(samples.max()) + 1 if samples.size else 0)
        return Trace(space, features, samples, {"source": str(path), "remap": "identity"})
    tok = np.asarray(rows, dtype=object).reshape(-1, features)
    local = np.stack([_first_seen_ids(tok[:, f], remap.maps[f]) for f in range(features)], axis=1) \
        if tok.shape[0] else np.empty((0, features), dtype=np.int64)
    sizes = remap.table_sizes
    remap.offsets = np.concatenate([[0], np.cumsum(sizes[:-1])]).astype(np.int64)
    remap.num_ids = int(sum(sizes))
    samples = local.astype(np.int64).reshape(-1, features) + remap.offsets
    return Trace(remap.num_ids, features, samples, {"source": str(path), "remap": "per_column"}, table_sizes=sizes)
