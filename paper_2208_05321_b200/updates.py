"""The reference simulator's deterministic per-batch update (simulator.py:229-260).

`update_row_scalars(unique_ids, counts, batch_seq, seed)[:, None] *
update_column_weights(dim, seed)` is the add the simulator applies to each unique
row (simulator.py:429-433). On B200 the whole product is fused into one device
kernel (`CacheStack.apply_synthetic_update` -> fc_apply_synthetic_update) with
fp32 round-to-nearest ops in numpy's order, so runs stay bit-comparable with the
reference. The host functions here feed the dense ReferenceStore mirror and the
per-column weights (D floats, computed once).
"""

from __future__ import annotations

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
_A = np.uint64(0x9E3779B97F4A7C15)
_B = np.uint64(0xBF58476D1CE4E5B9)
_C = np.uint64(0x94D049BB133111EB)


def hash_unit(values, salt: int) -> np.ndarray:
    """splitmix64 of (v*golden + salt), top 24 bits as a [0,1) float32."""
    with np.errstate(over="ignore"):
        h = np.asarray(values).astype(np.uint64) * _A + np.uint64(int(salt) % (1 << 64))
        h ^= h >> np.uint64(30)
        h *= _B
        h ^= h >> np.uint64(27)
        h *= _C
        h ^= h >> np.uint64(31)
    return (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)


def update_column_weights(embedding_dim: int, updates_seed: int) -> np.ndarray:
    """Per-column scale in [0.5, 1.5) (simulator.py:246-248)."""
    return hash_unit(np.arange(embedding_dim), updates_seed * 3 + 1) + np.float32(0.5)


def batch_salt(batch_seq: int, updates_seed: int) -> int:
    """The hash salt of one batch, reduced mod 2**64 as the reference does."""
    return ((batch_seq + 1) * GOLDEN + updates_seed) % (1 << 64)


def update_row_scalars(unique_ids, counts, batch_seq: int, updates_seed: int) -> np.ndarray:
    """Per-unique-id scalar for one batch (simulator.py:251-260)."""
    g = hash_unit(unique_ids, batch_salt(batch_seq, updates_seed)) - np.float32(0.5)
    return g * np.asarray(counts).astype(np.float32)
