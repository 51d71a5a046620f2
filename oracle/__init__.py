"""CPU oracle for the frequency-aware embedding cache path — TEST INFRASTRUCTURE ONLY.

This package is a plain-numpy restatement of the reference algorithm
(`/root/reference/pkg/src/freqcache`, the `freqcache` simulator of
arXiv 2208.05321) for the hot path named in BASELINE.json's north star:
frequency reorder, prepare-ids (Alg. 1), warmup, flush, lookup, update, plus a
restatement of the pooled EmbeddingBag and sparse SGD/Adagrad semantics the
reference lacks (pinned to torch's CPU `F.embedding_bag` / `torch.optim`).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it, and only as the checker or the timed CPU
baseline. The product package `paper_2208_05321_b200` never imports it: its
compute runs in `libfreqcache_b200.so` on the GPU and fails loudly without it.

Parity pinning: `tests/golden/make_golden.py` runs the real reference (importable
in the build container from /root/reference/pkg/src) and commits its outputs under
`tests/golden/`; `tests/test_oracle_golden.py` checks this restatement against
them, and against the known-answer cases of the reference's own tests.
"""

from .cache_oracle import (  # noqa: F401
    ABSENT,
    EMPTY,
    OracleBatchExceedsCapacity,
    OracleCache,
    OracleInsufficientEvictable,
    OracleInsufficientFreeSlots,
    OracleBufferTooSmall,
    chunk_messages,
    column_ranges,
    fast_capacity,
    frequency_counts,
    hash_unit,
    init_rows,
    rank_permutation,
    row_scalars,
    column_weights,
    pooled_bag,
    pooled_bag_backward_rows,
    sparse_sgd,
    sparse_adagrad,
    replay_law,
)
