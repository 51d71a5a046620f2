"""Shared replay drivers for the golden fixtures (used by CPU and GPU tests).

`sim_inputs(g)` unpacks a simulator fixture made by tests/golden/make_golden.py;
`run_sim(cache_factory, g)` runs the reference simulator's per-batch loop
(simulator.py:393-461: warmup(C), then per batch prepare -> gather_unique ->
apply_unique_update(row_scalars x column weights), then flush) against any cache
object exposing the OracleCache-shaped verbs.
"""

from __future__ import annotations

import numpy as np

from conftest import split


def sim_inputs(g):
    num_ids, dim, cap, batch, buf, init_seed, upd_seed, always = (int(v) for v in g["meta"])
    return {
        "num_ids": num_ids, "dim": dim, "capacity": cap, "batch_size": batch, "buffer_bytes": buf,
        "init_seed": init_seed, "updates_seed": upd_seed,
        "write_back": "always" if always else "dirty_only",
        "trace": g["trace"], "rank_of": g["rank_of"],
    }


def batches(trace, batch_size):
    for seq, start in enumerate(range(0, trace.shape[0], batch_size)):
        yield seq, trace[start:start + batch_size].reshape(-1)


def expect_batch_rows(g):
    return g["per_batch"], split(g["evicted"], g["evicted_off"]), split(g["admitted"], g["admitted_off"])


def bts_calls(g):
    """The scripted calls of the buffer_too_small fixture (make_golden.gen_buffer_too_small):
    (verb, buffer_bytes, write_back, ids) with verb in prepare / update / flush."""
    ids = split(g["call_ids"], g["call_ids_off"])
    for k in range(len(g["call_verb"])):
        yield (("prepare", "update", "flush")[int(g["call_verb"][k])], int(g["call_buf"][k]),
               "always" if int(g["call_always"][k]) else "dirty_only", np.asarray(ids[k], dtype=np.int64))
