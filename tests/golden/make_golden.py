"""Generate the golden vectors under tests/golden/ by running the REAL reference.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (`freqcache`, /root/reference/pkg/src) is a numpy simulator; this
script drives its public API on seeded inputs and records every output the GPU
build must reproduce bit-exactly (SURVEY.md §8c "Parity definition"): unique ids,
counts, ranks, slots, hit/miss/eviction counts, evicted/admitted rank lists,
transfer report rows/bytes/messages, the final slot table and the post-flush slow
tier. Pooled EmbeddingBag and sparse-optimizer vectors come from torch's CPU
implementation (the reference has no pooled module).

Outputs are small .npz files; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import os
import sys
from dataclasses import replace

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import freqcache  # noqa: E402
from freqcache import cache_manager as cm  # noqa: E402
from freqcache import simulator, workload  # noqa: E402
from freqcache.freq_stats import FrequencyTable, build_reorder, scan_frequencies  # noqa: E402
from freqcache.sharding import build_column_stacks, partition_columns, sharded_lookup  # noqa: E402
from freqcache.store import FastTierStore, init_reference_rows, init_stores  # noqa: E402
from freqcache.transmitter import TransferBuffer, Transmitter  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ragged(parts, dtype=np.int64):
    """Concatenate a list of 1-D arrays + their offsets."""
    lens = np.array([len(p) for p in parts], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    flat = np.concatenate([np.asarray(p, dtype=dtype) for p in parts]) if parts else np.empty(0, dtype)
    return flat, off


def report_rows(reports):
    """(rows, bytes, messages) per direction for one prepare call."""
    out = np.zeros(6, dtype=np.int64)
    for r in reports:
        k = 0 if r.direction == "to_slow" else 3
        out[k:k + 3] += (r.rows, r.bytes, r.messages)
    return out


def record_stream(stack, batches, deltas=None, unique_adds=None):
    """Drive stack.prepare over `batches`; optional per-batch update."""
    rec = {k: [] for k in ("unique_ids", "unique_ranks", "unique_counts", "unique_slots", "evicted", "admitted")}
    scal = []
    for seq, ids in enumerate(batches):
        prep = stack.prepare(ids, batch_seq=seq)
        ev = stack.events[-1]
        rec["unique_ids"].append(prep.unique_ids)
        rec["unique_ranks"].append(prep.unique_ranks)
        rec["unique_counts"].append(prep.unique_counts)
        rec["unique_slots"].append(prep.unique_slots)
        rec["evicted"].append(ev.evicted_ranks)
        rec["admitted"].append(ev.admitted_ranks)
        scal.append(np.concatenate([[prep.hits, prep.misses, prep.evictions], report_rows(prep.transfer_reports)]))
        if deltas is not None:
            stack.scatter_update(prep, deltas[seq])
        if unique_adds is not None:
            stack.apply_unique_update(prep, unique_adds(seq, prep))
    out = {}
    for k, parts in rec.items():
        out[k], out[k + "_off"] = ragged(parts)
    out["scalars"] = np.stack(scal).astype(np.int64) if scal else np.zeros((0, 9), np.int64)
    return out


def identity_map(num_ids):
    return build_reorder(FrequencyTable(counts=np.arange(num_ids, 0, -1, dtype=np.int64), num_ids=num_ids))


# ---------------------------------------------------------------------------
# 1. random workouts (test_cache_manager.py:253-301 style), both write-back modes
# ---------------------------------------------------------------------------

def gen_random_stream(name, write_back, num_ids=64, cap=8, dim=4, nb=120, seed=12, init_seed=11, zipf=True):
    if zipf:
        tr = workload.gen_zipf(num_ids, 1.2, 4 * num_ids, 1, seed=seed + 100)
        idx = build_reorder(scan_frequencies(tr, num_ids))
    else:
        idx = identity_map(num_ids)
    slow, _, ref = init_stores(num_ids, dim, cap / num_ids, init_seed=init_seed, idx_map=idx)
    slow0 = slow.rows.copy()
    fast = FastTierStore(slots=np.zeros((cap, dim), dtype=np.float32))
    stack = cm.CacheStack(idx_map=idx, slow=slow, fast=fast, transmitter=Transmitter(buffer=TransferBuffer(4096)),
                          reference=ref, log_events=True, write_back=write_back)
    rng = np.random.default_rng(seed)
    batches, deltas = [], []
    for _ in range(nb):
        size = int(rng.integers(1, cap + 1))
        ids = rng.integers(0, num_ids, size=size)
        batches.append(ids)
        deltas.append(rng.normal(0, 0.1, size=(size, dim)).astype(np.float32))
    rec = record_stream(stack, batches, deltas=deltas)
    rec["ids"], rec["ids_off"] = ragged(batches)
    rec["deltas"] = np.concatenate(deltas)
    flush = stack.flush()
    assert stack.first_divergence() is None
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"), **rec,
        rank_of=idx.rank_of, id_of=idx.id_of, slow0=slow0, slow_final=slow.rows,
        reference_final=ref.rows,
        slot_to_rank=stack.state.slot_to_rank, rank_to_slot=stack.state.rank_to_slot,
        dirty=stack.state.dirty, free_count=np.int64(stack.state.free_count),
        flush=np.array([flush.rows, flush.bytes, flush.messages], dtype=np.int64),
        meta=np.array([num_ids, cap, dim, 4096, 1 if write_back == "always" else 0], dtype=np.int64),
    )


# ---------------------------------------------------------------------------
# 2. simulator runs (simulator.py:353-522) with the oracle attached
# ---------------------------------------------------------------------------

def gen_sim(name, cfg, store_slow=True):
    trace = simulator.build_trace(cfg)
    rep = simulator.verify_against_oracle(cfg, trace)
    assert rep.ok
    seeds = simulator.derive_seeds(cfg.seed)
    metrics, stacks = simulator._run_stacks(replace(cfg, track_oracle=True, log_events=True), trace)
    st = stacks[0]
    evs = [e for e in st.events if e.batch_seq >= 0]
    ev_evicted, ev_evicted_off = ragged([e.evicted_ranks for e in evs])
    ev_admitted, ev_admitted_off = ragged([e.admitted_ranks for e in evs])
    pb = metrics.per_batch
    per_batch = np.stack([np.asarray(pb[k], dtype=np.int64) for k in
                          ("unique", "hits", "misses", "evictions", "rows_to_fast", "rows_to_slow",
                           "bytes_to_fast", "bytes_to_slow", "messages")], axis=1)
    s = metrics.summary
    extra = {}
    if store_slow:
        extra["slow_final"] = st.slow.rows
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"),
        trace=trace.samples, rank_of=st.idx_map.rank_of,
        meta=np.array([cfg.num_ids, cfg.embedding_dim, st.capacity, cfg.batch_size, cfg.buffer_bytes,
                       seeds["init"], seeds["updates"], 1 if cfg.write_back == "always" else 0], dtype=np.uint64),
        per_batch=per_batch, evicted=ev_evicted, evicted_off=ev_evicted_off,
        admitted=ev_admitted, admitted_off=ev_admitted_off,
        slot_to_rank=st.state.slot_to_rank, dirty=st.state.dirty,
        slow_final_sha=np.array(sha(st.slow.rows)),
        totals=np.array([s["hits"], s["misses"], s["evictions"], s["warmup"]["rows_to_fast"],
                         s["batch_phase"]["rows_to_fast"], s["batch_phase"]["rows_to_slow"],
                         s["flush"]["rows_to_slow"], s["batch_phase"]["messages_to_fast"],
                         s["batch_phase"]["messages_to_slow"]], dtype=np.int64),
        **extra,
    )


# ---------------------------------------------------------------------------
# 3. column sharding (sharding.py:62-118)
# ---------------------------------------------------------------------------

def gen_sharded():
    num_ids, dim = 600, 10
    trace = workload.gen_zipf(num_ids, 1.4, 2 * num_ids, 2, seed=0)
    idx = build_reorder(scan_frequencies(trace, num_ids))
    outs = {}
    for shards in (1, 2, 3, 4):
        stacks = build_column_stacks(idx, partition_columns(dim, shards), dim, 0.05, init_seed=7)
        for s in stacks:
            s.warmup(s.capacity)
        rows = [sharded_lookup(stacks, b.ids, b.seq) for b in workload.batches(trace, 12)]
        outs[f"lookup_{shards}"] = np.concatenate(rows)
    for s in (2, 3, 4):
        assert np.array_equal(outs["lookup_1"], outs[f"lookup_{s}"])
    np.savez_compressed(os.path.join(OUT, "sharded.npz"), trace=trace.samples, rank_of=idx.rank_of,
                        lookup=outs["lookup_1"], ranges3=np.array(partition_columns(10, 3).ranges))


# ---------------------------------------------------------------------------
# 4. small pure functions: reorder, init rows, update hash, capacity
# ---------------------------------------------------------------------------

def gen_functions():
    rng = np.random.default_rng(99)
    counts = [rng.integers(0, 5, size=int(n)) for n in rng.integers(1, 300, size=12)]
    counts.append(np.zeros(17, dtype=np.int64))
    rank_of = [build_reorder(FrequencyTable(counts=c, num_ids=c.size)).rank_of for c in counts]
    cflat, coff = ragged(counts)
    rflat, _ = ragged(rank_of)
    init = init_reference_rows(1000, 8, 123)
    ids = rng.integers(0, 10**9, size=4096)
    cnts = rng.integers(1, 50, size=4096)
    scal = np.stack([simulator.update_row_scalars(ids, cnts, seq, useed) for seq, useed in
                     ((0, 5), (7, 12345678901234), (1000, 2**63 + 11))])
    colw = np.stack([simulator.update_column_weights(d, s) for d, s in ((128, 5), (128, 12345678901234))])
    caps = np.array([freqcache.fast_capacity(n, r) for n, r in
                     ((1_000_000, 0.015), (33_762_577, 0.015), (9_445_823, 0.05), (204_184_588, 0.015),
                      (1000, 0.5), (2000, 0.05))], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "functions.npz"), counts=cflat, counts_off=coff, rank_of=rflat,
                        init_1000x8_s123=init, hash_ids=ids, hash_counts=cnts, row_scalars=scal,
                        colw=colw, capacities=caps)


# ---------------------------------------------------------------------------
# 5. pooled EmbeddingBag + sparse optimizers from torch CPU (not in reference)
# ---------------------------------------------------------------------------

def gen_embedding_bag():
    import torch
    import torch.nn.functional as F

    torch.manual_seed(0)
    g = np.random.default_rng(5)
    cases = {}
    for ci, (rows, dim, nbags, maxlen) in enumerate(((50, 8, 20, 4), (300, 128, 64, 1), (100, 64, 33, 7))):
        w = torch.from_numpy(g.uniform(-1, 1, (rows, dim)).astype(np.float32))
        lens = g.integers(0, maxlen + 1, size=nbags)
        if maxlen == 1:
            lens[:] = 1
        idx = torch.from_numpy(g.integers(0, rows, size=int(lens.sum())).astype(np.int64))
        off = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64))
        psw = torch.from_numpy(g.uniform(0, 1, size=idx.numel()).astype(np.float32))
        gout = torch.from_numpy(g.normal(0, 1, (nbags, dim)).astype(np.float32))
        for mode, use_w in (("sum", False), ("mean", False), ("sum", True)):
            wt = w.clone().requires_grad_(True)
            out = F.embedding_bag(idx, wt, off, mode=mode, per_sample_weights=psw if use_w else None)
            out.backward(gout)
            key = f"c{ci}_{mode}{'_w' if use_w else ''}"
            cases[key + "_out"] = out.detach().numpy()
            cases[key + "_grad"] = wt.grad.numpy()
            # one SGD and one Adagrad step on a dense copy with this gradient
            for oname, opt_cls, kw in (("sgd", torch.optim.SGD, {"lr": 0.05}),
                                       ("adagrad", torch.optim.Adagrad, {"lr": 0.05, "eps": 1e-10})):
                p = torch.nn.Parameter(w.clone())
                opt = opt_cls([p], **kw)
                for _ in range(2):
                    opt.zero_grad()
                    F.embedding_bag(idx, p, off, mode=mode, per_sample_weights=psw if use_w else None).backward(gout)
                    opt.step()
                cases[key + f"_{oname}2"] = p.detach().numpy()
        cases[f"c{ci}_w"] = w.numpy()
        cases[f"c{ci}_idx"] = idx.numpy()
        cases[f"c{ci}_off"] = off.numpy()
        cases[f"c{ci}_psw"] = psw.numpy()
        cases[f"c{ci}_gout"] = gout.numpy()
    np.savez_compressed(os.path.join(OUT, "embedding_bag.npz"), **cases)


def gen_sim_metrics():
    """RunMetrics documents of the reference simulator (simulator.py:525-528), without the
    wall-clock fields, for simulator.run on the GPU path to reproduce exactly."""
    import json

    docs = {}
    cfgs = {
        "preset_2shards_oracle": simulator.SimConfig(preset="criteo_like", num_ids=40_000, num_batches=10,
                                                     batch_size=200, embedding_dim=12, cache_ratio=0.05,
                                                     num_shards=2, seed=5, track_oracle=True, log_events=True),
        "exponent_always_rowwise": simulator.SimConfig(preset=None, exponent=1.05, num_ids=30_000, features=4,
                                                       num_batches=8, batch_size=300, embedding_dim=8,
                                                       cache_ratio=0.03, write_back="always",
                                                       policy="rowwise_transfer", buffer_bytes=4096, seed=9),
    }
    for name, cfg in cfgs.items():
        m = simulator.run(cfg)
        docs[name] = {"config": {k: v for k, v in vars(cfg).items()}, "metrics": json.loads(m.determinism_json())}
    with open(os.path.join(OUT, "sim_metrics.json"), "w") as fh:
        json.dump(docs, fh, sort_keys=True)


# ---------------------------------------------------------------------------
# 7. BufferTooSmall ordering (cache_manager.py:219-231,298-323; transmitter.py:85-88,160-164)
# ---------------------------------------------------------------------------

BTS_CALLS = [  # (verb, buffer bytes, write_back, ids); rows are 32 B (dim 8)
    ("prepare", 4096, "dirty_only", [1, 2, 3, 4]),  # fill the 4 slots
    ("prepare", 16, "dirty_only", [1, 2]),          # all hits: nothing moves, no error
    ("prepare", 16, "dirty_only", [5]),             # clean victim 4 evicted, then the admission raises
    ("update", 4096, "dirty_only", [1, 2]),         # rows 1, 2 dirty
    ("prepare", 16, "dirty_only", [6, 7]),          # needed 1: clean victim 3 evicted, admission raises
    ("prepare", 16, "dirty_only", [8]),             # free slots cover the miss: raises before any mutation
    ("prepare", 4096, "dirty_only", [8, 9]),        # admitted
    ("prepare", 16, "dirty_only", [10]),            # clean victim 9 evicted, admission raises
    ("prepare", 4096, "dirty_only", [10, 11]),      # clean victim 8 evicted + written nowhere, admitted
    ("update", 4096, "dirty_only", [1, 2, 10, 11]), # everything dirty
    ("prepare", 16, "dirty_only", [12]),            # dirty victim 11: the write-back raises before mutation
    ("prepare", 16, "always", [12]),                # same under write_back='always'
    ("flush", 16, "dirty_only", []),                # dirty rows: raises before mutation
    ("flush", 4096, "dirty_only", []),              # writes them back
    ("flush", 16, "dirty_only", []),                # nothing dirty: no error
    ("prepare", 16, "always", [1, 2, 10, 11]),      # all hits: no error
    ("prepare", 16, "always", [13]),                # 'always' writes even clean victims: raises before mutation
]


def gen_buffer_too_small():
    num_ids, cap, dim = 16, 4, 8
    idx = identity_map(num_ids)
    slow, _, ref = init_stores(num_ids, dim, cap / num_ids, init_seed=0, idx_map=idx)
    slow0 = slow.rows.copy()
    fast = FastTierStore(slots=np.zeros((cap, dim), dtype=np.float32))
    state = cm.CacheState(cap, num_ids)
    raised, s2r, dirty, free, slows = [], [], [], [], []
    prep = None
    for verb, buf, wb, ids in BTS_CALLS:
        tx = Transmitter(buffer=TransferBuffer(buf))
        err = 0
        try:
            if verb == "prepare":
                prep = cm.prepare_cache(state, idx, np.array(ids), tx, slow, fast, write_back=wb)
            elif verb == "update":
                prep = cm.prepare_cache(state, idx, np.array(ids), tx, slow, fast, write_back=wb)
                cm.scatter_update(state, fast, prep, np.full((len(ids), dim), 0.25, np.float32))
            else:
                cm.flush(state, tx, slow, fast)
        except freqcache.BufferTooSmall:
            err = 1
        raised.append(err)
        s2r.append(state.slot_to_rank.copy())
        dirty.append(state.dirty.copy())
        free.append(state.free_count)
        slows.append(slow.rows.copy())
    ids_flat, ids_off = ragged([c[3] for c in BTS_CALLS])
    np.savez_compressed(os.path.join(OUT, "buffer_too_small.npz"), slow0=slow0, raised=np.array(raised),
                        call_verb=np.array([("prepare", "update", "flush").index(c[0]) for c in BTS_CALLS]),
                        call_buf=np.array([c[1] for c in BTS_CALLS]),
                        call_always=np.array([int(c[2] == "always") for c in BTS_CALLS]),
                        call_ids=ids_flat, call_ids_off=ids_off,
                        slot_to_rank=np.array(s2r), dirty=np.array(dirty), free_count=np.array(free),
                        slow=np.array(slows), meta=np.array([num_ids, cap, dim], dtype=np.int64))


# ---------------------------------------------------------------------------
# 8. CSV trace ingestion (workload.py:276-392) and CSV-driven simulator runs (simulator.py:208-213)
# ---------------------------------------------------------------------------

CSV_CASES = {  # name -> (file text, load_csv kwargs); the reference's own test shapes (test_workload.py:112-166)
    "remap": ("f0,f1\nx,y\nx,z\n", {}),
    "remap_stable": ("f0,f1\na,b\nc,b\na,d\n", {}),
    "empty": ("", {}),
    "identity": ("a,b,c\n1,2,3\n4,5,6\n", {"id_remap": "identity", "num_ids": 10}),
    "subset": ("a,b,c\n1,2,3\n4,5,6\n", {"feature_columns": ["a", "c"], "id_remap": "identity", "num_ids": 10}),
    "malformed_skip": ("f0,f1\n1,2\n3\n", {"id_remap": "identity", "num_ids": 10, "on_error": "skip"}),
    "malformed_fail": ("f0,f1\n1,2\n3\n", {"id_remap": "identity", "num_ids": 10}),
    "badint_skip": ("f0,f1\n1,2\nx,3\n7,8\n", {"id_remap": "identity", "num_ids": 10, "on_error": "skip"}),
    "remap_blank_and_quoted": ('f0,f1,f2\n"a,b",,x\n,q,x\n"a,b",q,y\n\nz,,x\n', {}),
}


def gen_csv():
    import json
    import tempfile

    rng = np.random.default_rng(41)
    # a categorical log: 3 string columns with per-column vocabularies of different sizes
    lines = ["site,app,device"] + [f"s{a},app{b},d{c}" for a, b, c in zip(
        rng.zipf(1.6, 600) % 50, rng.zipf(1.4, 600) % 300, rng.integers(0, 7, 600))]
    CSV_CASES["categorical_log"] = ("\n".join(lines) + "\n", {})
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, (text, kw) in CSV_CASES.items():
            path = os.path.join(d, name + ".csv")
            with open(path, "w", newline="") as fh:
                fh.write(text)
            doc = {"text": text, "kwargs": kw}
            try:
                tr = workload.load_csv(path, **kw)
                doc.update(samples=tr.samples.tolist(), num_ids=tr.num_ids, features=tr.features,
                           table_sizes=tr.table_sizes)
            except ValueError as e:
                doc["error"] = str(e).replace(path, "<path>")
            out[name] = doc
    # save_csv bytes of a generated trace (the interchange format) and two simulator runs on CSV files
    tr = workload.gen_zipf(3000, 1.2, 500, 3, seed=43)
    path = os.path.join(OUT, "trace_global.csv")
    workload.save_csv(tr, path)
    with open(os.path.join(OUT, "trace_categorical.csv"), "w", newline="") as fh:
        fh.write(CSV_CASES["categorical_log"][0])
    runs = {}
    for name, cfg in {
        "global": simulator.SimConfig(preset=None, trace_path="tests/golden/trace_global.csv", trace_format="global",
                                      num_ids=3000, batch_size=40, embedding_dim=8, cache_ratio=0.05, seed=6,
                                      track_oracle=True),
        "categorical": simulator.SimConfig(preset=None, trace_path="tests/golden/trace_categorical.csv",
                                           trace_format="categorical", num_ids=1, batch_size=10, embedding_dim=4,
                                           cache_ratio=0.3, seed=7, write_back="always"),
    }.items():
        cwd = os.getcwd()
        os.chdir(os.path.dirname(os.path.dirname(OUT)))  # trace paths relative to the repo root
        try:
            m = simulator.run(cfg)
        finally:
            os.chdir(cwd)
        runs[name] = {"config": {k: v for k, v in vars(cfg).items()}, "metrics": json.loads(m.determinism_json())}
    with open(os.path.join(OUT, "csv.json"), "w") as fh:
        json.dump({"load_csv": out, "runs": runs, "trace_global_samples": tr.samples.tolist()}, fh, sort_keys=True)


def gen_tablewise():
    """Table-wise placement (plan_tables_greedy, sharding.py:158-172) and the load statistics
    (tablewise_imbalance / columnwise_imbalance, :183-205) on the Criteo sizes, a scaled copy
    and a tie-heavy random list, 1..8 shards."""
    import json

    from freqcache import sharding as sh

    rng = np.random.default_rng(5)
    lists = {"criteo": list(sh.CRITEO_KAGGLE_TABLE_SIZES), "criteo_div1000": sh.criteo_like_table_sizes(1000),
             "ties": rng.integers(1, 6, 40).tolist()}
    out = {}
    for name, sizes in lists.items():
        for w in range(1, 9):
            plan = sh.plan_tables_greedy(sizes, w)
            st = sh.tablewise_imbalance(plan)
            out[f"{name}/{w}"] = {"sizes": [int(x) for x in sizes], "assignment": plan.assignment.tolist(),
                                  "per_shard_rows": st.per_shard_rows.tolist(), "max_rows": st.max_rows,
                                  "mean_rows": st.mean_rows, "imbalance_ratio": st.imbalance_ratio}
    for dim in (128, 10):
        for w in range(1, 9):
            st = sh.columnwise_imbalance(sh.partition_columns(dim, w), 33_762_577)
            out[f"column/{dim}/{w}"] = {"per_shard_rows": st.per_shard_rows.tolist(), "max_rows": st.max_rows,
                                        "mean_rows": st.mean_rows, "imbalance_ratio": st.imbalance_ratio}
    with open(os.path.join(OUT, "tablewise.json"), "w") as fh:
        json.dump(out, fh, sort_keys=True)


def main():
    only = sys.argv[1:]  # e.g. `make_golden.py gen_tablewise`: regenerate just those
    if only:
        for name in only:
            globals()[name]()
        return
    gen_random_stream("stream_dirty_zipf", "dirty_only")
    gen_random_stream("stream_always_zipf", "always", seed=21, init_seed=3)
    gen_random_stream("stream_dirty_ident", "dirty_only", num_ids=48, cap=6, dim=10, nb=80, seed=6,
                      init_seed=2, zipf=False)
    small = simulator.SimConfig(preset=None, exponent=1.3, num_ids=2000, features=3, num_batches=40,
                                batch_size=16, embedding_dim=8, cache_ratio=0.05, seed=77)
    gen_sim("sim_small", small)
    gen_sim("sim_small_always", replace(small, write_back="always", seed=78))
    medium = simulator.SimConfig(preset=None, exponent=1.05, num_ids=200_000, features=26, num_batches=24,
                                 batch_size=128, embedding_dim=16, cache_ratio=0.03, seed=1,
                                 buffer_bytes=1 << 16)
    gen_sim("sim_medium", medium, store_slow=False)
    gen_sharded()
    gen_functions()
    gen_embedding_bag()
    gen_sim_metrics()
    gen_buffer_too_small()
    gen_csv()
    gen_tablewise()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
