"""CPU: pin the numpy oracle (oracle/) against the reference.

Two sources pin it: the known-answer cases of the reference's own tests
(/root/reference/pkg/tests/test_cache_manager.py etc., cited per test) restated
here, and the golden vectors tests/golden/*.npz that make_golden.py produced by
running the real reference. No GPU needed.
"""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import load_golden, split
from _replay import batches, expect_batch_rows, sim_inputs


def ident_cache(num_ids=32, dim=4, cap=8, seed=0, **kw):
    # identity idx_map: counts strictly decreasing in id (test_cache_manager.py:10-14)
    rank_of, id_of = oracle.rank_permutation(np.arange(num_ids, 0, -1))
    ref = oracle.init_rows(num_ids, dim, seed)
    return oracle.OracleCache(rank_of, ref[id_of].copy(), cap, buffer_bytes=4096, reference_rows=ref, **kw), id_of


# ---- known answers from the reference tests ---------------------------------

def test_kat_cold_start():  # test_cache_manager.py:36-41
    c, _ = ident_cache(cap=4)
    p = c.prepare([10, 11])
    assert (p["hits"], p["misses"], p["evictions"]) == (0, 2, 0)
    assert set(c.slot_rank[c.slot_rank >= 0].tolist()) == {10, 11}


def test_kat_alg1_hand_case():  # test_cache_manager.py:44-52
    c, _ = ident_cache(cap=2)
    c.prepare([0, 7], 0)
    p = c.prepare([0, 3], 1)
    assert (p["hits"], p["misses"], p["evictions"]) == (1, 1, 1)
    assert set(c.slot_rank.tolist()) == {0, 3}
    assert p["evicted"].tolist() == [7]


def test_kat_repeat_and_duplicates():  # :55-69
    c, _ = ident_cache(cap=4)
    c.prepare([1, 2, 3], 0)
    p = c.prepare([1, 2, 3], 1)
    assert (p["hits"], p["misses"], p["evictions"]) == (3, 0, 0) and p["reports"] == []
    c2, _ = ident_cache(cap=4)
    p = c2.prepare([5, 5, 5, 2])
    s = c2.occurrence_slots(p)
    assert p["hits"] + p["misses"] == 2 and s[0] == s[1] == s[2]


def test_kat_errors():  # :72-81, :98-102
    c, _ = ident_cache(cap=2)
    with pytest.raises(oracle.OracleBatchExceedsCapacity):
        c.prepare([1, 2, 3])
    c8, _ = ident_cache(num_ids=8, cap=4)
    with pytest.raises(ValueError, match="8"):
        c8.prepare([8])
    c.prepare([2, 5])
    with pytest.raises(oracle.OracleInsufficientEvictable):
        c.select_evictions(1, [2, 5])


def test_kat_select_evictions():  # :84-95
    c, _ = ident_cache(cap=4)
    c.prepare([2, 5, 9, 11])
    s = c.select_evictions(2, [9])
    assert set(c.slot_rank[s].tolist()) == {11, 5}
    assert c.select_evictions(0, []).size == 0


def test_kat_warmup():  # :105-134
    c, _ = ident_cache(cap=6)
    r = c.warmup(6)
    assert set(c.slot_rank.tolist()) == set(range(6)) and r["rows"] == 6 and not c.dirty.any()
    c, _ = ident_cache(cap=4)
    with pytest.raises(ValueError):
        c.warmup(5)
    c.warmup(2)
    with pytest.raises(ValueError, match="empty"):
        c.warmup(1)
    c, _ = ident_cache(cap=8)
    c.warmup(8)
    p = c.prepare([0, 3, 7, 7, 2])
    assert p["misses"] == 0 and p["hits"] == 4


def test_kat_write_back_modes():  # :137-174
    c, _ = ident_cache(cap=2)
    c.prepare([0])
    s = int(c.rank_slot[0])
    c.fast[s] += 1.0
    c.mark_dirty([s])
    upd = c.fast[s].copy()
    c.prepare([4, 5], 1)
    assert np.array_equal(c.slow[0], upd)
    c, _ = ident_cache(cap=2)
    c.prepare([0, 1])
    p = c.prepare([6, 7], 1)
    assert sum(r["bytes"] for r in p["reports"] if r["direction"] == "to_slow") == 0 and p["evictions"] == 2
    c, _ = ident_cache(cap=2, write_back="always")
    before = c.slow.copy()
    c.prepare([0, 1])
    p = c.prepare([6, 7], 1)
    assert sum(r["rows"] for r in p["reports"] if r["direction"] == "to_slow") == 2
    assert np.array_equal(c.slow, before)
    c, _ = ident_cache(cap=2)
    c.prepare([0])
    s = int(c.rank_slot[0])
    c.mark_dirty([s]); c.mark_dirty([s])
    assert c.flush()["rows"] == 1
    with pytest.raises(IndexError):
        c.mark_dirty([2])


def test_kat_flush_gather_scatter():  # :183-221
    c, _ = ident_cache(cap=4)
    c.prepare([1, 2])
    assert c.flush()["bytes"] == 0
    p = c.prepare([1, 2], 1)
    c.scatter_update(p, np.ones((2, 4), np.float32))
    assert c.flush()["rows"] == 2 and c.flush()["rows"] == 0
    c, _ = ident_cache(cap=6)
    ids = np.array([4, 9, 4, 1])
    p = c.prepare(ids)
    assert np.array_equal(c.gather(p), c.reference[ids])
    c, _ = ident_cache(cap=4)
    p = c.prepare([3, 3])
    base = c.fast[p["unique_slots"]].copy()
    c.scatter_update(p, np.full((2, 4), 0.125, np.float32))
    assert np.array_equal(c.fast[p["unique_slots"]], base + 0.25)


def test_kat_paper_literal():  # :224-238
    c, _ = ident_cache(cap=2, evict_mode="paper_literal")
    c.warmup(2)
    with pytest.raises(oracle.OracleInsufficientFreeSlots):
        c.prepare([5])
    c, _ = ident_cache(cap=4, evict_mode="paper_literal")
    assert c.prepare([1, 2])["misses"] == 2 and c.prepare([3, 4], 1)["misses"] == 2


def test_kat_chunk_plan():  # test_transmitter.py:27-47
    MiB = 2 ** 20
    assert oracle.chunk_messages(0, 512, MiB) == 0
    assert oracle.chunk_messages(16384, 512, 64 * MiB) == 1
    assert oracle.chunk_messages(16384, 512, MiB) == 8
    assert oracle.chunk_messages(3, 400, 1000) == 2
    with pytest.raises(oracle.OracleBufferTooSmall):
        oracle.chunk_messages(1, 2 * MiB, MiB)


def test_kat_reorder_and_capacity():  # test_freq_stats.py:95-107; test_store.py:14-23
    counts = np.zeros(10, np.int64)
    counts[[5, 2, 9]] = [3, 2, 1]
    rank_of, id_of = oracle.rank_permutation(counts)
    assert rank_of[5] == 0 and rank_of[2] == 1 and rank_of[9] == 2
    assert list(id_of[3:]) == [0, 1, 3, 4, 6, 7, 8]
    assert np.array_equal(oracle.rank_permutation(np.full(6, 7))[0], np.arange(6))
    assert oracle.fast_capacity(1_000_000, 0.015) == 15_000
    with pytest.warns(UserWarning):
        assert oracle.fast_capacity(100, 0.005) == 1
    assert oracle.column_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]


# ---- golden vectors from the real reference ---------------------------------

@pytest.mark.parametrize("name", ["stream_dirty_zipf", "stream_always_zipf", "stream_dirty_ident"])
def test_golden_random_stream(name):
    g = load_golden(name)
    num_ids, cap, dim, buf, always = (int(v) for v in g["meta"])
    ref = np.empty((num_ids, dim), np.float32)
    ref[g["id_of"]] = g["slow0"]
    c = oracle.OracleCache(g["rank_of"], g["slow0"].copy(), cap, buffer_bytes=buf,
                           write_back="always" if always else "dirty_only", reference_rows=ref)
    ids = split(g["ids"], g["ids_off"])
    deltas = split(g["deltas"], g["ids_off"])
    fields = {k: split(g[k], g[k + "_off"]) for k in
              ("unique_ids", "unique_ranks", "unique_counts", "unique_slots", "evicted", "admitted")}
    for b, batch in enumerate(ids):
        p = c.prepare(batch, b)
        for k in ("unique_ids", "unique_ranks", "unique_counts", "unique_slots", "evicted", "admitted"):
            assert np.array_equal(p[k], fields[k][b]), (b, k)
        rep = np.zeros(6, np.int64)
        for r in p["reports"]:
            o = 0 if r["direction"] == "to_slow" else 3
            rep[o:o + 3] += (r["rows"], r["bytes"], r["messages"])
        assert np.array_equal(np.concatenate([[p["hits"], p["misses"], p["evictions"]], rep]), g["scalars"][b])
        c.scatter_update(p, deltas[b])
        c.check_invariants()
    f = c.flush()
    assert [f["rows"], f["bytes"], f["messages"]] == g["flush"].tolist()
    assert np.array_equal(c.slot_rank, g["slot_to_rank"])
    assert np.array_equal(c.rank_slot, g["rank_to_slot"])
    assert np.array_equal(c.dirty, g["dirty"]) and c.free == int(g["free_count"])
    assert np.array_equal(c.slow, g["slow_final"])  # bitwise
    assert c.first_divergence(g["id_of"]) is None
    assert oracle.replay_law(c.events, num_ids) == []


def run_oracle_sim(g):
    s = sim_inputs(g)
    rank_of, id_of = oracle.rank_permutation(oracle.frequency_counts(s["trace"], s["num_ids"]))
    assert np.array_equal(rank_of, g["rank_of"])
    ref = oracle.init_rows(s["num_ids"], s["dim"], s["init_seed"])
    c = oracle.OracleCache(rank_of, ref[id_of], s["capacity"], buffer_bytes=s["buffer_bytes"],
                           write_back=s["write_back"], reference_rows=ref)
    c.warmup(s["capacity"])
    colw = oracle.column_weights(s["dim"], s["updates_seed"])
    rows = []
    for seq, ids in batches(s["trace"], s["batch_size"]):
        p = c.prepare(ids, seq)
        g_u = oracle.row_scalars(p["unique_ids"], p["unique_counts"], seq, s["updates_seed"])
        c.apply_unique_update(p, g_u[:, None] * colw[None, :])
        to_fast = sum(r["rows"] for r in p["reports"] if r["direction"] == "to_fast")
        to_slow = sum(r["rows"] for r in p["reports"] if r["direction"] == "to_slow")
        msgs = sum(r["messages"] for r in p["reports"])
        rows.append([p["unique_ids"].size, p["hits"], p["misses"], p["evictions"], to_fast, to_slow,
                     to_fast * s["dim"] * 4, to_slow * s["dim"] * 4, msgs])
    c.flush()
    return c, np.array(rows, np.int64), id_of


@pytest.mark.parametrize("name", ["sim_small", "sim_small_always", "sim_medium"])
def test_golden_simulator_run(name):
    g = load_golden(name)
    c, per_batch, id_of = run_oracle_sim(g)
    pb, evicted, admitted = expect_batch_rows(g)
    assert np.array_equal(per_batch, pb)
    evs = [e for e in c.events if e["batch_seq"] >= 0]
    for b, e in enumerate(evs):
        assert np.array_equal(e["evicted"], evicted[b]) and np.array_equal(e["admitted"], admitted[b])
    assert np.array_equal(c.slot_rank, g["slot_to_rank"]) and np.array_equal(c.dirty, g["dirty"])
    assert hashlib.sha256(c.slow.tobytes()).hexdigest() == str(g["slow_final_sha"])
    assert c.first_divergence(id_of) is None


def test_golden_functions():
    g = load_golden("functions")
    cs, offs = g["counts"], g["counts_off"]
    rs = split(g["rank_of"], offs)
    for i, cnt in enumerate(split(cs, offs)):
        assert np.array_equal(oracle.rank_permutation(cnt)[0], rs[i])
    assert np.array_equal(oracle.init_rows(1000, 8, 123), g["init_1000x8_s123"])
    for row, (seq, useed) in zip(g["row_scalars"], ((0, 5), (7, 12345678901234), (1000, 2**63 + 11))):
        assert np.array_equal(oracle.row_scalars(g["hash_ids"], g["hash_counts"], seq, useed), row)
    assert np.array_equal(oracle.column_weights(128, 5), g["colw"][0])
    assert np.array_equal(oracle.column_weights(128, 12345678901234), g["colw"][1])
    caps = [oracle.fast_capacity(n, r) for n, r in ((1_000_000, 0.015), (33_762_577, 0.015), (9_445_823, 0.05),
                                                    (204_184_588, 0.015), (1000, 0.5), (2000, 0.05))]
    assert caps == g["capacities"].tolist()


def test_golden_sharded_lookup():
    g = load_golden("sharded")
    assert [tuple(r) for r in g["ranges3"]] == oracle.column_ranges(10, 3)
    num_ids, dim = 600, 10
    ref = oracle.init_rows(num_ids, dim, 7)
    rank_of = g["rank_of"]
    id_of = np.argsort(rank_of)
    cap = oracle.fast_capacity(num_ids, 0.05)
    for shards in (1, 2, 3, 4):
        caches = [oracle.OracleCache(rank_of, np.ascontiguousarray(ref[:, a:b])[id_of], cap)
                  for a, b in oracle.column_ranges(dim, shards)]
        for c in caches:
            c.warmup(cap)
        out = []
        for seq, ids in batches(g["trace"], 12):
            preps = [c.prepare(ids, seq) for c in caches]
            out.append(np.concatenate([c.gather(p) for c, p in zip(caches, preps)], axis=1))
        assert np.array_equal(np.concatenate(out), g["lookup"])


CASES = [("sum", False), ("mean", False), ("sum", True)]


@pytest.mark.parametrize("ci", [0, 1, 2])
@pytest.mark.parametrize("mode,use_w", CASES)
def test_golden_embedding_bag(ci, mode, use_w):
    g = load_golden("embedding_bag")
    w, idx, off, psw, gout = (g[f"c{ci}_{k}"] for k in ("w", "idx", "off", "psw", "gout"))
    key = f"c{ci}_{mode}{'_w' if use_w else ''}"
    out = oracle.pooled_bag(w, idx, off, psw if use_w else None, mode)
    np.testing.assert_allclose(out, g[key + "_out"], rtol=1e-5, atol=1e-6)
    grad = oracle.pooled_bag_backward_rows(gout, idx, off, w.shape[0], psw if use_w else None, mode)
    np.testing.assert_allclose(grad, g[key + "_grad"], rtol=1e-5, atol=1e-6)
    touched = np.unique(idx)
    for name in ("sgd", "adagrad"):
        rows = w.copy()
        state = np.zeros_like(w)
        for _ in range(2):
            gr = oracle.pooled_bag_backward_rows(gout, idx, off, w.shape[0], psw if use_w else None, mode,
                                                 ) if True else None
            # torch's dense optimizer steps every row; rows with zero grad are unchanged for SGD
            # and Adagrad alike (g=0 -> no change), so a sparse update over the touched rows matches
            gr_rows = np.zeros_like(w, dtype=np.float64)
            gr_rows[touched] = gr[touched]
            if name == "sgd":
                oracle.sparse_sgd(rows, touched, gr_rows, 0.05)
            else:
                oracle.sparse_adagrad(rows, state, touched, gr_rows, 0.05, 1e-10)
        np.testing.assert_allclose(rows, g[key + f"_{name}2"], rtol=1e-5, atol=1e-6)


def test_mean_with_weights_rule():
    rows = np.arange(12, dtype=np.float32).reshape(4, 3)
    out = oracle.pooled_bag(rows, [0, 1, 3], [0, 2, 3], [0.5, 2.0, 1.0], mode="mean")
    np.testing.assert_allclose(out[0], (0.5 * rows[0] + 2.0 * rows[1]) / 2)
    np.testing.assert_allclose(out[1], rows[3])
    np.testing.assert_allclose(out[2], 0.0)  # empty bag


def test_golden_buffer_too_small_ordering():
    """A row larger than the staging buffer, replayed against the REAL reference's
    recorded outcome of every call: which calls raise BufferTooSmall, and the slot
    table, dirty bits, free count and slow tier after each (a dirty write-back raises
    before any mutation; clean victims are evicted before the admission raises)."""
    from _replay import bts_calls

    g = load_golden("buffer_too_small")
    num_ids, cap, dim = (int(v) for v in g["meta"])
    c = oracle.OracleCache(np.arange(num_ids), g["slow0"].copy(), cap)
    for k, (verb, buf, wb, ids) in enumerate(bts_calls(g)):
        c.buffer_bytes, c.write_back = buf, wb
        raised = 0
        try:
            if verb == "flush":
                c.flush()
            else:
                p = c.prepare(ids, k)
                if verb == "update":
                    c.scatter_update(p, np.full((ids.size, dim), 0.25, np.float32))
        except oracle.OracleBufferTooSmall:
            raised = 1
        assert raised == g["raised"][k], k
        assert np.array_equal(c.slot_rank, g["slot_to_rank"][k]), k
        assert np.array_equal(c.dirty, g["dirty"][k]) and c.free == g["free_count"][k], k
        assert np.array_equal(c.slow, g["slow"][k]), k
