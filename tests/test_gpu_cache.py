"""GPU parity: the CUDA cache (through the C ABI) against the reference's golden
vectors and the numpy oracle, bit-exact for every index/state output and for the
post-flush slow tier. Mirrors /root/reference/pkg/tests/test_cache_manager.py."""

import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from conftest import load_golden, split  # noqa: E402
from _replay import batches, expect_batch_rows, sim_inputs  # noqa: E402

pytestmark = pytest.mark.gpu

import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200 import cache_manager as cm  # noqa: E402


def identity_idx_map(num_ids):
    counts = np.arange(num_ids, 0, -1, dtype=np.int64)
    return fc.build_reorder(fc.FrequencyTable(counts=counts, num_ids=num_ids))


def build_stack(num_ids=32, dim=4, capacity=8, seed=0, **kw):
    idx = identity_idx_map(num_ids)
    slow, _, ref = fc.init_stores(num_ids, dim, capacity / num_ids, init_seed=seed, idx_map=idx)
    fast = fc.FastTierStore(slots=np.zeros((capacity, dim), dtype=np.float32))
    return fc.CacheStack(idx_map=idx, slow=slow, fast=fast, transmitter=fc.Transmitter(buffer=fc.TransferBuffer(4096)),
                         reference=ref, log_events=True, **kw)


def occupied(stack):
    return set(stack.state.occupied_ranks().tolist())


# ---------------- known answers (test_cache_manager.py) --------------------

def test_cold_start_two_misses():
    st = build_stack(capacity=4)
    p = st.prepare([10, 11], batch_seq=0)
    assert (p.hits, p.misses, p.evictions) == (0, 2, 0)
    assert occupied(st) == {10, 11}
    assert p.slot_of().keys() == {10, 11}


def test_alg1_hand_simulation():
    st = build_stack(capacity=2)
    st.prepare([0, 7], batch_seq=0)
    p = st.prepare([0, 3], batch_seq=1)
    assert (p.hits, p.misses, p.evictions) == (1, 1, 1)
    assert occupied(st) == {0, 3}
    assert st.events[-1].evicted_ranks.tolist() == [7]


def test_repeat_batch_and_duplicates():
    st = build_stack(capacity=4)
    st.prepare([1, 2, 3], batch_seq=0)
    p = st.prepare([1, 2, 3], batch_seq=1)
    assert (p.hits, p.misses, p.evictions) == (3, 0, 0)
    assert sum(r.bytes for r in p.transfer_reports) == 0
    st = build_stack(capacity=4)
    p = st.prepare([5, 5, 5, 2], batch_seq=0)
    s = p.slots_for_ids()
    assert p.hits + p.misses == 2 and s.shape == (4,) and s[0] == s[1] == s[2]


def test_errors_leave_state_untouched():
    st = build_stack(capacity=2)
    st.prepare([4], batch_seq=0)
    before = (st.state.slot_to_rank.copy(), st.state.rank_to_slot.copy(), st.state.free_count)
    with pytest.raises(cm.BatchExceedsCapacity):
        st.prepare([1, 2, 3], batch_seq=1)
    st8 = build_stack(num_ids=8, capacity=4)
    with pytest.raises(ValueError, match="8"):
        st8.prepare([8], batch_seq=0)
    with pytest.raises(ValueError, match="-3"):
        st8.prepare([1, -3, 9], batch_seq=0)
    after = (st.state.slot_to_rank, st.state.rank_to_slot, st.state.free_count)
    assert np.array_equal(before[0], after[0]) and np.array_equal(before[1], after[1]) and before[2] == after[2]
    # the failed calls left no per-batch residue: the next batch is exact
    p = st.prepare([4, 6], batch_seq=2)
    assert (p.hits, p.misses, p.evictions) == (1, 1, 0)
    st.state.check_invariants()


def test_select_evictions():
    st = build_stack(capacity=4)
    st.prepare([2, 5, 9, 11], batch_seq=0)
    slots = cm.select_evictions(st.state, 2, protected_ranks=[9])
    assert set(st.state.slot_to_rank[slots].tolist()) == {11, 5}
    assert st.state.slot_to_rank[slots].tolist() == [11, 5]  # descending ranks
    assert cm.select_evictions(st.state, 0, protected_ranks=[]).size == 0
    st2 = build_stack(capacity=2)
    st2.prepare([2, 5], batch_seq=0)
    with pytest.raises(cm.InsufficientEvictable):
        cm.select_evictions(st2.state, 1, protected_ranks=[2, 5])


def test_warmup():
    st = build_stack(capacity=6)
    rep = st.warmup(6)
    assert occupied(st) == set(range(6)) and rep.rows == 6 and not st.state.dirty.any()
    st = build_stack(capacity=4)
    assert st.warmup(0).rows == 0 and st.state.free_count == 4
    with pytest.raises(ValueError):
        st.warmup(5)
    st.warmup(2)
    with pytest.raises(ValueError, match="empty"):
        st.warmup(1)
    st = build_stack(capacity=8)
    st.warmup(8)
    p = st.prepare([0, 3, 7, 7, 2], batch_seq=0)
    assert p.misses == 0 and p.hits == 4


def test_dirty_write_back_and_modes():
    st = build_stack(capacity=2)
    st.prepare([0], batch_seq=0)
    slot = int(st.state.rank_to_slot[0])
    st.fast.slots[slot] += 1.0
    cm.mark_dirty(st.state, [slot])
    updated = st.fast.slots[slot].cpu().numpy().copy()
    st.prepare([4, 5], batch_seq=1)  # evicts rank 0
    torch.cuda.synchronize()
    assert np.array_equal(st.slow.rows[0], updated)
    st = build_stack(capacity=2)
    st.prepare([0, 1], batch_seq=0)
    p = st.prepare([6, 7], batch_seq=1)
    assert sum(r.bytes for r in p.transfer_reports if r.direction == "to_slow") == 0 and p.evictions == 2
    st = build_stack(capacity=2, write_back="always")
    before = st.slow.rows.copy()
    st.prepare([0, 1], batch_seq=0)
    p = st.prepare([6, 7], batch_seq=1)
    torch.cuda.synchronize()
    assert sum(r.rows for r in p.transfer_reports if r.direction == "to_slow") == 2
    assert np.array_equal(st.slow.rows, before)
    st = build_stack(capacity=2)
    st.prepare([0], batch_seq=0)
    slot = int(st.state.rank_to_slot[0])
    cm.mark_dirty(st.state, [slot])
    cm.mark_dirty(st.state, [slot])
    assert st.flush().rows == 1
    with pytest.raises(IndexError):
        cm.mark_dirty(st.state, [2])


def test_flush_gather_scatter():
    st = build_stack(capacity=4)
    st.prepare([1, 2], batch_seq=0)
    assert st.flush().bytes == 0
    p = st.prepare([1, 2], batch_seq=1)
    st.scatter_update(p, np.ones((2, 4), dtype=np.float32))
    assert st.flush().rows == 2 and st.flush().rows == 0
    assert occupied(st) == {1, 2}
    st = build_stack(capacity=6)
    ids = np.array([4, 9, 4, 1])
    p = st.prepare(ids, batch_seq=0)
    assert np.array_equal(st.gather(p).cpu().numpy(), st.reference.rows[ids])
    st = build_stack(capacity=4)
    p = st.prepare([1, 2], batch_seq=0)
    before = st.fast.slots.cpu().numpy().copy()
    st.scatter_update(p, np.zeros((2, 4), dtype=np.float32))
    assert np.array_equal(st.fast.slots.cpu().numpy(), before)
    assert st.state.dirty[p.unique_slots].all()
    st = build_stack(capacity=4)
    p = st.prepare(np.array([3, 3]), batch_seq=0)
    base = st.fast.slots.cpu().numpy()[p.unique_slots].copy()
    st.scatter_update(p, np.full((2, 4), 0.125, dtype=np.float32))
    assert np.array_equal(st.fast.slots.cpu().numpy()[p.unique_slots], base + 0.25)


def test_paper_literal():
    st = build_stack(capacity=2, evict_mode="paper_literal")
    st.warmup(2)
    with pytest.raises(cm.InsufficientFreeSlots):
        st.prepare([5], batch_seq=0)
    st = build_stack(capacity=4, evict_mode="paper_literal")
    assert st.prepare([1, 2], batch_seq=0).misses == 2
    assert st.prepare([3, 4], batch_seq=1).misses == 2


def test_buffer_too_small():
    idx = identity_idx_map(16)
    slow, _, _ = fc.init_stores(16, 8, 0.25, init_seed=0, idx_map=idx)
    st = fc.CacheStack(idx, slow, fc.FastTierStore(np.zeros((4, 8), np.float32)),
                       fc.Transmitter(buffer=fc.TransferBuffer(16)))
    with pytest.raises(fc.BufferTooSmall):
        st.prepare([1, 2], batch_seq=0)
    assert st.state.free_count == 4


@pytest.mark.parametrize("engine", ["zerocopy", "async"])
def test_golden_buffer_too_small_ordering(engine):
    """A row larger than the transmitter's staging buffer, call by call against the REAL
    reference's recorded outcome (tests/golden/buffer_too_small.npz): which calls raise
    BufferTooSmall and the slot table, dirty bits, free count and slow tier after each.
    A dirty write-back raises before any mutation; clean victims are evicted before the
    admission raises; hits raise nothing. The transmitter is passed per call, as in the
    reference's functional API."""
    from _replay import bts_calls

    g = load_golden("buffer_too_small")
    num_ids, cap, dim = (int(v) for v in g["meta"])
    idx = identity_idx_map(num_ids)
    state = cm.CacheState(cap, num_ids)
    slow = fc.SlowTierStore(g["slow0"].copy())
    fast = fc.FastTierStore(np.zeros((cap, dim), np.float32))
    state.bind(idx, slow, fast, fc.Transmitter(), engine=engine)
    for k, (verb, buf, wb, ids) in enumerate(bts_calls(g)):
        tx = fc.Transmitter(buffer=fc.TransferBuffer(buf))
        raised = 0
        try:
            if verb == "flush":
                cm.flush(state, tx, slow, fast)
            else:
                p = cm.prepare_cache(state, idx, ids, tx, slow, fast, write_back=wb, batch_seq=k)
                if verb == "update":
                    cm.scatter_update(state, fast, p, np.full((ids.size, dim), 0.25, np.float32))
        except fc.BufferTooSmall:
            raised = 1
        state.device.drain()
        torch.cuda.synchronize()
        assert raised == g["raised"][k], k
        assert np.array_equal(state.slot_to_rank, g["slot_to_rank"][k]), k
        assert np.array_equal(state.dirty, g["dirty"][k]) and state.free_count == g["free_count"][k], k
        assert np.array_equal(slow.rows, g["slow"][k]), k
        state.check_invariants()
    # the prefetch pipeline needs one row to fit (it decides before the dirty bits are final)
    dev = state.device
    if engine == "async":
        dev.set_buffer_bytes(16)
        with pytest.raises(fc.BufferTooSmall):
            dev.prepare_begin(np.array([1]))


def test_event_log_jsonl_roundtrip(tmp_path):
    st = build_stack(capacity=2)
    st.prepare([0, 7], batch_seq=0)
    st.prepare([0, 3], batch_seq=1)
    path = tmp_path / "events.jsonl"
    cm.write_events_jsonl(st.events, path)
    loaded = cm.read_events_jsonl(path)
    assert len(loaded) == 2 and loaded[1].evicted_ranks.tolist() == [7] and loaded[1].policy == "freq_lfu"


def test_fault_injection_detected():
    st = build_stack(num_ids=16, capacity=4, seed=2)
    p = st.prepare([5], batch_seq=0)
    st.scatter_update(p, np.ones((1, 4), dtype=np.float32))
    st.state.clear_dirty()
    st.flush()
    div = st.first_divergence()
    assert div is not None and div["id"] == 5


# ---------------- golden vectors from the real reference ------------------

def golden_stack(g, write_back):
    num_ids, cap, dim, buf, _ = (int(v) for v in g["meta"])
    idx = fc.IdxMap(rank_of=g["rank_of"], id_of=g["id_of"])
    ref = np.empty((num_ids, dim), np.float32)
    ref[g["id_of"]] = g["slow0"]
    return fc.CacheStack(idx, fc.SlowTierStore(g["slow0"].copy()), fc.FastTierStore(np.zeros((cap, dim), np.float32)),
                         fc.Transmitter(buffer=fc.TransferBuffer(buf)), reference=fc.ReferenceStore(ref),
                         write_back=write_back, log_events=True)


@pytest.mark.parametrize("name", ["stream_dirty_zipf", "stream_always_zipf", "stream_dirty_ident"])
def test_golden_random_stream(name):
    g = load_golden(name)
    st = golden_stack(g, "always" if int(g["meta"][4]) else "dirty_only")
    ids = split(g["ids"], g["ids_off"])
    deltas = split(g["deltas"], g["ids_off"])
    want = {k: split(g[k], g[k + "_off"]) for k in
            ("unique_ids", "unique_ranks", "unique_counts", "unique_slots", "evicted", "admitted")}
    for b, batch in enumerate(ids):
        p = st.prepare(batch, b)
        got = {"unique_ids": p.unique_ids, "unique_ranks": p.unique_ranks, "unique_counts": p.unique_counts,
               "unique_slots": p.unique_slots, "evicted": st.events[-1].evicted_ranks,
               "admitted": st.events[-1].admitted_ranks}
        for k in want:
            assert np.array_equal(got[k], want[k][b]), (b, k, got[k], want[k][b])
        rep = np.zeros(6, np.int64)
        for r in p.transfer_reports:
            o = 0 if r.direction == "to_slow" else 3
            rep[o:o + 3] += (r.rows, r.bytes, r.messages)
        assert np.array_equal(np.concatenate([[p.hits, p.misses, p.evictions], rep]), g["scalars"][b]), b
        st.scatter_update(p, deltas[b])
    f = st.flush()
    assert [f.rows, f.bytes, f.messages] == g["flush"].tolist()
    assert np.array_equal(st.state.slot_to_rank, g["slot_to_rank"])
    assert np.array_equal(st.state.rank_to_slot, g["rank_to_slot"])
    assert np.array_equal(st.state.dirty, g["dirty"]) and st.state.free_count == int(g["free_count"])
    assert np.array_equal(st.slow.rows, g["slow_final"])  # bitwise
    assert st.first_divergence() is None


def run_gpu_sim(g, update="synthetic"):
    """update="synthetic": the fused on-device update (k_synthetic); "unique": the
    reference simulator's own path (simulator.py:429-433), host row_scalars x column
    weights through CacheStack.apply_unique_update (k_unique_add), with every batch's
    gather_unique rows checked bitwise against the dense mirror first."""
    s = sim_inputs(g)
    freq = fc.scan_frequencies(s["trace"], s["num_ids"])
    idx = fc.build_reorder(freq)
    assert np.array_equal(idx.rank_of, g["rank_of"])
    slow, fast, ref = fc.init_stores(s["num_ids"], s["dim"], s["capacity"] / s["num_ids"], s["init_seed"], idx)
    fast = fc.FastTierStore(np.zeros((s["capacity"], s["dim"]), np.float32))
    st = fc.CacheStack(idx, slow, fast, fc.Transmitter(buffer=fc.TransferBuffer(s["buffer_bytes"])), reference=ref,
                       write_back=s["write_back"], log_events=True)
    st.warmup(s["capacity"])
    colw = fc.update_column_weights(s["dim"], s["updates_seed"])
    rows = []
    for seq, ids in batches(s["trace"], s["batch_size"]):
        p = st.prepare(ids, seq)
        rows_u = st.gather_unique(p)
        if update == "synthetic":
            st.apply_synthetic_update(p, seq, s["updates_seed"], colw)
        else:
            assert np.array_equal(rows_u.cpu().numpy(), st.reference.rows[p.unique_ids]), seq  # bitwise
            gs = fc.update_row_scalars(p.unique_ids, p.unique_counts, seq, s["updates_seed"])
            st.apply_unique_update(p, gs[:, None] * colw[None, :])
        tf = sum(r.rows for r in p.transfer_reports if r.direction == "to_fast")
        ts = sum(r.rows for r in p.transfer_reports if r.direction == "to_slow")
        rows.append([p.num_unique, p.hits, p.misses, p.evictions, tf, ts, tf * s["dim"] * 4, ts * s["dim"] * 4,
                     sum(r.messages for r in p.transfer_reports)])
    st.flush()
    torch.cuda.synchronize()
    return st, np.array(rows, np.int64)


@pytest.mark.parametrize("name", ["sim_small", "sim_small_always", "sim_medium"])
@pytest.mark.parametrize("update", ["synthetic", "unique"])
def test_golden_simulator_run(name, update):
    g = load_golden(name)
    st, per_batch = run_gpu_sim(g, update)
    pb, evicted, admitted = expect_batch_rows(g)
    assert np.array_equal(per_batch, pb)
    evs = [e for e in st.events if e.batch_seq >= 0]
    for b, e in enumerate(evs):
        assert np.array_equal(e.evicted_ranks, evicted[b]), b
        assert np.array_equal(e.admitted_ranks, admitted[b]), b
    assert np.array_equal(st.state.slot_to_rank, g["slot_to_rank"])
    assert np.array_equal(st.state.dirty, g["dirty"])
    assert hashlib.sha256(st.slow.rows.tobytes()).hexdigest() == str(g["slow_final_sha"])
    assert st.first_divergence() is None


def test_golden_sharded_lookup():
    g = load_golden("sharded")
    num_ids, dim = 600, 10
    idx = fc.IdxMap(rank_of=g["rank_of"], id_of=np.argsort(g["rank_of"]))
    for shards in (1, 2, 3, 4):
        stacks = fc.build_column_stacks(idx, fc.partition_columns(dim, shards), dim, 0.05, init_seed=7)
        for s in stacks:
            s.warmup(s.capacity)
        out = [fc.sharded_lookup(stacks, ids, seq).cpu().numpy() for seq, ids in batches(g["trace"], 12)]
        assert np.array_equal(np.concatenate(out), g["lookup"]), shards


# ---------------- randomized parity at larger sizes against the oracle ------

@pytest.mark.parametrize("num_ids,cap,dim,nb,bsz,always,engine", [
    (50_000, 3_000, 32, 40, 2_000, False, "zerocopy"),
    (200_000, 12_000, 128, 12, 9_000, True, "zerocopy"),
    (7_001, 700, 12, 30, 500, False, "zerocopy"),
    (50_000, 3_000, 32, 40, 2_000, False, "async"),
    (200_000, 12_000, 128, 12, 9_000, True, "async"),
    (3_000, 400, 16, 60, 350, False, "async"),  # tiny cache: ranks bounce out and back in while pending
])
def test_random_parity_vs_oracle(num_ids, cap, dim, nb, bsz, always, engine):
    rng = np.random.default_rng(num_ids)
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.05
    perm = rng.permutation(num_ids)
    trace = perm[rng.choice(num_ids, size=(nb, bsz), p=p / p.sum())]
    counts = oracle.frequency_counts(trace, num_ids)
    rank_of, id_of = oracle.rank_permutation(counts)
    ref = oracle.init_rows(num_ids, dim, 3)
    wb = "always" if always else "dirty_only"
    orc = oracle.OracleCache(rank_of, ref[id_of].copy(), cap, write_back=wb, buffer_bytes=1 << 16)
    st = fc.CacheStack(fc.IdxMap(rank_of, id_of), fc.SlowTierStore(ref[id_of].copy()),
                       fc.FastTierStore(np.zeros((cap, dim), np.float32)),
                       fc.Transmitter(buffer=fc.TransferBuffer(1 << 16)), write_back=wb, log_events=True,
                       engine=engine)
    orc.warmup(cap // 2)
    st.warmup(cap // 2)
    colw = oracle.column_weights(dim, 9)
    for b in range(nb):
        a = orc.prepare(trace[b], b)
        q = st.prepare(trace[b], b)
        for k in ("unique_ids", "unique_ranks", "unique_counts", "unique_slots"):
            assert np.array_equal(getattr(q, k), a[k]), (b, k)
        assert (q.hits, q.misses, q.evictions) == (a["hits"], a["misses"], a["evictions"])
        assert np.array_equal(st.events[-1].evicted_ranks, a["evicted"])
        assert np.array_equal(st.events[-1].admitted_ranks, a["admitted"])
        assert np.array_equal(q.slots_for_ids(), orc.occurrence_slots(a))
        gs = oracle.row_scalars(a["unique_ids"], a["unique_counts"], b, 9)
        orc.apply_unique_update(a, gs[:, None] * colw[None, :])
        st.apply_synthetic_update(q, b, 9, colw)
    assert st.flush().rows == orc.flush()["rows"]
    torch.cuda.synchronize()
    assert np.array_equal(st.state.slot_to_rank, orc.slot_rank)
    assert np.array_equal(st.state.rank_to_slot, orc.rank_slot)
    assert np.array_equal(st.slow.rows, orc.slow)
    st.state.check_invariants()


def test_empty_batch():
    st = build_stack(capacity=4)
    p = st.prepare(np.empty(0, dtype=np.int64), batch_seq=0)
    assert (p.hits, p.misses, p.evictions) == (0, 0, 0) and p.unique_ids.size == 0
    assert st.gather(p).shape == (0, 4)
