"""GPU parity of the prefetch pipeline (fc_prepare_begin / fc_prepare_commit).

Batch t+1's prepare is launched BEFORE batch t's row update runs (the update is
queued on the main stream after the prefetch), exactly the overlap the pipeline
exists for. Everything must stay bit-identical to the sequential reference order
prepare(t) -> update(t) -> prepare(t+1): unique ids / ranks / counts / slots,
hits / misses / evictions, evicted and admitted lists, transfer reports, slot
tables, dirty bits and the post-flush slow tier (reference:
/root/reference/pkg/src/freqcache/cache_manager.py:234-348, simulator.py:416-461)."""

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
from paper_2208_05321_b200.embedding import CachedEmbeddingBag  # noqa: E402


def golden_stack(g, write_back):
    num_ids, cap, dim, buf, _ = (int(v) for v in g["meta"])
    idx = fc.IdxMap(rank_of=g["rank_of"], id_of=g["id_of"])
    ref = np.empty((num_ids, dim), np.float32)
    ref[g["id_of"]] = g["slow0"]
    return fc.CacheStack(idx, fc.SlowTierStore(g["slow0"].copy()), fc.FastTierStore(np.zeros((cap, dim), np.float32)),
                         fc.Transmitter(buffer=fc.TransferBuffer(buf)), reference=fc.ReferenceStore(ref),
                         write_back=write_back, log_events=True, engine="async")


@pytest.mark.parametrize("name", ["stream_dirty_zipf", "stream_always_zipf", "stream_dirty_ident"])
def test_prefetched_golden_stream(name):
    g = load_golden(name)
    st = golden_stack(g, "always" if int(g["meta"][4]) else "dirty_only")
    ids = split(g["ids"], g["ids_off"])
    deltas = split(g["deltas"], g["ids_off"])
    want = {k: split(g[k], g[k + "_off"]) for k in
            ("unique_ids", "unique_ranks", "unique_counts", "unique_slots", "evicted", "admitted")}
    p = st.prepare(ids[0], 0)
    for b in range(len(ids)):
        got = {"unique_ids": p.unique_ids, "unique_ranks": p.unique_ranks, "unique_counts": p.unique_counts,
               "unique_slots": p.unique_slots, "evicted": st.events[-1].evicted_ranks,
               "admitted": st.events[-1].admitted_ranks}
        for k in want:
            assert np.array_equal(got[k], want[k][b]), (b, k)
        rep = np.zeros(6, np.int64)
        for r in p.transfer_reports:
            o = 0 if r.direction == "to_slow" else 3
            rep[o:o + 3] += (r.rows, r.bytes, r.messages)
        assert np.array_equal(np.concatenate([[p.hits, p.misses, p.evictions], rep]), g["scalars"][b]), b
        if b + 1 < len(ids):
            st.prefetch(ids[b + 1], b + 1)  # batch b+1's prepare is in flight ...
        st.scatter_update(p, deltas[b])     # ... while batch b's update is queued behind it
        if b + 1 < len(ids):
            p = st.prepare(ids[b + 1], b + 1)  # commit
    f = st.flush()
    assert [f.rows, f.bytes, f.messages] == g["flush"].tolist()
    assert np.array_equal(st.state.slot_to_rank, g["slot_to_rank"])
    assert np.array_equal(st.state.rank_to_slot, g["rank_to_slot"])
    assert np.array_equal(st.state.dirty, g["dirty"]) and st.state.free_count == int(g["free_count"])
    assert np.array_equal(st.slow.rows, g["slow_final"])  # bitwise
    assert st.first_divergence() is None


@pytest.mark.parametrize("name", ["sim_small", "sim_small_always", "sim_medium"])
def test_prefetched_simulator_run(name):
    g = load_golden(name)
    s = sim_inputs(g)
    idx = fc.build_reorder(fc.scan_frequencies(s["trace"], s["num_ids"]))
    slow, _, ref = fc.init_stores(s["num_ids"], s["dim"], s["capacity"] / s["num_ids"], s["init_seed"], idx)
    fast = fc.FastTierStore(np.zeros((s["capacity"], s["dim"]), np.float32))
    st = fc.CacheStack(idx, slow, fast, fc.Transmitter(buffer=fc.TransferBuffer(s["buffer_bytes"])), reference=ref,
                       write_back=s["write_back"], log_events=True, engine="async")
    st.warmup(s["capacity"])
    colw = fc.update_column_weights(s["dim"], s["updates_seed"])
    bl = list(batches(s["trace"], s["batch_size"]))
    rows = []
    p = st.prepare(bl[0][1], 0)
    for i, (seq, _) in enumerate(bl):
        tf = sum(r.rows for r in p.transfer_reports if r.direction == "to_fast")
        ts = sum(r.rows for r in p.transfer_reports if r.direction == "to_slow")
        rows.append([p.num_unique, p.hits, p.misses, p.evictions, tf, ts, tf * s["dim"] * 4, ts * s["dim"] * 4,
                     sum(r.messages for r in p.transfer_reports)])
        if i + 1 < len(bl):
            st.prefetch(bl[i + 1][1], bl[i + 1][0])
        st.gather_unique(p)
        st.apply_synthetic_update(p, seq, s["updates_seed"], colw)
        if i + 1 < len(bl):
            p = st.prepare(bl[i + 1][1], bl[i + 1][0])
    st.flush()
    torch.cuda.synchronize()
    pb, evicted, admitted = expect_batch_rows(g)
    assert np.array_equal(np.array(rows, np.int64), pb)
    evs = [e for e in st.events if e.batch_seq >= 0]
    for b, e in enumerate(evs):
        assert np.array_equal(e.evicted_ranks, evicted[b]), b
        assert np.array_equal(e.admitted_ranks, admitted[b]), b
    assert np.array_equal(st.state.slot_to_rank, g["slot_to_rank"])
    assert np.array_equal(st.state.dirty, g["dirty"])
    assert hashlib.sha256(st.slow.rows.tobytes()).hexdigest() == str(g["slow_final_sha"])


@pytest.mark.parametrize("depth", [1, 2])
@pytest.mark.parametrize("num_ids,cap,dim,nb,bsz,always", [
    (50_000, 3_000, 32, 40, 2_000, False),
    (200_000, 12_000, 128, 12, 9_000, True),
    (3_000, 400, 16, 60, 350, False),   # tiny cache: ranks bounce out and back while their write-back is pending
    (5_000, 900, 8, 50, 600, False),
])
def test_prefetched_random_parity_vs_oracle(num_ids, cap, dim, nb, bsz, always, depth):
    """depth 1: prefetch(b+1) after prepare(b); depth 2: prefetch(b+1) BEFORE prepare(b),
    so two prefetches are outstanding and batch b+1's index phase runs ahead of commit(b)."""
    rng = np.random.default_rng(num_ids + 1)
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.05
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(nb, bsz), p=p / p.sum())]
    rank_of, id_of = oracle.rank_permutation(oracle.frequency_counts(trace, num_ids))
    ref = oracle.init_rows(num_ids, dim, 3)
    wb = "always" if always else "dirty_only"
    orc = oracle.OracleCache(rank_of, ref[id_of].copy(), cap, write_back=wb, buffer_bytes=1 << 16)
    st = fc.CacheStack(fc.IdxMap(rank_of, id_of), fc.SlowTierStore(ref[id_of].copy()),
                       fc.FastTierStore(np.zeros((cap, dim), np.float32)),
                       fc.Transmitter(buffer=fc.TransferBuffer(1 << 16)), write_back=wb, log_events=True,
                       engine="async")
    orc.warmup(cap // 2)
    st.warmup(cap // 2)
    colw = oracle.column_weights(dim, 9)
    ids = [trace[b] for b in range(nb)]
    if depth == 1:
        q = st.prepare(ids[0], 0)
    else:
        st.prefetch(ids[0], 0)
    for b in range(nb):
        if depth == 2:
            if b + 1 < nb:
                st.prefetch(ids[b + 1], b + 1)
            q = st.prepare(ids[b], b)  # commits the older of the two outstanding prefetches
        a = orc.prepare(ids[b], b)
        for k in ("unique_ids", "unique_ranks", "unique_counts", "unique_slots"):
            assert np.array_equal(getattr(q, k), a[k]), (b, k)
        assert (q.hits, q.misses, q.evictions) == (a["hits"], a["misses"], a["evictions"])
        assert np.array_equal(st.events[-1].evicted_ranks, a["evicted"])
        assert np.array_equal(st.events[-1].admitted_ranks, a["admitted"])
        assert np.array_equal(q.slots_for_ids(), orc.occurrence_slots(a))
        if b + 1 < nb and depth == 1:
            st.prefetch(ids[b + 1], b + 1)
        gs = oracle.row_scalars(a["unique_ids"], a["unique_counts"], b, 9)
        orc.apply_unique_update(a, gs[:, None] * colw[None, :])
        st.apply_synthetic_update(q, b, 9, colw)
        if b + 1 < nb and depth == 1:
            q = st.prepare(ids[b + 1], b + 1)
    assert st.flush().rows == orc.flush()["rows"]
    torch.cuda.synchronize()
    assert np.array_equal(st.state.slot_to_rank, orc.slot_rank)
    assert np.array_equal(st.state.rank_to_slot, orc.rank_slot)
    assert np.array_equal(st.slow.rows, orc.slow)
    st.state.check_invariants()


def test_prefetch_errors_and_mixing():
    num_ids, cap, dim = 64, 4, 8
    idx = fc.IdxMap(np.arange(num_ids), np.arange(num_ids))
    slow, _, ref = fc.init_stores(num_ids, dim, cap / num_ids, init_seed=1, idx_map=idx)
    st = fc.CacheStack(idx, slow, fc.FastTierStore(np.zeros((cap, dim), np.float32)), fc.Transmitter(),
                       reference=ref, log_events=True, engine="async")
    st.prepare(np.array([1, 2]), 0)
    before = (st.state.slot_to_rank.copy(), st.state.rank_to_slot.copy(), st.state.free_count)
    bad = np.array([1, 2, 3, 4, 5])
    st.prefetch(bad, 1)
    with pytest.raises(cm.BatchExceedsCapacity):  # reported at commit; nothing mutated
        st.prepare(bad, 1)
    assert np.array_equal(st.state.slot_to_rank, before[0]) and st.state.free_count == before[2]
    oob = np.array([3, 99])
    st.prefetch(oob, 2)
    with pytest.raises(ValueError, match="99"):
        st.prepare(oob, 2)
    # a sync verb refuses while a prefetch is outstanding
    nxt = np.array([7, 8])
    st.prefetch(nxt, 3)
    with pytest.raises(Exception):
        st.state.device.flush()
    p = st.prepare(nxt, 3)  # commits the prefetch
    assert (p.hits, p.misses, p.evictions) == (0, 2, 0)
    # a prefetch of X followed by prepare(Y): X is executed first, then Y
    x, y = np.array([9, 10]), np.array([11, 12])
    st.prefetch(x, 4)
    p = st.prepare(y, 5)
    assert (p.hits, p.misses, p.evictions) == (0, 2, 2)
    # X evicted the largest unprotected ranks 8, 7; Y then evicted 10, 9 (identity reorder)
    assert set(st.state.occupied_ranks().tolist()) == {1, 2, 11, 12}
    # mix pipelined and synchronous prepares; then flush matches the reference mirror
    q = st.prepare(np.array([9, 11]), 6)
    st.scatter_update(q, np.ones((2, dim), np.float32))
    st.prefetch(np.array([1, 2, 3]), 7)
    q = st.prepare(np.array([1, 2, 3]), 7)
    st.scatter_update(q, np.full((3, dim), 0.5, np.float32))
    st.flush()
    torch.cuda.synchronize()
    assert st.first_divergence() is None
    st.state.check_invariants()


@pytest.mark.parametrize("optimizer,mode,bags", [("sgd", "sum", False), ("adagrad", "mean", True)])
def test_module_prefetch_depth2_matches_sequential(optimizer, mode, bags):
    """prefetch(t+1) called BEFORE forward(t) (two outstanding): bit-identical tables and
    optimizer state to training without prefetch."""
    rng = np.random.default_rng(15)
    num_ids, dim, steps, B = 20_000, 32, 10, 3_000
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.1
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(steps, B), p=p / p.sum())]
    w0 = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
    idx = fc.build_reorder(fc.scan_frequencies(trace, num_ids))
    grads = [rng.standard_normal((B // 3 if bags else B, dim)).astype(np.float32) for _ in range(steps)]
    offs = torch.arange(0, B, 3) if bags else None

    def train(depth2):
        m = CachedEmbeddingBag(num_ids, dim, 0.1, mode=mode, weight=w0, idx_map=idx, optimizer=optimizer, lr=0.05)
        ids = [torch.from_numpy(trace[s]) for s in range(steps)]
        if depth2:
            m.prefetch(ids[0])
        for s in range(steps):
            if depth2 and s + 1 < steps:
                m.prefetch(ids[s + 1])
                assert m.cache.prefetch_depth == 2
            out = m(ids[s], offs)
            out.backward(torch.from_numpy(grads[s]).cuda())
        m.flush()
        return m.weight().copy(), (m.optimizer_state().copy() if optimizer == "adagrad" else None)

    w_seq, s_seq = train(False)
    w_pf, s_pf = train(True)
    assert np.array_equal(w_seq, w_pf)
    if s_seq is not None:
        assert np.array_equal(s_seq, s_pf)


def test_module_prefetch_two_ahead_before_backward():
    """prefetch(t+2) after forward(t) and BEFORE backward(t), with t+1 still outstanding:
    t+2's miss staging must wait for commit(t+1)'s write-back marks (a dirty row evicted
    by t+1 and re-admitted by t+2 comes from the write-back stage, not the stale slow
    tier). Small cache + skewed ids make that round trip frequent. Bit-identical to
    training without prefetch."""
    rng = np.random.default_rng(21)
    num_ids, dim, steps, B = 6_000, 32, 14, 2_000
    p = 1.0 / np.arange(1, num_ids + 1) ** 0.9
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(steps, B), p=p / p.sum())]
    w0 = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
    idx = fc.build_reorder(fc.scan_frequencies(trace, num_ids))
    grads = [rng.standard_normal((B, dim)).astype(np.float32) for _ in range(steps)]

    def train(ahead):
        m = CachedEmbeddingBag(num_ids, dim, 0.25, mode="sum", weight=w0, idx_map=idx, lr=0.05)
        ids = [torch.from_numpy(trace[s]) for s in range(steps)]
        if ahead:
            m.prefetch(ids[0])
            m.prefetch(ids[1])
        for s in range(steps):
            out = m(ids[s])  # commits s; s+1 stays outstanding
            if ahead and s + 2 < steps:
                m.prefetch(ids[s + 2])  # begun behind the uncommitted s+1, before backward(s)
                assert m.cache.prefetch_depth == 2
            out.backward(torch.from_numpy(grads[s]).cuda())
        m.flush()
        return m.weight().copy()

    assert np.array_equal(train(False), train(True))


def test_prefetch_depth2_limits_and_mismatch():
    """A third outstanding begin is refused; a prepare of ids that match neither
    prefetch runs both prefetched batches first (FIFO), then the ids."""
    num_ids, cap, dim = 64, 4, 8
    idx = fc.IdxMap(np.arange(num_ids), np.arange(num_ids))
    slow, _, ref = fc.init_stores(num_ids, dim, cap / num_ids, init_seed=1, idx_map=idx)
    st = fc.CacheStack(idx, slow, fc.FastTierStore(np.zeros((cap, dim), np.float32)), fc.Transmitter(),
                       reference=ref, log_events=True, engine="async")
    st.prepare(np.array([1, 2]), 0)
    a, b = np.array([3, 4]), np.array([5, 6])
    st.prefetch(a, 1)
    st.prefetch(b, 2)
    with pytest.raises(RuntimeError, match="two prefetched"):
        st.prefetch(np.array([7]), 3)
    p = st.prepare(np.array([1, 7]), 3)  # a, then b, then [1, 7]
    # a filled the two free slots; b evicted the largest unprotected ranks 4, 3; [1, 7]
    # hits 1 and evicts 6 for 7 (identity reorder)
    assert (p.hits, p.misses, p.evictions) == (1, 1, 1)
    assert set(st.state.occupied_ranks().tolist()) == {1, 2, 5, 7}
    # the bypassed prefetches are logged like the prepares they are (events in batch order)
    assert [e.batch_seq for e in st.events] == [0, 1, 2, 3]
    assert set(st.events[2].evicted_ranks.tolist()) == {3, 4}
    # ids equal to the SECOND outstanding prefetch: the first is committed, then the second is the result
    st.prefetch(np.array([8]), 4)
    st.prefetch(np.array([9, 1]), 5)
    p = st.prepare(np.array([9, 1]), 5)
    assert (p.hits, p.misses) == (1, 1)
    assert [e.batch_seq for e in st.events] == [0, 1, 2, 3, 4, 5]
    st.flush()
    torch.cuda.synchronize()
    assert st.first_divergence() is None
    st.state.check_invariants()


def test_prefetch_depth2_error_in_first():
    """Two outstanding, the older one invalid: its commit raises and mutates nothing; the
    newer one (whose index phase ran behind the failed one) then commits exactly as a
    plain prepare would after the error."""
    num_ids, cap, dim = 64, 4, 8
    idx = fc.IdxMap(np.arange(num_ids), np.arange(num_ids))
    slow, _, ref = fc.init_stores(num_ids, dim, cap / num_ids, init_seed=1, idx_map=idx)
    st = fc.CacheStack(idx, slow, fc.FastTierStore(np.zeros((cap, dim), np.float32)), fc.Transmitter(),
                       reference=ref, log_events=True, engine="async")
    orc = oracle.OracleCache(np.arange(num_ids), np.zeros((num_ids, dim), np.float32), cap)
    for ids in ([1, 2], [3, 4, 5]):
        st.prepare(np.array(ids), 0)
        orc.prepare(np.array(ids), 0)
    for bad, err in ((np.array([1, 2, 3, 9, 10]), cm.BatchExceedsCapacity), (np.array([7, 99]), ValueError)):
        good = np.array([6, 3, 7])
        st.prefetch(bad, 1)
        st.prefetch(good, 2)
        with pytest.raises(err):
            st.prepare(bad, 1)
        p = st.prepare(good, 2)
        a = orc.prepare(good, 2)
        assert (p.hits, p.misses, p.evictions) == (a["hits"], a["misses"], a["evictions"])
        assert np.array_equal(p.unique_slots, a["unique_slots"])
        assert np.array_equal(st.state.slot_to_rank, orc.slot_rank)
    st.flush()
    torch.cuda.synchronize()
    assert st.first_divergence() is None
    st.state.check_invariants()


@pytest.mark.parametrize("optimizer,mode,bags", [("sgd", "sum", False), ("adagrad", "mean", True)])
def test_module_prefetch_matches_sequential(optimizer, mode, bags):
    """Training through CachedEmbeddingBag with prefetch() gives bit-identical tables
    (and optimizer state) to training without it; both match the dense oracle."""
    rng = np.random.default_rng(5)
    num_ids, dim, steps, B = 20_000, 32, 12, 3_000
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.1
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(steps, B), p=p / p.sum())]
    w0 = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
    idx = fc.build_reorder(fc.scan_frequencies(trace, num_ids))
    grads = [rng.standard_normal((B // 3 if bags else B, dim)).astype(np.float32) for _ in range(steps)]
    offs = torch.arange(0, B, 3) if bags else None

    def train(prefetch):
        m = CachedEmbeddingBag(num_ids, dim, 0.1, mode=mode, weight=w0, idx_map=idx, optimizer=optimizer, lr=0.05)
        ids = [torch.from_numpy(trace[s]) for s in range(steps)]
        for s in range(steps):
            out = m(ids[s], offs)
            if prefetch and s + 1 < steps:
                m.prefetch(ids[s + 1])
            out.backward(torch.from_numpy(grads[s]).cuda())
        m.flush()
        return m.weight().copy(), (m.optimizer_state().copy() if optimizer == "adagrad" else None)

    w_seq, s_seq = train(False)
    w_pf, s_pf = train(True)
    assert np.array_equal(w_seq, w_pf)
    if s_seq is not None:
        assert np.array_equal(s_seq, s_pf)
    # dense references on the full table, both held to the north star's 1e-5 relative:
    # (1) the oracle restatement (float64 gradients and optimizer arithmetic, rows stored
    #     as float32 after each step) -- deterministic;
    # (2) torch's CPU EmbeddingBag + torch.optim. Its sparse-gradient coalesce reduces
    #     duplicate rows with a thread-parallel sum whose order can change from run to run;
    #     pinned to one thread here so that the reference itself is reproducible.
    dense = w0.copy()
    state = np.zeros_like(w0)
    off_np = offs.numpy() if bags else np.arange(B)
    for s in range(steps):
        grad = oracle.pooled_bag_backward_rows(grads[s], trace[s], off_np, num_ids, None, mode)
        touched = np.unique(trace[s])
        if optimizer == "sgd":
            oracle.sparse_sgd(dense, touched, grad, 0.05)
        else:
            oracle.sparse_adagrad(dense, state, touched, grad, 0.05, 1e-10)
    np.testing.assert_allclose(w_pf, dense, rtol=1e-5, atol=1e-6)
    if s_pf is not None:
        np.testing.assert_allclose(s_pf, state, rtol=1e-5, atol=1e-6)
    nthreads = torch.get_num_threads()
    torch.set_num_threads(1)
    try:
        emb = torch.nn.EmbeddingBag(num_ids, dim, mode=mode, sparse=True)
        emb.weight.data = torch.from_numpy(w0.copy())
        opt = (torch.optim.SGD if optimizer == "sgd" else torch.optim.Adagrad)(emb.parameters(), lr=0.05)
        for s in range(steps):
            o = emb(torch.from_numpy(trace[s]), offs if bags else torch.arange(0, B))
            opt.zero_grad()
            o.backward(torch.from_numpy(grads[s]))
            opt.step()
    finally:
        torch.set_num_threads(nthreads)
    np.testing.assert_allclose(w_pf, emb.weight.detach().numpy(), rtol=1e-5, atol=1e-6)


def test_prefetched_paper_literal_vs_oracle():
    """evict_mode='paper_literal' (needed = max(0, U - C), cache_manager.py:293-296) through
    the pipeline, including the InsufficientFreeSlots error once the tier is full."""
    num_ids, cap, dim = 4_000, 500, 8
    rng = np.random.default_rng(2)
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.1
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(12, 120), p=p / p.sum())]
    rank_of, id_of = oracle.rank_permutation(oracle.frequency_counts(trace, num_ids))
    ref = oracle.init_rows(num_ids, dim, 4)
    orc = oracle.OracleCache(rank_of, ref[id_of].copy(), cap, evict_mode="paper_literal")
    st = fc.CacheStack(fc.IdxMap(rank_of, id_of), fc.SlowTierStore(ref[id_of].copy()),
                       fc.FastTierStore(np.zeros((cap, dim), np.float32)), fc.Transmitter(),
                       evict_mode="paper_literal", log_events=True, engine="async")
    ids = [trace[b] for b in range(trace.shape[0])]
    for b in range(len(ids)):
        try:
            a = orc.prepare(ids[b], b)
        except oracle.OracleInsufficientFreeSlots:
            st.prefetch(ids[b], b)
            with pytest.raises(cm.InsufficientFreeSlots):
                st.prepare(ids[b], b)
            break
        st.prefetch(ids[b], b)
        q = st.prepare(ids[b], b)
        assert (q.hits, q.misses, q.evictions) == (a["hits"], a["misses"], a["evictions"])
        assert np.array_equal(q.unique_slots, a["unique_slots"])
    st.state.check_invariants()
    assert np.array_equal(st.state.slot_to_rank, orc.slot_rank)


def test_stress_shape_adagrad_through_module():
    """configs[4]'s index shape (25.5M rows, 0.5% cache, uniform ids, 65,536 lookups per
    step) trained with Adagrad through CachedEmbeddingBag + prefetch: the flushed table
    and optimizer state equal a dense torch Adagrad (rtol 1e-5); nearly every lookup
    misses, so the state rows ride every admission and write-back."""
    num_ids, dim, steps, B = 25_523_073, 4, 5, 65_536
    rng = np.random.default_rng(8)
    trace = rng.integers(0, num_ids, size=(steps, B))
    w0 = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
    grads = [rng.standard_normal((B, dim)).astype(np.float32) for _ in range(steps)]
    idx = fc.build_reorder(fc.scan_frequencies(trace, num_ids))
    m = CachedEmbeddingBag(num_ids, dim, 0.005, mode="sum", weight=w0, idx_map=idx, optimizer="adagrad", lr=0.1)
    ids = [torch.from_numpy(trace[s]) for s in range(steps)]
    out = m(ids[0])
    for s in range(steps):
        if s + 1 < steps:
            m.prefetch(ids[s + 1])
        out.backward(torch.from_numpy(grads[s]).cuda())
        if s + 1 < steps:
            out = m(ids[s + 1])
    m.flush()
    emb = torch.nn.EmbeddingBag(num_ids, dim, mode="sum", sparse=True)
    emb.weight.data = torch.from_numpy(w0.copy())
    opt = torch.optim.Adagrad(emb.parameters(), lr=0.1, eps=1e-10)
    for s in range(steps):
        o = emb(torch.from_numpy(trace[s]), torch.arange(0, B))
        opt.zero_grad()
        o.backward(torch.from_numpy(grads[s]))
        opt.step()
    touched = np.unique(trace)
    np.testing.assert_allclose(m.weight()[touched], emb.weight.detach().numpy()[touched], rtol=1e-5, atol=1e-6)
    state = opt.state[emb.weight]["sum"].numpy()
    np.testing.assert_allclose(m.optimizer_state()[touched], state[touched], rtol=1e-5, atol=1e-7)
    assert np.array_equal(m.weight()[:1000], np.where(np.isin(np.arange(1000), touched)[:, None],
                                                      m.weight()[:1000], w0[:1000]))


def test_prefetch_device_ids_written_on_main_stream():
    """prefetch() of device ids that the current stream is still producing: the index
    phase (on its own stream) must read them only after they are written. The ids are
    written behind a ~2 ms spin on the main stream; the outcome must equal prefetching
    ids that were complete long before (ready event) and training without prefetch."""
    rng = np.random.default_rng(8)
    num_ids, dim, steps, B = 20_000, 32, 6, 3_000
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.1
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(steps, B), p=p / p.sum())]
    w0 = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
    idx = fc.build_reorder(fc.scan_frequencies(trace, num_ids))
    grads = [torch.from_numpy(rng.standard_normal((B, dim)).astype(np.float32)).cuda() for _ in range(steps)]
    src = torch.from_numpy(trace).cuda()

    def train(kind):
        m = CachedEmbeddingBag(num_ids, dim, 0.1, mode="sum", weight=w0, idx_map=idx, lr=0.05)
        ready = torch.cuda.Event()
        ready.record()
        nxt = None
        for s in range(steps):
            cur = nxt if nxt is not None else src[s].clone()
            out = m(cur)
            nxt = None
            if kind != "none" and s + 1 < steps:
                if kind == "late":  # the next ids are still being written when prefetch is called
                    nxt = torch.full_like(src[s + 1], -7)
                    torch.cuda._sleep(4_000_000)
                    nxt.copy_(src[s + 1])
                    m.prefetch(nxt)
                else:
                    nxt = src[s + 1]
                    m.prefetch(nxt, ready=ready)
            out.backward(grads[s])
        m.flush()
        return m.weight().copy()

    w_none = train("none")
    assert np.array_equal(train("late"), w_none)
    assert np.array_equal(train("ready"), w_none)


def test_prefetch_clean_victims_ship_exact_writebacks():
    """Read-only (forward-only) steps evict clean rows: the write-back engine switches to
    shipping exactly the dirty count (here 0) instead of the whole victim stage, then back
    when training resumes. Tables bit-identical to the synchronous run; the exact D2H
    byte count is reported by fc_profile."""
    rng = np.random.default_rng(33)
    num_ids, dim, B = 20_000, 32, 3_000
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.05
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(24, B), p=p / p.sum())]
    w0 = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
    idx = fc.build_reorder(fc.scan_frequencies(trace[:4], num_ids))
    grads = [rng.standard_normal((B, dim)).astype(np.float32) for _ in range(24)]
    train_steps = set(range(0, 4)) | set(range(16, 24))  # steps 4..15 read only

    def run(prefetch):
        m = CachedEmbeddingBag(num_ids, dim, 0.12, mode="sum", weight=w0, idx_map=idx, lr=0.05)
        ids = [torch.from_numpy(trace[s]) for s in range(24)]
        m.cache.profile(True)
        stats = []
        for s in range(24):
            out = m(ids[s])
            if prefetch and s + 1 < 24:
                m.prefetch(ids[s + 1])
            if s in train_steps:
                out.backward(torch.from_numpy(grads[s]).cuda())
            if s == 15:
                m.cache.drain()
                stats.append(m.cache.profile(True))
        m.flush()
        stats.append(m.cache.profile(False))
        return m.weight().copy(), stats

    w_seq, _ = run(False)
    w_pf, st = run(True)
    assert np.array_equal(w_seq, w_pf)
    # during the read-only phase most write-back jobs shipped nothing: far fewer D2H bytes
    # than one victim stage per job
    ro = st[0]
    assert ro["writeback_rows"] > 0  # the first read-only steps still evict rows trained earlier
    assert ro["writeback_d2h_bytes"] < 0.5 * ro["victim_bytes"], ro


def test_sync_prepare_into_a_prefetched_buffer_gets_its_own_sort():
    """A pipelined prepare leaves the digit histograms of its inverse for that batch's
    backward (keyed by the inverse buffer). A batch committed without a backward, whose
    buffer a synchronous prepare of another batch then reuses, must not lend it its
    histograms: the backward of the new batch is checked row by row."""
    from paper_2208_05321_b200.device import DeviceCache

    num, dim, cap, n, lr = 20_000, 32, 8_000, 6_000, 0.1
    rng = np.random.default_rng(21)
    rows = fc.store.pinned_empty((num, dim))
    rows[...] = rng.uniform(-1, 1, (num, dim)).astype(np.float32)
    dc = DeviceCache(num, cap, dim, device="cuda")
    dc.set_idx_map(np.arange(num))
    dc.attach_slow(rows)
    dc.set_engine("async")
    a = torch.from_numpy(rng.integers(0, num // 2, n).astype(np.int32)).cuda()
    b = torch.from_numpy(rng.integers(num // 2, num, n).astype(np.int32)).cuda()
    dc.prepare_begin(a)
    _, ua, ca, ra, sa, inv_a, _ = dc.prepare_commit()  # committed, never backwarded
    # a synchronous prepare of batch b written into batch a's buffers (fc_prepare directly)
    import ctypes

    from paper_2208_05321_b200 import _lib

    k = min(n, cap)
    base = inv_a.data_ptr() - 4 * (4 * k)  # prepare_commit's buffer: [uids|ucnt|uranks|uslots] (k each) + inverse
    info = _lib.PrepareInfo()
    ptr = lambda off: ctypes.c_void_p(base + 4 * off)  # noqa: E731
    assert _lib.load().fc_prepare(dc.h, ctypes.c_void_p(b.data_ptr()), 4, n, 1, ptr(0), ptr(k), ptr(2 * k),
                                  ptr(3 * k), ptr(4 * k), dc.stream(), ctypes.byref(info)) == 0
    buf = torch.empty(0, dtype=torch.int32, device="cuda").set_(inv_a.untyped_storage())  # the same allocation
    u = int(info.unique)
    ucnt = buf[(base - buf.data_ptr()) // 4 + k:][:u]
    uslots = buf[(base - buf.data_ptr()) // 4 + 3 * k:][:u]
    inverse = inv_a
    reused = True
    grad = torch.from_numpy(rng.standard_normal((n, dim)).astype(np.float32)).cuda()
    before = dc.fast_rows[uslots.long()].double()
    gsum = torch.zeros((u, dim), dtype=torch.float64, device="cuda").index_add_(0, inverse.long(), grad.double())
    dc.backward_update(uslots, inverse, ucnt, None, n, False, None, "sum", grad, "sgd", lr, 1e-10)
    torch.cuda.synchronize()
    after = dc.fast_rows[uslots.long()].double()
    np.testing.assert_allclose(after.cpu().numpy(), (before - lr * gsum).cpu().numpy(), rtol=1e-5, atol=1e-5)
    print("inverse buffer reused:", reused)
