"""GPU: bounded staging buffers and the memory report.

The write-back and admission stages start at buffer_bytes worth of rows (like the
reference's 64 MiB TransferBuffer, transmitter.py:19,75-94) and grow only when a batch
needs more. FC_STAGE_ROWS forces a tiny start so every overflow path runs: the sync
prepare's read-back-and-grow before its eviction kernel, the pipeline commit's growth of
the write-back stages, and the admission rows past the stage that the commit copies from
their newest copy. Cache decisions and the post-flush slow tier must stay bit-exact with
the oracle. The device memory report (fc_memory_bytes, CacheStack.device_memory; the
reference's own memory_report, cache_manager.py:553-562, keeps its formula because the
simulator's RunMetrics embed it) must account for the device memory the cache really
takes (cudaMemGetInfo delta)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_2208_05321_b200 as fc  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("depth", [0, 1, 2])
def test_tiny_stages_grow_and_stay_exact(depth, monkeypatch):
    monkeypatch.setenv("FC_STAGE_ROWS", "48")
    num_ids, cap, dim, nb, bsz = 20_000, 1_500, 32, 24, 1_200
    rng = np.random.default_rng(77)
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.05
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(nb, bsz), p=p / p.sum())]
    rank_of, id_of = oracle.rank_permutation(oracle.frequency_counts(trace, num_ids))
    ref = oracle.init_rows(num_ids, dim, 4)
    orc = oracle.OracleCache(rank_of, ref[id_of].copy(), cap)
    st = fc.CacheStack(fc.IdxMap(rank_of, id_of), fc.SlowTierStore(ref[id_of].copy()),
                       fc.FastTierStore(np.zeros((cap, dim), np.float32)), fc.Transmitter(), log_events=True,
                       engine="async")
    orc.warmup(cap // 3)
    st.warmup(cap // 3)
    colw = oracle.column_weights(dim, 5)
    ids = [trace[b] for b in range(nb)]
    if depth == 2:
        st.prefetch(ids[0], 0)
    big_miss = 0
    q = st.prepare(ids[0], 0) if depth != 2 else None
    for b in range(nb):
        if depth == 2:
            if b + 1 < nb:
                st.prefetch(ids[b + 1], b + 1)
            q = st.prepare(ids[b], b)
        a = orc.prepare(ids[b], b)
        assert np.array_equal(q.unique_slots, a["unique_slots"]), b
        assert (q.hits, q.misses, q.evictions) == (a["hits"], a["misses"], a["evictions"]), b
        assert np.array_equal(st.events[-1].evicted_ranks, a["evicted"]), b
        big_miss = max(big_miss, a["misses"])
        if depth == 1 and b + 1 < nb:
            st.prefetch(ids[b + 1], b + 1)
        gs = oracle.row_scalars(a["unique_ids"], a["unique_counts"], b, 5)
        orc.apply_unique_update(a, gs[:, None] * colw[None, :])
        st.apply_synthetic_update(q, b, 5, colw)
        if depth != 2 and b + 1 < nb:
            q = st.prepare(ids[b + 1], b + 1)
    assert big_miss > 48  # the overflow paths ran
    assert st.flush().rows == orc.flush()["rows"]
    torch.cuda.synchronize()
    assert np.array_equal(st.state.slot_to_rank, orc.slot_rank)
    assert np.array_equal(st.slow.rows, orc.slow)
    m = st.device_memory()
    assert m["wb_stage_rows"] > 48
    if depth:
        assert m["admission_stage_rows"] > 48


def _lib_bytes(fn):
    """Device bytes `fn` allocates outside torch's caching allocator (cudaMemGetInfo delta
    minus torch's reserved delta)."""
    import gc

    gc.collect()  # caches of earlier tests release their device memory first
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    f0, _ = torch.cuda.mem_get_info()
    r0 = torch.cuda.memory_reserved()
    out = fn()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    f1, _ = torch.cuda.mem_get_info()
    r1 = torch.cuda.memory_reserved()
    return (f0 - f1) - (r1 - r0), out


def test_memory_report_matches_device_allocations():
    from paper_2208_05321_b200.embedding import CachedEmbeddingBag

    num_ids, dim = 4_000_000, 128
    rng = np.random.default_rng(5)
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.05
    batches = [torch.from_numpy(rng.choice(num_ids, size=60_000, p=p / p.sum()).astype(np.int32))
               for _ in range(6)]

    def build_and_run():
        m = CachedEmbeddingBag(num_ids, dim, 0.015, mode="sum", lr=0.1)
        m.prefetch(batches[0])
        for b in range(5):
            out = m(batches[b])
            m.prefetch(batches[b + 1])
            out.backward(torch.ones_like(out))
        return m

    m0 = build_and_run()  # loads every kernel the run uses (lazy module loading takes device memory once)
    m0.flush()
    del m0
    used, m = _lib_bytes(build_and_run)
    rep = m.cache.memory()
    total = rep["device_total_bytes"]
    fast = rep["fast_rows_bytes"]
    print(f"cudaMemGetInfo delta (lib) {used / 2**20:.1f} MiB, reported {total / 2**20:.1f} MiB, "
          f"fast tier {fast / 2**20:.1f} MiB, staging {rep['staging_bytes'] / 2**20:.1f} MiB, {rep}")
    # what the report cannot see: the driver's GPU page tables for the pinned, device-mapped
    # host memory the cache maps (slow tier + write-back staging), 8 B per 4 KiB page,
    # allocated in 2 MiB pages
    mapped = m.slow_rows.nbytes + rep["pinned_staging_bytes"]
    page_tables = (mapped // 4096 * 8 + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    assert total <= used <= total + page_tables + 0.01 * used, (used, total, page_tables)
    # staging bounded by the 64 MiB buffer budget per stage, not by capacity
    row = 4 * dim
    assert rep["wb_stage_rows"] <= max(64 * 2**20 // row, 1024)
    assert rep["staging_bytes"] <= 6 * 64 * 2**20 + 6 * 4 * rep["wb_stage_rows"]  # 4 write-back + 2 admission


@pytest.mark.parametrize("gbps", ["12", "40"])
def test_paced_staging_stays_exact(gbps, monkeypatch):
    """FC_XFER_GBPS paces the TMA miss staging (%globaltimer-spaced bulk copies); the
    decisions and the post-flush table are unchanged."""
    monkeypatch.setenv("FC_XFER_GBPS", gbps)
    num_ids, cap, dim, nb, bsz = 30_000, 2_000, 32, 10, 2_500
    rng = np.random.default_rng(9)
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.05
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(nb, bsz), p=p / p.sum())]
    rank_of, id_of = oracle.rank_permutation(oracle.frequency_counts(trace, num_ids))
    ref = oracle.init_rows(num_ids, dim, 2)
    orc = oracle.OracleCache(rank_of, ref[id_of].copy(), cap)
    st = fc.CacheStack(fc.IdxMap(rank_of, id_of), fc.SlowTierStore(ref[id_of].copy()),
                       fc.FastTierStore(np.zeros((cap, dim), np.float32)), fc.Transmitter(), engine="async")
    orc.warmup(cap)
    st.warmup(cap)
    colw = oracle.column_weights(dim, 3)
    q = st.prepare(trace[0], 0)
    for b in range(nb):
        a = orc.prepare(trace[b], b)
        assert np.array_equal(q.unique_slots, a["unique_slots"]), b
        if b + 1 < nb:
            st.prefetch(trace[b + 1], b + 1)
        gs = oracle.row_scalars(a["unique_ids"], a["unique_counts"], b, 3)
        orc.apply_unique_update(a, gs[:, None] * colw[None, :])
        st.apply_synthetic_update(q, b, 3, colw)
        if b + 1 < nb:
            q = st.prepare(trace[b + 1], b + 1)
    st.flush()
    orc.flush()
    torch.cuda.synchronize()
    assert np.array_equal(st.slow.rows, orc.slow)
