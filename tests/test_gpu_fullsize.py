"""Parity at BASELINE.json's full index sizes (GPU): the real num_ids, capacities and
batch shapes of configs[1], [2] and [4], with a narrow row width so the numpy oracle
finishes in seconds (the index work — dedup, lookups, victim choice, slot assignment,
write-back selection — does not depend on the width; the row kernels are covered at
width 128 elsewhere). Runs through the prefetch pipeline with the simulator's update
queued behind each prefetch. Bit-exact per batch (unique ids/ranks/counts/slots,
hits/misses/evictions, evicted and admitted lists) and at the end (slot tables, dirty
bits, post-flush slow tier). Reference: cache_manager.py:234-415, simulator.py:416-461."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200 import workload  # noqa: E402

CASES = {
    # configs[1]: Criteo-Kaggle shape
    "criteo_kaggle": dict(num_ids=33_762_577, ratio=0.015, alpha=1.05, batch=16384, features=26, batches=6),
    # configs[2]: Avazu shape, 5% cache, batch 65,536 x 22, cold start (eviction-heavy warm-up)
    "avazu": dict(num_ids=9_445_823, ratio=0.05, alpha=1.05, batch=65536, features=22, batches=4, cold=True),
    # configs[4] per-GPU share: uniform ids, 0.5% cache, 65,536 lookups per step
    "stress": dict(num_ids=25_523_073, ratio=0.005, alpha=None, batch=65536, features=1, batches=6),
    # configs[3]: Criteo-1TB shape (26 tables capped at 40M, 204,184,588 rows), 1.5% cache; a
    # column-sharded rank prepares the GLOBAL batch of 8 ranks (8 x 16,384 x 26 = 3.4M ids)
    "criteo_1tb_colshard8": dict(num_ids=204_184_588, ratio=0.015, alpha=1.05, batch=8 * 16384, features=26,
                                 batches=3),
}
DIM = 4


@pytest.mark.parametrize("name", list(CASES))
def test_fullsize_parity(name):
    c = CASES[name]
    n_ids, nb = c["num_ids"], c["batches"]
    if c["alpha"] is None:
        tr = workload.gen_uniform(n_ids, nb * c["batch"], c["features"], 11)
    else:
        tr = workload.gen_zipf(n_ids, c["alpha"], nb * c["batch"], c["features"], 11, device="cuda")
    ids = [tr.samples[b * c["batch"]:(b + 1) * c["batch"]].reshape(-1) for b in range(nb)]
    freq, idx = fc.build_reorder_device(tr.samples, n_ids)
    assert np.array_equal(freq.counts, oracle.frequency_counts(tr.samples, n_ids))
    if n_ids < 100_000_000:  # the host lexsort of 204M keys alone takes minutes; reorder parity is
        assert np.array_equal(idx.rank_of, oracle.rank_permutation(freq.counts)[0])  # covered elsewhere
    cap = fc.fast_capacity(n_ids, c["ratio"])
    rng = np.random.default_rng(3)
    slow0 = rng.standard_normal((n_ids, DIM), dtype=np.float32)
    orc = oracle.OracleCache(idx.rank_of, slow0.copy(), cap)
    st = fc.CacheStack(idx, fc.SlowTierStore(slow0.copy()), fc.FastTierStore(np.zeros((cap, DIM), np.float32)),
                       fc.Transmitter(), log_events=True, engine="async")
    if not c.get("cold"):
        orc.warmup(cap)
        st.warmup(cap)
    colw = oracle.column_weights(DIM, 5)
    q = st.prepare(ids[0], 0)
    for b in range(nb):
        a = orc.prepare(ids[b], b)
        for k in ("unique_ids", "unique_ranks", "unique_counts", "unique_slots"):
            assert np.array_equal(getattr(q, k), a[k]), (name, b, k)
        assert (q.hits, q.misses, q.evictions) == (a["hits"], a["misses"], a["evictions"]), (name, b)
        assert np.array_equal(st.events[-1].evicted_ranks, a["evicted"]), (name, b)
        assert np.array_equal(st.events[-1].admitted_ranks, a["admitted"]), (name, b)
        if b + 1 < nb:
            st.prefetch(ids[b + 1], b + 1)
        g = oracle.row_scalars(a["unique_ids"], a["unique_counts"], b, 5)
        orc.apply_unique_update(a, g[:, None] * colw[None, :])
        st.apply_synthetic_update(q, b, 5, colw)
        if b + 1 < nb:
            q = st.prepare(ids[b + 1], b + 1)
    assert st.flush().rows == orc.flush()["rows"]
    torch.cuda.synchronize()
    assert np.array_equal(st.state.slot_to_rank, orc.slot_rank)
    assert np.array_equal(st.state.dirty, orc.dirty)
    assert np.array_equal(st.slow.rows, orc.slow)  # bitwise, the whole 33.8M-row slow tier


# ---------------------------------------------------------------------------- width 128
# The row kernels at BASELINE's real widths and sizes, through the training module with
# the depth-2 prefetch pipeline and the async write-back engine: pooled forward
# (k_pool1), fused backward + SGD / Adagrad (grouping of 426k-1.7M occurrences), miss
# staging (TMA), write-back staging + host scatter, flush. The oracle keeps a float64
# mirror of the touched rows only (the untouched ones are checked unchanged on a sample).
ROWCASES = {
    # configs[1] at width 128: 33.8M x 128 fp32 (17.3 GB pinned slow tier), sum, SGD
    "criteo_kaggle_d128": dict(num_ids=33_762_577, dim=128, ratio=0.015, alpha=1.05, batch=16384, features=26,
                               steps=4, optimizer="sgd", mode="sum", psw=False),
    # configs[2] at width 64: mean pooling with per-sample weights, 5% cache, cold start
    "avazu_d64": dict(num_ids=9_445_823, dim=64, ratio=0.05, alpha=1.05, batch=65536, features=22, steps=3,
                      optimizer="sgd", mode="mean", psw=True, cold=True),
    # configs[4] per-GPU share at width 128: uniform ids, 0.5% cache, Adagrad state cached with the rows
    "stress_d128": dict(num_ids=25_523_073, dim=128, ratio=0.005, alpha=None, batch=65536, features=1, steps=4,
                        optimizer="adagrad", mode="sum", psw=False),
}


@pytest.mark.parametrize("name", list(ROWCASES))
def test_fullsize_rows_training(name):
    from paper_2208_05321_b200.embedding import CachedEmbeddingBag

    c = ROWCASES[name]
    n_ids, D, S, B, F = c["num_ids"], c["dim"], c["steps"], c["batch"], c["features"]
    # the frequency reorder scans a longer trace than the steps trained (as a real run's
    # would), so the warmed cache does not already hold every id of the trained batches
    if c["alpha"] is None:
        tr = workload.gen_uniform(n_ids, 8 * S * B, F, 12)
    else:
        tr = workload.gen_zipf(n_ids, c["alpha"], 8 * S * B, F, 12, device="cuda")
    _, idx = fc.build_reorder_device(tr.samples, n_ids)
    rows = fc.store.pinned_empty((n_ids, D))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    tt = torch.from_numpy(rows)
    for lo in range(0, n_ids, 1 << 21):  # seeded rows, generated on the GPU into pinned memory
        hi = min(lo + (1 << 21), n_ids)
        tt[lo:hi].copy_(torch.rand((hi - lo, D), generator=gen, device="cuda") - 0.5)
    torch.cuda.synchronize()
    ids = [tr.samples[s * B:(s + 1) * B].reshape(-1).astype(np.int64) for s in range(S)]
    touched = np.unique(np.concatenate(ids))
    mirror = rows[idx.rank_of[touched]].astype(np.float64)  # float64 oracle rows of the touched ids
    state = np.zeros_like(mirror)
    sample = np.random.default_rng(0).choice(n_ids, 4096, replace=False)
    sample = sample[~np.isin(sample, touched)]
    untouched0 = rows[idx.rank_of[sample]].copy()
    m = CachedEmbeddingBag(n_ids, D, c["ratio"], mode=c["mode"], idx_map=idx, optimizer=c["optimizer"], lr=0.05,
                           slow_rows=rows, warmup=not c.get("cold"))
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    n = B * F
    psw = torch.rand(n, generator=g, device="cuda") if c["psw"] else None
    psw_np = psw.cpu().numpy().astype(np.float64) if c["psw"] else None
    dev_ids = [torch.from_numpy(x).cuda() for x in ids]
    m.prefetch(dev_ids[0])
    moved = np.zeros(2, np.int64)
    for s in range(S):
        if s + 1 < S:
            m.prefetch(dev_ids[s + 1])  # depth 2
        out = m(dev_ids[s], None, psw)
        moved += (m.last_info.misses, m.last_info.evictions)
        pos = np.searchsorted(touched, ids[s])
        coef = psw_np if psw_np is not None else np.ones(n)
        want = mirror[pos] * coef[:, None]  # bag size 1: mean == sum
        np.testing.assert_allclose(out.detach().cpu().numpy(), want, rtol=1e-5, atol=1e-6, err_msg=f"{name} fwd {s}")
        gout = torch.randn((n, D), generator=g, device="cuda") * 0.01
        out.backward(gout)
        gsum = np.zeros_like(mirror)
        np.add.at(gsum, pos, gout.cpu().numpy().astype(np.float64) * coef[:, None])
        u = np.unique(pos)
        if c["optimizer"] == "sgd":
            mirror[u] -= 0.05 * gsum[u]
        else:
            state[u] += gsum[u] ** 2
            mirror[u] -= 0.05 * gsum[u] / (np.sqrt(state[u]) + 1e-10)
        mirror[u] = mirror[u].astype(np.float32)
        state[u] = state[u].astype(np.float32)
    assert moved[0] > 0 and moved[1] > 0, moved
    m.flush()
    torch.cuda.synchronize()
    np.testing.assert_allclose(m.slow_rows[idx.rank_of[touched]], mirror, rtol=1e-5, atol=1e-6)
    if c["optimizer"] == "adagrad":
        np.testing.assert_allclose(m.slow_state[idx.rank_of[touched]], state, rtol=1e-5, atol=1e-7)
    assert np.array_equal(m.slow_rows[idx.rank_of[sample]], untouched0)
