"""GPU: the cached EmbeddingBag forward and fused backward+optimizer against torch's
CPU F.embedding_bag / torch.optim (golden vectors) and the oracle's restatement.
Tolerance (north star): 1e-5 relative on fp32 pooled outputs and updated rows."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from conftest import load_golden  # noqa: E402

pytestmark = pytest.mark.gpu

from paper_2208_05321_b200 import FrequencyTable, build_reorder  # noqa: E402
from paper_2208_05321_b200.embedding import CachedEmbeddingBag  # noqa: E402

RTOL, ATOL = 1e-5, 1e-6
CASES = [("sum", False), ("mean", False), ("sum", True)]


@pytest.mark.parametrize("ci", [0, 1, 2])
@pytest.mark.parametrize("mode,use_w", CASES)
def test_pooled_forward_matches_torch(ci, mode, use_w):
    g = load_golden("embedding_bag")
    w, idx, off, psw = (g[f"c{ci}_{k}"] for k in ("w", "idx", "off", "psw"))
    m = CachedEmbeddingBag(w.shape[0], w.shape[1], cache_ratio=1.0, mode=mode, weight=w)
    out = m(torch.from_numpy(idx), torch.from_numpy(off), torch.from_numpy(psw) if use_w else None)
    key = f"c{ci}_{mode}{'_w' if use_w else ''}"
    np.testing.assert_allclose(out.detach().cpu().numpy(), g[key + "_out"], rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("ci", [0, 1, 2])
@pytest.mark.parametrize("mode,use_w", CASES)
@pytest.mark.parametrize("opt", ["sgd", "adagrad"])
def test_backward_optimizer_matches_torch(ci, mode, use_w, opt):
    g = load_golden("embedding_bag")
    w, idx, off, psw, gout = (g[f"c{ci}_{k}"] for k in ("w", "idx", "off", "psw", "gout"))
    m = CachedEmbeddingBag(w.shape[0], w.shape[1], cache_ratio=1.0, mode=mode, weight=w, optimizer=opt, lr=0.05,
                           eps=1e-10)
    go = torch.from_numpy(gout).cuda()
    for _ in range(2):
        out = m(torch.from_numpy(idx), torch.from_numpy(off), torch.from_numpy(psw) if use_w else None)
        out.backward(go)
    m.flush()
    key = f"c{ci}_{mode}{'_w' if use_w else ''}_{opt}2"
    np.testing.assert_allclose(m.weight(), g[key], rtol=RTOL, atol=ATOL)


def test_mean_with_weights_and_empty_bags():
    rng = np.random.default_rng(3)
    w = rng.uniform(-1, 1, (40, 16)).astype(np.float32)
    lens = np.array([0, 3, 1, 0, 5, 2])
    idx = rng.integers(0, 40, lens.sum())
    off = np.concatenate([[0], np.cumsum(lens)[:-1]])
    psw = rng.uniform(0, 1, idx.size).astype(np.float32)
    m = CachedEmbeddingBag(40, 16, cache_ratio=1.0, mode="mean", weight=w)
    out = m(torch.from_numpy(idx), torch.from_numpy(off), torch.from_numpy(psw)).detach().cpu().numpy()
    np.testing.assert_allclose(out, oracle.pooled_bag(w, idx, off, psw, "mean"), rtol=RTOL, atol=ATOL)
    assert np.all(out[0] == 0) and np.all(out[3] == 0)
    # include_last_offset layout
    m2 = CachedEmbeddingBag(40, 16, cache_ratio=1.0, mode="sum", weight=w, include_last_offset=True)
    off2 = np.concatenate([off, [idx.size]])
    out2 = m2(torch.from_numpy(idx), torch.from_numpy(off2.astype(np.int32))).detach().cpu().numpy()
    np.testing.assert_allclose(out2, oracle.pooled_bag(w, idx, off2, None, "sum", True), rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("opt", ["sgd", "adagrad"])
def test_training_through_small_cache_equals_dense(opt):
    """Rows move host<->HBM between steps (2% cache); the trained table must equal
    dense training on the same batches (oracle restatement of torch.optim)."""
    rng = np.random.default_rng(11)
    num, dim, nbags, steps = 20_000, 32, 256, 12
    p = 1.0 / np.arange(1, num + 1) ** 1.1
    perm = rng.permutation(num)
    w0 = rng.uniform(-0.1, 0.1, (num, dim)).astype(np.float32)
    trace = [perm[rng.choice(num, size=nbags * 3, p=p / p.sum())] for _ in range(steps)]
    counts = np.bincount(np.concatenate(trace), minlength=num)
    idx_map = build_reorder(FrequencyTable(counts=counts, num_ids=num))
    m = CachedEmbeddingBag(num, dim, cache_ratio=0.05, mode="mean", weight=w0, idx_map=idx_map, optimizer=opt,
                           lr=0.1)
    dense = w0.copy()
    state = np.zeros_like(w0)
    off = np.arange(0, nbags * 3, 3)
    moved = np.zeros(2, np.int64)  # misses, evictions over the run
    for s in range(steps):
        ids = trace[s]
        gout = rng.normal(0, 1, (nbags, dim)).astype(np.float32)
        out = m(torch.from_numpy(ids), torch.from_numpy(off))
        moved += (m.last_info.misses, m.last_info.evictions)
        np.testing.assert_allclose(out.detach().cpu().numpy(), oracle.pooled_bag(dense, ids, off, None, "mean"),
                                   rtol=RTOL, atol=ATOL)
        out.backward(torch.from_numpy(gout).cuda())
        grad = oracle.pooled_bag_backward_rows(gout, ids, off, num, None, "mean")
        touched = np.unique(ids)
        if opt == "sgd":
            oracle.sparse_sgd(dense, touched, grad, 0.1)
        else:
            oracle.sparse_adagrad(dense, state, touched, grad, 0.1, 1e-10)
    assert moved[0] > 0 and moved[1] > 0, moved  # rows really crossed the host link both ways
    m.flush()
    np.testing.assert_allclose(m.weight(), dense, rtol=RTOL, atol=ATOL)
    if opt == "adagrad":
        np.testing.assert_allclose(m.optimizer_state(), state, rtol=RTOL, atol=ATOL)


def test_hot_row_long_segment():
    """One id repeated far beyond one reduction part (exercises the multi-part combine)."""
    num, dim = 1000, 64
    w = np.random.default_rng(0).uniform(-1, 1, (num, dim)).astype(np.float32)
    ids = np.concatenate([np.full(5000, 7), np.arange(100)])
    np.random.default_rng(1).shuffle(ids)
    m = CachedEmbeddingBag(num, dim, cache_ratio=0.2, mode="sum", weight=w, lr=0.001)
    out = m(torch.from_numpy(ids))
    gout = np.random.default_rng(2).normal(0, 1, (ids.size, dim)).astype(np.float32)
    out.backward(torch.from_numpy(gout).cuda())
    m.flush()
    grad = oracle.pooled_bag_backward_rows(gout, ids, np.arange(ids.size), num)
    want = w.copy()
    oracle.sparse_sgd(want, np.unique(ids), grad, 0.001)
    np.testing.assert_allclose(m.weight(), want, rtol=1e-5, atol=2e-6)


@pytest.mark.parametrize("num,sizes,prefetch", [(3_000, [500, 4_000, 120, 4_000, 9_000, 37, 9_000], False),
                                                (200, [4_000, 120, 4_000, 500, 9_000, 300, 2_000, 9_000], False),
                                                (200, [4_000, 120, 4_000, 500, 9_000, 300, 2_000, 9_000], True)])
def test_backward_sequence_of_batch_sizes_reuses_sort_state(num, sizes, prefetch):
    """Back-to-back fused backwards of growing and shrinking batches (the fix-up clears the
    next sort's state instead of a memset, DESIGN 4b) with a scatter_update in between,
    against dense SGD: every step within 1e-5. The second case draws from 200 ids, so every
    batch has duplicates (the radix-grouped path, never the all-distinct direct one) and the
    sort state's address moves with n on a scratch that does not grow."""
    dim, lr = 16, 0.05
    rng = np.random.default_rng(11)
    w = rng.uniform(-0.1, 0.1, (num, dim)).astype(np.float32)
    m = CachedEmbeddingBag(num, dim, cache_ratio=1.0, mode="sum", weight=w, lr=lr)
    dense = w.astype(np.float64)
    batches = [torch.from_numpy(rng.integers(0, num, n)) for n in sizes]
    if prefetch:  # pipelined: the index phase makes the sort histograms, sizes still change
        m.prefetch(batches[0])
    for s, n in enumerate(sizes):
        ids = batches[s].numpy()
        gout = rng.standard_normal((n, dim)).astype(np.float32)
        out = m(batches[s])
        if prefetch and s + 1 < len(sizes) and s != 3:
            m.prefetch(batches[s + 1])
        np.testing.assert_allclose(out.detach().cpu().numpy(), dense[ids], rtol=RTOL, atol=ATOL)
        out.backward(torch.from_numpy(gout).cuda())
        np.add.at(dense, ids, -lr * gout.astype(np.float64))
        if s == 3:  # another sort on the same scratch leaves its state behind
            st = m.cache
            info, uids, ucnt, uranks, uslots, inverse, _ = st.prepare(torch.from_numpy(ids[:50]).cuda())
            deltas = torch.zeros((50, dim), dtype=torch.float32, device="cuda")
            st.scatter_update(uslots, inverse, ucnt, deltas)
    m.flush()
    np.testing.assert_allclose(m.weight(), dense, rtol=RTOL, atol=ATOL)
