import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2208_05321_b200 as fc
from paper_2208_05321_b200.embedding import CachedEmbeddingBag

rng = np.random.default_rng(21)
num_ids, dim, steps, B = 6_000, 32, 14, 2_000
p = 1.0 / np.arange(1, num_ids + 1) ** 0.9
trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(steps, B), p=p / p.sum())]
w0 = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
idx = fc.build_reorder(fc.scan_frequencies(trace, num_ids))
grads = [rng.standard_normal((B, dim)).astype(np.float32) for _ in range(steps)]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3

def train(ahead, s_before=False, s_after=False, s_fwd=False):
    m = CachedEmbeddingBag(num_ids, dim, 0.25, mode="sum", weight=w0, idx_map=idx, lr=0.05)
    ids = [torch.from_numpy(trace[s]) for s in range(n)]
    infos = []
    if ahead:
        m.prefetch(ids[0]); m.prefetch(ids[1])
    for s in range(n):
        out = m(ids[s])
        if s_fwd: torch.cuda.synchronize()
        infos.append((m.last_info.unique, m.last_info.hits, m.last_info.misses, m.last_info.evictions))
        if ahead and s + 2 < n:
            m.prefetch(ids[s + 2])
        if s_before: torch.cuda.synchronize()
        out.backward(torch.from_numpy(grads[s]).cuda())
        if s_after: torch.cuda.synchronize()
    m.flush()
    return m.weight().copy(), infos

a, ia = train(False)
for kw in [dict(), dict(s_before=True), dict(s_after=True), dict(s_before=True, s_after=True), dict(s_fwd=True, s_before=True, s_after=True)]:
    b, ib = train(True, **kw)
    d = np.argwhere(a != b)
    print(kw, np.array_equal(a, b), ia == ib, len(d), np.unique(d[:, 0])[:10].tolist(), flush=True)

import oracle
rank_of = idx.rank_of
orc = oracle.OracleCache(rank_of, np.zeros((num_ids, 1), np.float32), fc.fast_capacity(num_ids, 0.25))
orc.warmup(orc.capacity if hasattr(orc, "capacity") else fc.fast_capacity(num_ids, 0.25))
ev = []
for s in range(n):
    a_ = orc.prepare(trace[s], s)
    ev.append((set(a_["evicted"].tolist()), set(a_["admitted"].tolist()) if "admitted" in a_ else set()))
d = np.unique(np.argwhere(a != b)[:, 0])
for rid in d[:12]:
    r = int(rank_of[rid])
    print("id", rid, "rank", r, "in batches", [int(rid in set(trace[s].tolist())) for s in range(n)],
          "evicted by", [s for s in range(n) if r in ev[s][0]], "admitted by", [s for s in range(n) if r in ev[s][1]],
          "rank<cap", r < orc.capacity if hasattr(orc, 'capacity') else None)
print(list(a_.keys()))
