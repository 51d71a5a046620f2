import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2208_05321_b200 as fc
from paper_2208_05321_b200.embedding import CachedEmbeddingBag

rng = np.random.default_rng(21)
num_ids, dim, steps, B = 6_000, 32, 3, 2_000
p = 1.0 / np.arange(1, num_ids + 1) ** 0.9
trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(steps, B), p=p / p.sum())]
w0 = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
idx = fc.build_reorder(fc.scan_frequencies(trace, num_ids))
grads = [rng.standard_normal((B, dim)).astype(np.float32) for _ in range(steps)]

def train(ahead, ring=True, dev_ids=False, late_bwd=False):
    m = CachedEmbeddingBag(num_ids, dim, 0.25, mode="sum", weight=w0, idx_map=idx, lr=0.05)
    m.cache.prefetch_ring = ring
    ids = [torch.from_numpy(trace[s]) for s in range(steps)]
    if dev_ids:
        ids = [i.cuda() for i in ids]
    infos = []
    if ahead:
        m.prefetch(ids[0]); m.prefetch(ids[1])
    for s in range(steps):
        out = m(ids[s])
        infos.append((m.last_info.unique, m.last_info.hits, m.last_info.misses, m.last_info.evictions))
        if ahead and s + 2 < steps:
            m.prefetch(ids[s + 2])
        torch.cuda.synchronize()
        out.backward(torch.from_numpy(grads[s]).cuda())
        torch.cuda.synchronize()
    m.flush()
    return m.weight().copy(), infos

a, ia = train(False)
for kw in [dict(), dict(ring=False), dict(dev_ids=True)]:
    b, ib = train(True, **kw)
    print(kw, np.array_equal(a, b), ia == ib, ia, ib, np.argwhere(a != b)[:5].tolist())
