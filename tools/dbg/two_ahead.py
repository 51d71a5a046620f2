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

def train(ahead, nsteps, sync=False, depth2=False):
    m = CachedEmbeddingBag(num_ids, dim, 0.25, mode="sum", weight=w0, idx_map=idx, lr=0.05)
    ids = [torch.from_numpy(trace[s]) for s in range(nsteps)]
    if ahead:
        m.prefetch(ids[0]); m.prefetch(ids[1])
    if depth2:
        m.prefetch(ids[0])
    for s in range(nsteps):
        if depth2 and s + 1 < nsteps:
            m.prefetch(ids[s + 1])
        out = m(ids[s])
        if ahead and s + 2 < nsteps:
            m.prefetch(ids[s + 2])
        if sync:
            torch.cuda.synchronize()
        out.backward(torch.from_numpy(grads[s]).cuda())
    m.flush()
    return m.weight().copy()

for n in range(2, steps + 1):
    a = train(False, n)
    r = [np.array_equal(a, train(True, n)), np.array_equal(a, train(True, n, sync=True)), np.array_equal(a, train(False, n, depth2=True))]
    print(n, r, flush=True)
