"""Diagnostics: Adagrad + mean + bags training through CachedEmbeddingBag vs a float64
numpy reference and torch's float32 CPU Adagrad (which one deviates?)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_05321_b200 as fc
from paper_2208_05321_b200.embedding import CachedEmbeddingBag

rng = np.random.default_rng(5)
num_ids, dim, steps, B = 20_000, 32, 12, 3_000
p = 1.0 / np.arange(1, num_ids + 1) ** 1.1
trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(steps, B), p=p / p.sum())]
w0 = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
idx = fc.build_reorder(fc.scan_frequencies(trace, num_ids))
grads = [rng.standard_normal((B // 3, dim)).astype(np.float32) for _ in range(steps)]
offs = torch.arange(0, B, 3)

# float64 reference
w = w0.astype(np.float64).copy(); G = np.zeros_like(w)
for s in range(steps):
    ids = trace[s]; bag = np.arange(B) // 3
    g = np.zeros_like(w)
    np.add.at(g, ids, grads[s][bag].astype(np.float64) / 3.0)
    t = np.unique(ids)
    G[t] += g[t] ** 2
    w[t] -= 0.05 * g[t] / (np.sqrt(G[t]) + 1e-10)

emb = torch.nn.EmbeddingBag(num_ids, dim, mode="mean", sparse=True)
emb.weight.data = torch.from_numpy(w0.copy())
opt = torch.optim.Adagrad(emb.parameters(), lr=0.05)
for s in range(steps):
    o = emb(torch.from_numpy(trace[s]), offs)
    opt.zero_grad(); o.backward(torch.from_numpy(grads[s])); opt.step()
wt = emb.weight.detach().numpy()
print("torch fp32 vs f64: max abs", np.abs(wt - w).max())
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    m = CachedEmbeddingBag(num_ids, dim, 0.1, mode="mean", weight=w0, idx_map=idx, optimizer="adagrad", lr=0.05)
    ids = [torch.from_numpy(trace[s]) for s in range(steps)]
    for s in range(steps):
        out = m(ids[s], offs)
        if s + 1 < steps and rep % 2:
            m.prefetch(ids[s + 1])
        out.backward(torch.from_numpy(grads[s]).cuda())
    m.flush()
    wg = m.weight()
    print(f"rep {rep} ours vs f64: max abs {np.abs(wg - w).max():.3e}; vs torch {np.abs(wg - wt).max():.3e}")
