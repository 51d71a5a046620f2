"""Per-step phase timings of the module API right after setup (debug tool)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200.embedding import CachedEmbeddingBag  # noqa: E402

cfg = bench.CONFIGS["small"]
dev = torch.device("cuda", 0)
samples, rank_of, id_of, cap = bench.make_workload(cfg, 40, device=dev)
D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
N = B * F
rows = fc.store.pinned_empty((cfg["num_ids"], D))
bench.fill_pinned(torch, rows, dev, 1)
mod = CachedEmbeddingBag(cfg["num_ids"], D, cfg["ratio"], idx_map=fc.IdxMap(rank_of, id_of), lr=0.05,
                         slow_rows=rows, engine=sys.argv[1] if len(sys.argv) > 1 else "zerocopy")
gout = bench.make_grad(N, D, dev)
ids_host = torch.from_numpy(samples).pin_memory()
for s in range(16):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = mod(ids_host[s * B:(s + 1) * B].reshape(-1))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    out.backward(gout)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"step {s:2d} fwd {(t1 - t0) * 1e3:8.2f} bwd-call {(t2 - t1) * 1e3:8.2f} bwd-sync {(t3 - t2) * 1e3:8.2f} ms",
          flush=True)
