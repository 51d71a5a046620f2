"""Where does the end-to-end (public API) step spend its time? CUDA events around
each phase of CachedEmbeddingBag forward + loss + backward on the cfg2 workload.

    python tools/e2e_probe.py [--config small]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200.embedding import CachedEmbeddingBag  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="criteo_kaggle")
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda", 0)
samples, rank_of, id_of, cap = bench.make_workload(cfg, 30, device=dev)
D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
N = B * F
rows = fc.store.pinned_empty((cfg["num_ids"], D))
bench.fill_pinned(torch, rows, dev, 1)
mod = CachedEmbeddingBag(cfg["num_ids"], D, cfg["ratio"], idx_map=fc.IdxMap(rank_of, id_of), lr=0.05,
                         slow_rows=rows)
gout = bench.make_grad(N, D, dev)
ids_host = torch.from_numpy(samples).pin_memory()
names = ["h2d", "forward", "loss", "backward", "item"]
tot = {k: 0.0 for k in names}
wall = {k: 0.0 for k in names}
for s in range(args.steps + 3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    ev[0].record()
    ids = ids_host[s * B:(s + 1) * B].reshape(-1).to(dev, non_blocking=True)
    ev[1].record(); t.append(time.perf_counter())
    out = mod(ids)
    ev[2].record(); t.append(time.perf_counter())
    loss = (out * gout).sum()
    ev[3].record(); t.append(time.perf_counter())
    loss.backward()
    ev[4].record(); t.append(time.perf_counter())
    _ = loss.item()
    ev[5].record(); t.append(time.perf_counter())
    torch.cuda.synchronize()
    if s >= 3:
        for i, k in enumerate(names):
            tot[k] += ev[i].elapsed_time(ev[i + 1]) / args.steps
            wall[k] += (t[i + 1] - t[i]) * 1e3 / args.steps
print("gpu ms:", {k: round(v, 3) for k, v in tot.items()}, "sum", round(sum(tot.values()), 3))
print("host ms:", {k: round(v, 3) for k, v in wall.items()}, "sum", round(sum(wall.values()), 3))
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    for s in range(3):
        ids = ids_host[s * B:(s + 1) * B].reshape(-1).to(dev, non_blocking=True)
        out = mod(ids)
        loss = (out * gout).sum()
        loss.backward()
        loss.item()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12))
