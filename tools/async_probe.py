"""Device-timed training steps of the async engine with/without profiling and the clock sampler."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200.embedding import CachedEmbeddingBag  # noqa: E402

cfg = bench.CONFIGS["criteo_kaggle"]
dev = torch.device("cuda", 0)
samples, rank_of, id_of, cap = bench.make_workload(cfg, 64, device=dev)
D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
N = B * F
rows = fc.store.pinned_empty((cfg["num_ids"], D))
bench.fill_pinned(torch, rows, dev, 1)
mod = CachedEmbeddingBag(cfg["num_ids"], D, cfg["ratio"], idx_map=fc.IdxMap(rank_of, id_of), lr=0.05,
                         slow_rows=rows, engine=sys.argv[1])
dc = mod.cache
gout = bench.make_grad(N, D, dev)
ids_dev = torch.from_numpy(samples).to(dev)
out = torch.empty((N, D), device=dev)
s_next = [0]


def step():
    s = s_next[0]
    s_next[0] += 1
    info, uids, ucnt, uranks, uslots, inverse, _ = dc.prepare(ids_dev[s * B:(s + 1) * B].reshape(-1), s)
    dc.pooled(uslots, inverse, N, out=out)
    dc.backward_update(uslots, inverse, ucnt, None, N, False, None, "sum", gout, "sgd", 0.05, 0.0)


for _ in range(5):
    step()
for prof in (False, True):
    for sampler in (False, True):
        torch.cuda.synchronize()
        dc.profile(prof)
        ctx = bench.ClockSampler(0) if sampler else None
        if ctx:
            ctx.__enter__()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        a.record()
        for _ in range(10):
            step()
        b.record()
        torch.cuda.synchronize()
        w = (time.perf_counter() - t) / 10 * 1e3
        if ctx:
            ctx.__exit__(None, None, None)
        p = dc.profile(False)
        print(f"{sys.argv[1]} profile={prof} sampler={sampler}: {a.elapsed_time(b) / 10:.3f} ms/step gpu, {w:.3f} wall",
              {k: round(v / max(p['calls'], 1), 3) for k, v in p.items() if k in ('prepare_ms', 'transfer_ms')}, flush=True)
