"""Timeline of the prefetch pipeline on the bench workload (diagnostics).

    python tools/pipeline_timeline.py [--config criteo_kaggle] [--steps 8]

Prints, per step, when (ms) the index phase, the miss staging (transfer stream),
the commit, the pooled forward and the backward ran, from tagged CUDA events
(fc_trace) on every stream, plus host-side waits."""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200.embedding import CachedEmbeddingBag  # noqa: E402

NAMES = {1: "idx0", 2: "idx1", 3: "xfr0", 4: "xfr1", 5: "cmt0", 6: "cmt1", 10: "pool0", 11: "pool1", 12: "bwd1",
         20: "idx.marked", 21: "idx.unique", 22: "idx.info+inverse", 23: "idx.victims", 24: "idx.admit"}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="criteo_kaggle")
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--no-prefetch", action="store_true")
ap.add_argument("--serial-index", action="store_true", help="backward waits for the next index phase")
ap.add_argument("--index-stream", choices=["main", "side"], default="main")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
N = B * F
nb = args.steps + 8
samples, rank_of, id_of, cap = bench.make_workload(cfg, 64, device=dev)
rows = fc.store.pinned_empty((cfg["num_ids"], D))
bench.fill_pinned(torch, rows, dev, bench.SEED)
main = torch.cuda.Stream(dev)
with torch.cuda.stream(main):
    mod = CachedEmbeddingBag(cfg["num_ids"], D, cfg["ratio"], mode="sum", idx_map=fc.IdxMap(rank_of, id_of),
                             optimizer="sgd", lr=bench.LR, slow_rows=rows, warmup=True, engine="async")
    dc = mod.cache
    dc.index_on_main = args.index_stream == "main"
    ids_dev = torch.from_numpy(samples).to(dev)
    out = torch.empty((N, D), device=dev)
    gout = bench.make_grad(N, D, dev)
    b = [ids_dev[s * B:(s + 1) * B].reshape(-1) for s in range(nb)]
    pf = not args.no_prefetch
    host = []

    def step(s):
        t0 = time.perf_counter()
        if pf:
            info, uids, ucnt, uranks, uslots, inv, _ = dc.prepare_commit()
        else:
            info, uids, ucnt, uranks, uslots, inv, _ = dc.prepare(b[s], s)
        t1 = time.perf_counter()
        dc.trace_mark(10)
        dc.pooled(uslots, inv, N, out=out)
        dc.trace_mark(11)
        if pf:
            dc.prepare_begin(b[s + 1], s + 1)
            if args.serial_index:
                torch.cuda.current_stream().wait_stream(dc.index_stream)
        t2 = time.perf_counter()
        dc.backward_update(uslots, inv, ucnt, None, N, False, None, "sum", gout, "sgd", bench.LR, 0.0)
        dc.trace_mark(12)
        host.append((t1 - t0, t2 - t1, time.perf_counter() - t2))

    if pf:
        dc.prepare_begin(b[0], 0)
    for s in range(3):
        step(s)
    torch.cuda.synchronize()
    dc.trace(True)
    dc.profile(True)
    host.clear()
    for s in range(3, 3 + args.steps):
        step(s)
    torch.cuda.synchronize()
    prof = dc.profile(False)
    tags, ms = dc.trace_read()
    dc.trace(False)
    ev = [(NAMES.get(int(t), str(t)), float(m)) for t, m in zip(tags, ms)]
    # print in time order
    for name, m in sorted(ev, key=lambda x: x[1]):
        print(f"{m:9.3f} {name}")
    pools = [m for n, m in ev if n == "pool0"]
    print("step period (pool0 to pool0) ms:", np.round(np.diff(pools), 3).tolist())
    print("priority range", torch.cuda.Stream.priority_range())
    print("profile:", {k: round(v, 3) if isinstance(v, float) else v for k, v in prof.items()})
    print("host ms per step (commit wait, pool+begin launch, bwd launch):",
          [tuple(round(x * 1e3, 3) for x in h) for h in host])
