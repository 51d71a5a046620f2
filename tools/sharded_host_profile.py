"""Host time of the row-sharded module's step (forward / prefetch / backward) at world 1
over NCCL, for a bench config at a given per-rank batch (the strong-scaling share), next to
the device step time; then a cProfile of the same loop. Diagnostics for the sharded path's
fixed per-step cost.  usage: sharded_host_profile.py [config] [batch] [steps]"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200.distributed import CudaShard, RowShardedEmbedding, shard_rows_for_rank  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "criteo_kaggle"])
cfg["batch"] = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1, device_id=dev)
D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
N = B * F
nb = 2 * steps + 40
(samples, counts), rank_of, id_of, cap = bench.make_workload(cfg, nb, device=dev, keep_counts=True)
idx = shard_rows_for_rank(counts, 0, 1)
rows = fc.store.pinned_empty((idx.num_ids, D))
bench.fill_pinned(torch, rows, dev, bench.SEED)
shard = CudaShard(idx.num_ids, D, fc.fast_capacity(idx.num_ids, cfg["ratio"]), rows, idx, lr=0.05, device=dev,
                  global_num_ids=cfg["num_ids"])
mod = RowShardedEmbedding(shard, 1, 0, mode="sum", device=dev)
gout = bench.make_grad(N, D, dev)
ids_dev = torch.from_numpy(samples).to(dev)
ready = torch.cuda.Event()
ready.record()
bv = [ids_dev[k * B:(k + 1) * B].reshape(-1) for k in range(nb)]
T = {"forward": 0.0, "prefetch": 0.0, "backward": 0.0}


def loop(k0, k1, timed=False):
    pc = time.perf_counter
    for k in range(k0, k1):
        t0 = pc()
        out = mod(bv[k])
        t1 = pc()
        mod.prefetch(bv[k + 1], ready=ready)
        t2 = pc()
        out.backward(gout)
        t3 = pc()
        if timed:
            T["forward"] += t1 - t0
            T["prefetch"] += t2 - t1
            T["backward"] += t3 - t2


with torch.cuda.stream(torch.cuda.Stream()):
    mod.prefetch(bv[0], ready=ready)
    loop(0, 20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t = time.perf_counter()
    loop(20, 20 + steps, True)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / steps * 1e3
    print(f"config {sys.argv[1:2]} batch {B}: device {e0.elapsed_time(e1) / steps:.3f} ms/step, host wall {wall:.3f} "
          f"ms/step; host per call: " + ", ".join(f"{k} {v / steps * 1e3:.3f} ms" for k, v in T.items()))
    pr = cProfile.Profile()
    pr.enable()
    loop(20 + steps, 20 + 2 * steps)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(30)
mod.flush()
dist.destroy_process_group()
