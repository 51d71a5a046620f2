"""Where a module step's host time goes: wraps every libfreqcache_b200 entry point with a
perf_counter timer (C time incl. launches and host waits), times forward / prefetch /
backward per call, and reports both next to the device step time. Column-wise or
row-wise module at world 1 over NCCL, or the unsharded CachedEmbeddingBag.
usage: host_breakdown.py {column,row,single} [dim] [batch] [steps]"""
import collections
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200 import _lib  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "column"
cfg = dict(bench.CONFIGS["criteo_kaggle"])
cfg["dim"] = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg["batch"] = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 200

lib = _lib.load()
C = collections.defaultdict(lambda: [0, 0.0])


class Timed:
    def __init__(self, name, fn):
        self.name, self.fn = name, fn

    def __call__(self, *a):
        t = time.perf_counter()
        r = self.fn(*a)
        c = C[self.name]
        c[0] += 1
        c[1] += time.perf_counter() - t
        return r


# wrap the entry points the module path calls (ctypes attributes are created on first access)
for name in ("fc_prepare_begin", "fc_prepare_commit", "fc_prepare", "fc_pooled_forward", "fc_pool", "fc_backward_update",
             "fc_route", "fc_pool_rows", "fc_route_grads", "fc_drain_stream"):
    if hasattr(lib, name):
        setattr(lib, name, Timed(name, getattr(lib, name)))

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
N = B * F
nb = 2 * steps + 40
keep = kind == "row"
w = bench.make_workload(cfg, nb, device=dev, keep_counts=keep)
samples, rank_of, id_of, cap = w
if keep:
    samples, counts = samples
if kind != "single":
    dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1, device_id=dev)
from paper_2208_05321_b200.distributed import (ColumnShardedEmbedding, CudaShard, RowShardedEmbedding,  # noqa: E402
                                               shard_rows_for_rank)
from paper_2208_05321_b200.embedding import CachedEmbeddingBag  # noqa: E402

if kind == "column":
    rows = fc.store.pinned_empty((cfg["num_ids"], D))
    bench.fill_pinned(torch, rows, dev, bench.SEED)
    shard = CudaShard(cfg["num_ids"], D, cap, rows, fc.IdxMap(rank_of, id_of), lr=0.05, device=dev)
    mod = ColumnShardedEmbedding(shard, D, 1, 0, mode="sum", device=dev)
elif kind == "row":
    idx = shard_rows_for_rank(counts, 0, 1)
    rows = fc.store.pinned_empty((idx.num_ids, D))
    bench.fill_pinned(torch, rows, dev, bench.SEED)
    shard = CudaShard(idx.num_ids, D, fc.fast_capacity(idx.num_ids, cfg["ratio"]), rows, idx, lr=0.05, device=dev,
                      global_num_ids=cfg["num_ids"])
    mod = RowShardedEmbedding(shard, 1, 0, mode="sum", device=dev)
else:
    rows = fc.store.pinned_empty((cfg["num_ids"], D))
    bench.fill_pinned(torch, rows, dev, bench.SEED)
    mod = CachedEmbeddingBag(cfg["num_ids"], D, cfg["ratio"], mode="sum", idx_map=fc.IdxMap(rank_of, id_of), lr=0.05,
                             slow_rows=rows, warmup=True)
gout = bench.make_grad(N, D, dev)
ids_host = torch.from_numpy(samples).pin_memory()
hb = [ids_host[k * B:(k + 1) * B].reshape(-1) for k in range(nb)]
T = collections.defaultdict(float)
d2 = kind == "single"


def loop(k0, k1, timed):
    pc = time.perf_counter
    for k in range(k0, k1):
        t0 = pc()
        if d2:
            mod.prefetch(hb[k + 1])
        t1 = pc()
        out = mod(hb[k])
        t2 = pc()
        if not d2:
            mod.prefetch(hb[k + 1])
        t3 = pc()
        out.backward(gout)
        t4 = pc()
        if timed:
            T["prefetch"] += (t1 - t0) + (t3 - t2)
            T["forward"] += t2 - t1
            T["backward"] += t4 - t3


with torch.cuda.stream(torch.cuda.Stream()):
    if d2:
        mod.prefetch(hb[0])
    loop(0, 20, False)
    torch.cuda.synchronize()
    C.clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t = time.perf_counter()
    loop(20, 20 + steps, True)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / steps * 1e3
print(f"{kind} dim {D} batch {B}: wall {wall:.3f} ms/step, device {e0.elapsed_time(e1) / steps:.3f} ms/step")
print("  host per step: " + ", ".join(f"{k} {v / steps * 1e3:.3f} ms" for k, v in T.items()))
for name, (n, s) in sorted(C.items(), key=lambda x: -x[1][1]):
    print(f"  {name:20s} {n / steps:4.1f} calls/step  {s / steps * 1e3:.3f} ms/step  ({s / max(n, 1) * 1e6:.1f} us/call)")
mod.flush()
if dist.is_initialized():
    dist.destroy_process_group()
