"""Which API call stalls in the module-path (e2e) loop? Per-step host time of
forward / prefetch / backward for a bench config (diagnostics)."""
import os, sys, time
import numpy as np
import torch
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2208_05321_b200 as fc
from paper_2208_05321_b200.embedding import CachedEmbeddingBag

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "avazu"]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
N = B * F
samples, rank_of, id_of, cap = bench.make_workload(cfg, 64, device=dev)
rows = fc.store.pinned_empty((cfg["num_ids"], D))
bench.fill_pinned(torch, rows, dev, bench.SEED)
with torch.cuda.stream(torch.cuda.Stream()):
    mod = CachedEmbeddingBag(cfg["num_ids"], D, cfg["ratio"], mode=cfg.get("mode", "sum"), idx_map=fc.IdxMap(rank_of, id_of),
                             optimizer=cfg.get("optimizer", "sgd"), lr=0.05, slow_rows=rows, warmup=True)
    psw = torch.rand(N, device=dev) if cfg.get("psw") else None
    gout = bench.make_grad(N, D, dev)
    ids_host = torch.from_numpy(samples).pin_memory()
    hb = [ids_host[k * B:(k + 1) * B].reshape(-1) for k in range(60)]
    for k in range(5):
        mod(hb[k], None, psw).backward(gout)
    torch.cuda.synchronize()
    rec = []
    out = mod(hb[5], None, psw)
    for k in range(5, 55):
        t0 = time.perf_counter()
        mod.prefetch(hb[k + 1])
        t1 = time.perf_counter()
        out.backward(gout)
        t2 = time.perf_counter()
        out = mod(hb[k + 1], None, psw)
        t3 = time.perf_counter()
        rec.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3))
    torch.cuda.synchronize()
    r = np.array(rec)
    print("median prefetch/backward/forward ms:", np.median(r, 0).round(3), " max:", r.max(0).round(2))
    for i, x in enumerate(rec):
        if max(x) > 5:
            print("step", i, [round(v, 2) for v in x])
