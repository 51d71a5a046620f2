"""cProfile of the module-path (e2e) training loop for a bench config: where the host time of
forward / prefetch / backward goes (diagnostics; the small config is host-bound)."""
import cProfile
import os
import pstats
import sys

import torch

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200.embedding import CachedEmbeddingBag  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "small"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
N = B * F
nb = steps + 20
samples, rank_of, id_of, cap = bench.make_workload(cfg, nb, device=dev)
rows = fc.store.pinned_empty((cfg["num_ids"], D))
bench.fill_pinned(torch, rows, dev, bench.SEED)
mod = CachedEmbeddingBag(cfg["num_ids"], D, cfg["ratio"], mode=cfg.get("mode", "sum"), idx_map=fc.IdxMap(rank_of, id_of),
                         optimizer=cfg.get("optimizer", "sgd"), lr=0.05, slow_rows=rows, warmup=True)
gout = bench.make_grad(N, D, dev)
ids_host = torch.from_numpy(samples).pin_memory()
hb = [ids_host[k * B:(k + 1) * B].reshape(-1) for k in range(nb)]


def loop(k0, k1):
    for k in range(k0, k1):
        mod.prefetch(hb[k + 1])
        out = mod(hb[k])
        out.backward(gout)
        _ = mod.last_info.hits
    torch.cuda.synchronize()


mod.prefetch(hb[0])  # depth 2: batch k+1 is begun before batch k's forward commits k
loop(0, 10)
pr = cProfile.Profile()
import time  # noqa: E402
t = time.perf_counter()
pr.enable()
loop(10, 10 + steps)
pr.disable()
el = time.perf_counter() - t
print(f"{steps} steps in {el * 1e3:.1f} ms = {el / steps * 1e3:.3f} ms/step (profiled)")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
