"""Compare end-to-end step variants on the cached EmbeddingBag (debug tool)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200.embedding import CachedEmbeddingBag  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "small"]
dev = torch.device("cuda", 0)
samples, rank_of, id_of, cap = bench.make_workload(cfg, 40, device=dev)
D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
N = B * F
rows = fc.store.pinned_empty((cfg["num_ids"], D))
bench.fill_pinned(torch, rows, dev, 1)
mod = CachedEmbeddingBag(cfg["num_ids"], D, cfg["ratio"], idx_map=fc.IdxMap(rank_of, id_of), lr=0.05,
                         slow_rows=rows, engine="zerocopy")
gout = bench.make_grad(N, D, dev)
ids_host = torch.from_numpy(samples).pin_memory()
ids_dev = ids_host.to(dev)


def run(name, fn, steps=10, start=0):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for k in range(steps):
        fn(start + k)
    torch.cuda.synchronize()
    print(f"{name:40s} {(time.perf_counter() - t) / steps * 1e3:8.3f} ms/step", flush=True)


def v_backward_host(s):
    out = mod(ids_host[s * B:(s + 1) * B].reshape(-1))
    out.backward(gout)


def v_backward_dev(s):
    out = mod(ids_dev[s * B:(s + 1) * B].reshape(-1))
    out.backward(gout)


def v_loss(s):
    out = mod(ids_host[s * B:(s + 1) * B].reshape(-1))
    loss = (out * gout).sum()
    loss.backward()
    loss.item()


def v_fwd_only(s):
    with torch.no_grad():
        mod(ids_host[s * B:(s + 1) * B].reshape(-1))


def v_clone_grad(s):
    out = mod(ids_host[s * B:(s + 1) * B].reshape(-1))
    out.backward(gout.clone())


for name, fn in (("forward only (no_grad)", v_fwd_only), ("out.backward(gout) host ids", v_backward_host),
                 ("out.backward(gout) device ids", v_backward_dev), ("loss.backward()", v_loss),
                 ("out.backward(gout.clone())", v_clone_grad), ("out.backward(gout) again", v_backward_host)):
    run(name, fn, 8, 3)
