"""Host-path A/B of the module API: the small config's e2e loop (CachedEmbeddingBag, pinned
host ids, two batches in flight) with the package imported from a given directory.
usage: e2e_ab.py PKG_PARENT_DIR [steps]   (FC_LIB_PATH may point both variants at one .so)"""
import os
import sys
import time

sys.path.insert(0, os.path.abspath(sys.argv[1]))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200 import workload  # noqa: E402
from paper_2208_05321_b200.embedding import CachedEmbeddingBag  # noqa: E402

steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
num, dim, B, F = 1_000_000, 128, 1024, 26
tr = workload.gen_zipf(num, 1.05, (steps + 40) * B, F, 1)
idx = fc.build_reorder(fc.scan_frequencies(tr.samples, num))
mod = CachedEmbeddingBag(num, dim, 0.015, mode="sum", idx_map=idx, lr=0.05, warmup=True)
ids = torch.from_numpy(tr.samples.astype(np.int32)).pin_memory()
hb = [ids[k * B:(k + 1) * B].reshape(-1) for k in range(steps + 40)]
gout = torch.randn(B * F, dim, device="cuda")
with torch.cuda.stream(torch.cuda.Stream()):
    mod.prefetch(hb[0])
    for k in range(20):
        mod.prefetch(hb[k + 1])
        mod(hb[k]).backward(gout)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for k in range(20, 20 + steps):
        mod.prefetch(hb[k + 1])
        out = mod(hb[k])
        out.backward(gout)
        _ = mod.last_info.hits
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / steps * 1e3
print(f"{sys.argv[1]}: {ms:.3f} ms/step, {B * F / ms / 1e3:.1f} M lookups/s (module e2e, small config)")
