"""Isolated fused backward (grouping + reduction + optimizer step) at a bench config's shape.

Usage: python tools/bwd_bench.py [--config criteo_kaggle] [--optim sgd|adagrad] [--steps 20]

Builds real batches of the config's id stream (the reference generator, seed 1), dedups them
with torch.unique (the same ascending order and inverse prepare produces), places the unique
rows at random distinct slots of a cache of the config's capacity, and times
DeviceCache.backward_update alone with CUDA events. Algorithmic bytes per call:
N*(4D + 4 order + 4 key) + U*8D (row read-modify-write) [+ U*8D Adagrad state].
Also checks the updated rows against a float64 torch reference (rtol 1e-5)."""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2208_05321_b200 import workload  # noqa: E402
from paper_2208_05321_b200.device import DeviceCache  # noqa: E402
from paper_2208_05321_b200.store import fast_capacity  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="criteo_kaggle")
    ap.add_argument("--optim", default="sgd")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--batches", type=int, default=4)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    D, cap = cfg["dim"], fast_capacity(cfg["num_ids"], cfg["ratio"])
    if cfg["alpha"] is None:
        tr = workload.gen_uniform(cfg["num_ids"], a.batches * cfg["batch"], cfg["features"], bench.SEED)
    else:
        tr = workload.gen_zipf(cfg["num_ids"], cfg["alpha"], a.batches * cfg["batch"], cfg["features"], bench.SEED,
                               device=dev)
    samples = torch.as_tensor(np.asarray(tr.samples)).to(dev)
    sw = D if a.optim == "adagrad" else 0
    dc = DeviceCache(cfg["num_ids"], cap, D, state_width=sw, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    dc.fast_rows.copy_(torch.rand((cap, D), device=dev, generator=g) - 0.5)
    if sw:
        dc.fast_state.zero_()
    lr = 0.01
    batches = []
    for b in range(a.batches):
        ids = samples[b * cfg["batch"]:(b + 1) * cfg["batch"]].reshape(-1)
        uids, inv, ucnt = torch.unique(ids, sorted=True, return_inverse=True, return_counts=True)
        U = uids.numel()
        uslots = torch.randperm(cap, device=dev, generator=g)[:U].int()
        grad = torch.randn((ids.numel(), D), device=dev, generator=g)
        batches.append((uslots, inv.int(), ucnt.int(), grad))
    N = batches[0][1].numel()

    # correctness once (float64 reference of the same update)
    uslots, inv, ucnt, grad = batches[0]
    before = dc.fast_rows.double().clone()
    st_before = dc.fast_state.double().clone() if sw else None
    dc.backward_update(uslots, inv, ucnt, None, N, False, None, "sum", grad, a.optim, lr, 1e-10)
    torch.cuda.synchronize()
    gsum = torch.zeros((uslots.numel(), D), dtype=torch.float64, device=dev).index_add_(0, inv.long(), grad.double())
    want = before.clone()
    if sw:
        s = st_before[uslots.long()] + gsum * gsum
        want[uslots.long()] -= lr * gsum / (s.sqrt() + 1e-10)
    else:
        want[uslots.long()] -= lr * gsum
    diff = (dc.fast_rows.double() - want).abs()
    err = (diff / want.abs().clamp_min(1e-2)).max().item()
    abs_err = diff.max().item()
    touched = int((dc.fast_rows.double() != before).any(1).sum().item())

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    for k in range(3):
        uslots, inv, ucnt, grad = batches[k % len(batches)]
        dc.backward_update(uslots, inv, ucnt, None, N, False, None, "sum", grad, a.optim, lr, 1e-10)
    torch.cuda.synchronize()
    ms = []
    for k in range(a.steps):
        uslots, inv, ucnt, grad = batches[k % len(batches)]
        ev[k].record()
        dc.backward_update(uslots, inv, ucnt, None, N, False, None, "sum", grad, a.optim, lr, 1e-10)
        ev[k + 1].record()
    torch.cuda.synchronize()
    ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(a.steps)]
    U = float(np.mean([b[0].numel() for b in batches]))
    algo = N * (4 * D + 8) + U * 8 * D * (2 if sw else 1)
    avg = float(np.mean(ms))
    hbm, src = bench.hbm_peak()
    print(json.dumps({"config": a.config, "optim": a.optim, "N": N, "U_avg": U, "D": D, "ms_avg": avg,
                      "ms_min": float(np.min(ms)), "algorithmic_bytes": algo, "GBps": algo / (avg * 1e-3) / 1e9,
                      "frac_hbm": algo / (avg * 1e-3) / 1e9 / hbm, "hbm_peak": hbm, "peak_source": src,
                      "max_rel_err_vs_f64": err, "max_abs_err": abs_err, "rows_touched": touched, "U_first": int(batches[0][0].numel())}))


if __name__ == "__main__":
    main()
