#!/usr/bin/env python
"""bench.py — cached-embedding lookups/s on B200 (BASELINE.json metric).

Workload (N=1): BASELINE configs[1], the Criteo-Kaggle shape — 33,762,577 rows x
dim 128 fp32, frequency-reordered cache at 1.5% (506,438 slots), Zipf(1.05) ids
from the reference generator's stream, batch 16384 x 26 (425,984 lookups/step).
One step (--step train, default) = the cached EmbeddingBag's training step:
prepare_cache (cache_manager.py:234-348) -> pooled forward (sum, one id per
(sample, feature)) -> fused backward + sparse SGD on the cached rows, all in
libfreqcache_b200 kernels. --step sim runs the reference simulator's per-batch
work instead (prepare -> lookup -> deterministic row update, simulator.py:416-455).
At N>1 GPUs the table is row-sharded (id % N) with NCCL id/row all-to-alls and
every rank processes its own 16384 x 26 ids per step (weak scaling).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config small] [--step sim]

`--impl reference` times the reference CPU path (the oracle port in oracle/; the
Python reference itself cannot run on the GPU box) on the same workload and step:
prepare + gather + scatter_update(-lr * grad). Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

# more hardware work queues than torch's/the library's streams: no false dependencies
# between the index, transfer, copy-engine and compute streams (set before CUDA init)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# rank 0 prints exactly one JSON line on stdout: keep NCCL's banner / logs on stderr
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE configs[1]
    "criteo_kaggle": dict(num_ids=33_762_577, dim=128, ratio=0.015, alpha=1.05, batch=16384, features=26),
    # BASELINE configs[0] (reference CPU-runnable case)
    "small": dict(num_ids=1_000_000, dim=128, ratio=0.015, alpha=1.05, batch=1024, features=26),
    # BASELINE configs[2]: Avazu shape, mean pooling with per-sample weights (sum(w*row)/L), 5% cache,
    # batch 65,536 (the paper's Avazu batch); Zipf(1.05) like the other configs
    "avazu": dict(num_ids=9_445_823, dim=64, ratio=0.05, alpha=1.05, batch=65536, features=22, mode="mean",
                  psw=True),
    # BASELINE configs[4], one GPU's share of the 8-GPU job: 204,184,588 rows / 8 (row-sharded),
    # uniform ids, 0.5% cache, 65,536 lookups per step (SURVEY 8d instantiation (i)), Adagrad with the
    # optimizer state cached and written back with its rows
    "stress": dict(num_ids=25_523_073, dim=128, ratio=0.005, alpha=None, batch=65536, features=1,
                   optimizer="adagrad"),
    # BASELINE configs[3]: MLPerf DLRM Criteo-1TB shape, 26 tables capped at 40M rows (204,184,588 rows,
    # TorchRec's MLPerf sizes), dim 128, 1.5% cache (3,062,768 slots), one global Zipf(1.05)
    # law (the reference's model); the reference shards it column-wise (--shard column) at 2/4/8 GPUs
    "criteo_1tb": dict(num_ids=204_184_588, dim=128, ratio=0.015, alpha=1.05, batch=16384, features=26),
}
SEED = 1
UPDATES_SEED = 7
METRIC = "cached-embedding lookups/sec"
# kernels launched per step (checked against the ncu launch list, profiles/r01_launches_*):
# synchronous prepare = k_clear_pending + 16 (k_begin, k_mark_ids, 4 compactions x (count + emit),
# k_unique_info, k_inverse, k_plan, k_evict_async, k_admit_async_tma, k_finish); pooled forward 1;
# sim update 1; backward = radix sort (histogram + 2 one-sweep passes) + fused stream + fix-up = 5
# (4 after a pipelined prepare: its index phase makes the histograms)
KERNELS_PER_STEP = 17 + 1 + 1
KERNELS_PER_TRAIN_STEP = 17 + 1 + 5
# prefetch pipeline (round 2, fused index phase): 11 index kernels (k_begin, k_mark_ids, ids count +
# emit, k_unique_info, k_inverse_plan, victims+misses count, victims emit with their slot-table
# changes, misses emit + free-slot count, free-slot emit with the admissions' slot-table changes,
# k_finish_publish) + k_admit_stage_tma + k_clear_pending, k_evict_commit, k_admit_commit = 15
# instead of the synchronous prepare's 17
PIPELINE_EXTRA_KERNELS = 15 - 17
PIPELINE_BWD_SAVED = 1  # the fused backward after a pipelined prepare: no histogram kernel
# row-sharded training step (profiles/r01_launches_sharded*): fc_route 6 (k_begin, k_route_mark,
# count + emit, k_route_inverse, k_route_finish) + the owner's pipelined prepare 17 + 4 + the
# requester's gradient reduction 5 + the owner's apply (k_bwd_direct when every received id is
# distinct, always at world 1; else the 5-kernel grouped backward) + row return (peer memory:
# k_pool_to_peers + k_gather_from_peers; NCCL: the owner's k_pool1) + the requester's k_pool1
SHARDED_BASE_KERNELS = 6 + 17 + 5 + 1  # + PIPELINE_EXTRA_KERNELS when prefetching
# miss staging / admission through the TMA bulk-copy engine (row width a multiple of 16 B;
# FC_XFER_TMA=0 / FC_NO_TMA=1 select the SM-load kernels)
TMA = os.environ.get("FC_XFER_TMA", "1") != "0" and not os.environ.get("FC_NO_TMA")
KSTEPS = 5  # extra steps timed kernel by kernel after the timed region


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- workload
def make_workload(cfg, n_batches, device=None, keep_counts=False):
    from paper_2208_05321_b200 import workload
    from paper_2208_05321_b200.store import fast_capacity

    t0 = time.perf_counter()
    if cfg["alpha"] is None:
        tr = workload.gen_uniform(cfg["num_ids"], n_batches * cfg["batch"], cfg["features"], SEED)
    else:
        tr = workload.gen_zipf(cfg["num_ids"], cfg["alpha"], n_batches * cfg["batch"], cfg["features"], SEED,
                               device=device)
    t1 = time.perf_counter()
    # frequency reorder over the whole trace (simulator.py:363-364)
    if device is not None:  # libfreqcache_b200's fc_build_reorder (bincount + stable radix argsort on device)
        from paper_2208_05321_b200.freq_stats import build_reorder_device

        freq, idx = build_reorder_device(tr.samples, cfg["num_ids"], device, keep_counts=keep_counts)
        id_of = idx.id_of
        counts_np = freq.counts if keep_counts else None
    else:
        counts = np.bincount(tr.samples.reshape(-1), minlength=cfg["num_ids"])
        id_of = np.argsort(-counts, kind="stable").astype(np.int64)
    rank_of = np.empty_like(id_of)
    rank_of[id_of] = np.arange(id_of.size, dtype=np.int64)
    log(f"[bench] trace {tr.samples.shape} in {t1 - t0:.1f}s, reorder {time.perf_counter() - t1:.1f}s")
    samples = (tr.samples, counts_np) if (keep_counts and device is not None) else tr.samples
    return samples, rank_of, id_of, fast_capacity(cfg["num_ids"], cfg["ratio"])


# ----------------------------------------------------------------------------- measurement helpers
_NVML_POLLER = r"""
import sys, time
import pynvml as nv
nv.nvmlInit()
try:
    h = nv.nvmlDeviceGetHandleByPciBusId(sys.argv[1])
except Exception:
    h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[2]))
reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
print("ready", flush=True)
while True:
    t = time.monotonic()
    print("%.6f,%d,%d,%d" % (t, nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx, reasons(h)), flush=True)
    time.sleep(float(sys.argv[3]))
"""


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: an NVML poller in
    its own process (no GIL shared with the timed loop) prints CLOCK_MONOTONIC-stamped
    samples every 2 ms; only those between entering and leaving the region are kept.
    Falls back to `nvidia-smi -lms 100` when nvidia-ml-py is missing."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    BITS = [0x8, 0x40, 0x20, 0x4]  # nvmlClocksThrottleReason{HwSlowdown,HwThermal,SwThermal,SwPowerCap}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.period = float(os.environ.get("FC_CLOCK_POLL_MS", "2")) / 1e3
        self.rows = []  # (sm_mhz, max_mhz, [4 bools])
        self.proc = None
        self.source = None
        self.lines = []

    def _start_nvml(self):
        bus = ""
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.gpu)
            bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
        except Exception:
            pass
        proc = subprocess.Popen([sys.executable, "-c", _NVML_POLLER, bus, str(self.gpu), str(self.period)],
                                stdout=subprocess.PIPE,
                                stderr=subprocess.DEVNULL, text=True)
        if proc.stdout.readline().strip() != "ready":
            proc.kill()
            raise RuntimeError("NVML poller did not start")
        self.th = threading.Thread(target=lambda: self.lines.extend(proc.stdout), daemon=True)
        self.th.start()
        return proc

    def __enter__(self):
        try:
            self.proc = self._start_nvml()
            self.source = "nvml poller, %g ms" % (self.period * 1e3)
        except Exception:
            self.proc = None
        if self.proc is None:
            try:
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                              "--format=csv,noheader,nounits", "-lms", "100"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.source = "nvidia-smi, 100 ms"
                self.th = threading.Thread(target=self._read_smi, daemon=True)
                self.th.start()
            except Exception:
                self.proc = None
        self.t0 = time.monotonic()
        return self

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                self.rows.append((float(parts[0]), float(parts[1]) if parts[1].replace(".", "").isdigit() else None,
                                  [p == "Active" for p in parts[2:]]))

    def __exit__(self, *a):
        self.t1 = time.monotonic()
        if self.proc is None:
            return
        time.sleep(0.01 if self.source.startswith("nvml") else 0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        if self.source.startswith("nvml"):
            parsed = []
            for line in self.lines:
                try:
                    t, sm, mx, r = line.strip().split(",")
                    parsed.append((float(t), (float(sm), float(mx), [bool(int(r) & b) for b in self.BITS])))
                except ValueError:
                    continue
            self.rows = [row for t, row in parsed if self.t0 <= t <= self.t1]
            if not self.rows and parsed:  # a region shorter than the poll interval: the nearest sample
                t, row = min(parsed, key=lambda tr: min(abs(tr[0] - self.t0), abs(tr[0] - self.t1)))
                if min(abs(t - self.t0), abs(t - self.t1)) < 0.02:
                    self.rows = [row]
                    self.source += " (region shorter than the poll interval: nearest sample, within 20 ms)"

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0,
                    "source": self.source}
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows if r[1] is not None]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2][i]})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": self.source}


def host_link_peaks(torch, dev):
    """Pinned cudaMemcpy bandwidth H2D / D2H / both at once (the host-link roofline)."""
    n = 256 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def best(fn, reps=5):
        b = 1e9
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize(dev)
            b = min(b, time.perf_counter() - t)
        return b

    best(lambda: d.copy_(h, non_blocking=True), 2)

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    r = {"h2d_GBps": n / best(lambda: d.copy_(h, non_blocking=True)) / 1e9,
         "d2h_GBps": n / best(lambda: h.copy_(d, non_blocking=True)) / 1e9,
         "bidir_GBps": 2 * n / best(both) / 1e9}
    del h, h2, d, d2
    return r


def gpu_local_cpus(index):
    """The GPU's NUMA-local CPU list (sysfs), where the library pins the slow tier and binds its threads."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(index)
        bus = "%04x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
        return open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
    except Exception:
        return None


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- CPU reference arm
def make_grad(n, D, device=None):
    """The fixed upstream gradient of the pooled output used by every training step."""
    g = np.random.default_rng(SEED + 1).standard_normal((n, D), dtype=np.float32) * np.float32(0.01)
    if device is None:
        return g
    import torch

    return torch.from_numpy(g).to(device)


def run_cpu_reference(samples, rank_of, cap, cfg, steps, warmup, step_kind, batch_mult=1, time_budget_s=None):
    """The reference's per-batch loop on host cores through the numpy oracle port.
    train: prepare + gather (bag-size-1 pooled forward) + scatter_update(-lr * grad)
    (cache_manager.py:234-348, 418-438); sim: prepare + gather + apply_unique_update
    (simulator.py:419-433). The slow tier is a lazily materialised buffer."""
    import oracle

    D = cfg["dim"]
    slow = np.empty((cfg["num_ids"], D), dtype=np.float32)  # lazily zero-filled pages
    orc = oracle.OracleCache(rank_of, slow, cap)
    orc.warmup(cap)
    colw = oracle.column_weights(D, UPDATES_SEED)
    B = cfg["batch"] * batch_mult
    n = B * cfg["features"]
    deltas = -LR * make_grad(n, D)
    times = []
    t_start = time.perf_counter()
    for s in range(warmup + steps):
        ids = samples[s * B:(s + 1) * B].reshape(-1)
        t = time.perf_counter()
        p = orc.prepare(ids, s)
        _ = orc.gather(p)
        if step_kind == "train":
            orc.scatter_update(p, deltas[:ids.size])
        else:
            g = oracle.row_scalars(p["unique_ids"], p["unique_counts"], s, UPDATES_SEED)
            orc.apply_unique_update(p, g[:, None] * colw[None, :])
        dt = time.perf_counter() - t
        if s >= warmup:
            times.append(dt)
        if time_budget_s and time.perf_counter() - t_start > time_budget_s and len(times) >= 3:
            break
    return {"step_s": float(np.mean(times)), "steps": len(times), "lookups_per_s": n / float(np.mean(times))}


# ----------------------------------------------------------------------------- GPU arm
LR = 0.05


def fill_pinned(torch, rows, dev, seed):
    """Seeded uniform(+-0.5/D) rows generated on the GPU and written into pinned host memory."""
    t = torch.from_numpy(rows)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    D = rows.shape[1]
    chunk = 1 << 20
    for lo in range(0, rows.shape[0], chunk):
        hi = min(lo + chunk, rows.shape[0])
        t[lo:hi].copy_((torch.rand((hi - lo, D), generator=g, device=dev) - 0.5) * (1.0 / D))
    torch.cuda.synchronize(dev)


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/ncu_traffic.json, written by tools/ncu_summary.py), or None."""
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[kernel]["traffic_bytes"])
    except Exception:
        return None


def rooflines(prof, pool_ms, N, D, links, engine="async", pipelined=False, psw=False, bwd_ms=None, U=None,
              adagrad=False):
    hbm, hbm_src = hbm_peak()
    xfer_ms = prof["transfer_ms"] / max(prof["transfer_launches"] if pipelined else prof["calls"], 1)
    xfer_bytes = prof["host_link_bytes"] / max(prof["calls"], 1)
    if pipelined:  # admissions staged host -> HBM on the transfer stream; write-backs on the copy engine
        kname, peak, src = ("k_admit_stage_tma" if TMA else "k_admit_stage"), links["h2d_GBps"], \
            "pinned cudaMemcpy H2D, measured in this run"
    elif engine == "async":  # admissions only (H2D); write-backs ride the copy engine off the critical path
        kname, peak, src = ("k_admit_async_tma" if TMA else "k_admit_async"), links["h2d_GBps"], \
            "pinned cudaMemcpy H2D, measured in this run"
    else:
        kname, peak, src = "k_transfer_rows", links["bidir_GBps"], "pinned cudaMemcpy H2D+D2H concurrently, measured"
    r_xfer = {"kernel": kname, "bound": "host_link",
              "achieved": xfer_bytes / max(xfer_ms * 1e-3, 1e-12) / 1e9, "peak": peak, "unit": "GB/s",
              "traffic": ncu_traffic(kname), "traffic_note": "DRAM bytes only; the host-link bytes do not touch HBM",
              "algorithmic_bytes_per_launch": xfer_bytes, "launch_ms": xfer_ms,
              "writeback_d2h_bytes_per_step": prof.get("writeback_d2h_bytes", 0) / max(prof["calls"], 1),
              "peak_source": src}
    r_xfer["frac"] = r_xfer["achieved"] / r_xfer["peak"]
    out = [r_xfer]
    if pool_ms:
        # per occurrence: inverse + slot + row read (+ weight); per bag (= occurrence here): row write
        pool_bytes = N * (4 * D + 8 + (4 if psw else 0)) + N * 4 * D
        pool_avg = float(np.mean(pool_ms))
        r_pool = {"kernel": "k_pool1", "bound": "hbm", "achieved": pool_bytes / (pool_avg * 1e-3) / 1e9, "peak": hbm,
                  "unit": "GB/s", "traffic": ncu_traffic("k_pool1"),
                  "traffic_note": "below the algorithmic bytes: repeated head rows hit in L2",
                  "algorithmic_bytes_per_launch": pool_bytes, "launch_ms": pool_avg,
                  "peak_source": hbm_src}
        r_pool["frac"] = r_pool["achieved"] / r_pool["peak"]
        out.append(r_pool)
    if bwd_ms and U:
        # fused backward + optimizer (radix grouping, k_bwd_stream, k_bwd_fixup): per occurrence
        # its gradient row + sort key + order entry; per unique row a read-modify-write of the
        # row (+ the Adagrad state row)
        bwd_bytes = N * (4 * D + 8) + U * 8 * D * (2 if adagrad else 1)
        bwd_avg = float(np.mean(bwd_ms))
        r_bwd = {"kernel": "backward (k_os_hist + 2 x k_os_scatter + k_bwd_stream + k_bwd_fixup)", "bound": "hbm",
                 "achieved": bwd_bytes / (bwd_avg * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                 "traffic": ncu_traffic("k_bwd_stream"),
                 "traffic_note": "ncu DRAM bytes of k_bwd_stream alone", "algorithmic_bytes_per_launch": bwd_bytes,
                 "launch_ms": bwd_avg, "peak_source": hbm_src}
        r_bwd["frac"] = r_bwd["achieved"] / r_bwd["peak"]
        out.append(r_bwd)
    out.sort(key=lambda r: -r["launch_ms"])
    return out


def workload_config(args, cfg, world):
    """The workload both arms measure (identical dicts: the driver compares them)."""
    D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
    shard = args.shard
    return {"workload": args.config + (f"@batch{args.batch}" if args.batch else "") + (f"@dim{args.dim}" if args.dim else ""), "num_rows": cfg["num_ids"], "dim": D, "cache_ratio": cfg["ratio"],
            "zipf_alpha": cfg["alpha"], "batch_per_gpu": B, "global_batch": B * world, "features": F,
            "lookups_per_step": B * F * world, "batch_scaling": args.batch_scaling if world > 1 else None,
            "pooling": cfg.get("mode", "sum") + (" with per-sample weights" if cfg.get("psw") else "") + ", bag size 1",
            "optimizer": cfg.get("optimizer", "sgd"), "ids": "uniform" if cfg["alpha"] is None else f"zipf({cfg['alpha']})",
            "step": ("forward (prepare + pooled gather) + backward/update" if args.step == "train"
                     else "prepare + pooled forward + simulator row update"),
            "write_back": "dirty_only", "evict_mode": "occupancy_aware",
            "parallelism": "single" if shard is None else f"{shard}wise{world}",
            "l2": "inputs larger than L2 (fast tier %d MB, id/rank maps %d MB, new batch every step)"
                  % (fc_capacity(cfg) * D * 4 >> 20, cfg["num_ids"] * 12 >> 20)}


def scaling_kind(args, world):
    """strong: the config's batch is the global batch, split over the N data-parallel ranks
    (the reference's multi-GPU model: every shard serves the one global batch);
    weak: every rank takes the config's batch (global batch x N)."""
    return "weak" if world == 1 else args.batch_scaling


def fc_capacity(cfg):
    return max(1, int(cfg["ratio"] * cfg["num_ids"]))


def trace_batches(args, world):
    """Batches of B samples per rank in the generated trace (the frequency reorder scans all
    of them; both arms generate the same trace for the same --steps/--warmup/--gpus)."""
    per_rank = args.trace_batches // world if args.batch_scaling == "weak" else args.trace_batches
    return max(per_rank, args.warmup + 2 * args.steps + 2 * KSTEPS + 2)


def launches_per_step(args, shard_mode, pipelined, world):
    """Our kernels launched per timed step (checked against the ncu launch lists in profiles/)."""
    if shard_mode is None:
        if args.step == "sim":
            return KERNELS_PER_STEP + (PIPELINE_EXTRA_KERNELS if pipelined else 0)
        return KERNELS_PER_TRAIN_STEP + (PIPELINE_EXTRA_KERNELS - PIPELINE_BWD_SAVED if pipelined else 0)
    if shard_mode == "column":  # prepare of the global batch + pool + fused backward (NCCL kernels not counted)
        peer = args.peer or (world > 1 and not args.no_peer)  # + the gradient-column gather over peer memory
        return KERNELS_PER_TRAIN_STEP + (PIPELINE_EXTRA_KERNELS - PIPELINE_BWD_SAVED if pipelined else 0) + int(peer)
    return (SHARDED_BASE_KERNELS + (PIPELINE_EXTRA_KERNELS if pipelined else 0) + (1 if world == 1 else 5)
            + (2 if args.peer else 1))


def table_placement(cfg, world):
    """--shard table: one table per sparse feature, laid out contiguously -- Criteo Kaggle's own
    26 cardinalities when the config has its 33,762,577 rows (sharding.py:26-30), else equal
    tables -- placed by the reference's largest-first greedy (plan_tables_greedy,
    sharding.py:158-172)."""
    from paper_2208_05321_b200.distributed import TablePlacement
    from paper_2208_05321_b200.sharding import CRITEO_KAGGLE_TABLE_SIZES

    T = cfg["features"]
    if sum(CRITEO_KAGGLE_TABLE_SIZES) == cfg["num_ids"]:
        sizes = np.asarray(CRITEO_KAGGLE_TABLE_SIZES, dtype=np.int64)
    else:
        sizes = np.full(T, cfg["num_ids"] // T, dtype=np.int64)
        sizes[:cfg["num_ids"] % T] += 1
    return TablePlacement.balanced(sizes, world)


def run_ours(args, cfg, torch, rank, world):
    import paper_2208_05321_b200 as fc
    from paper_2208_05321_b200.embedding import CachedEmbeddingBag

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    W, K = args.warmup, args.steps
    D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
    N = B * F
    n_batches = trace_batches(args, world)
    # global batch = world x B samples; this rank's slice is rows [rank*B, (rank+1)*B) of each global batch
    shard_mode = args.shard
    sharded = shard_mode is not None
    rowwise = shard_mode in ("row", "table")  # owner-local reorders need the id counts
    samples, rank_of, id_of, cap = make_workload(cfg, n_batches * world, device=dev, keep_counts=rowwise)
    counts = None
    if rowwise:
        samples, counts = samples
    links = host_link_peaks(torch, dev)
    gout = make_grad(N, D, dev)
    MODE, OPT = cfg.get("mode", "sum"), cfg.get("optimizer", "sgd")
    psw = None
    if cfg.get("psw"):  # per-sample weights ~ U(0, 1), seeded, one per lookup
        g = torch.Generator(device=dev)
        g.manual_seed(SEED + 2)
        psw = torch.rand(N, generator=g, device=dev)

    def local_batch(s):
        lo = (s * world + rank) * B
        return lo, lo + B

    t0 = time.perf_counter()
    if not sharded:
        rows = fc.store.pinned_empty((cfg["num_ids"], D))
        fill_pinned(torch, rows, dev, SEED)
        mod = CachedEmbeddingBag(cfg["num_ids"], D, cfg["ratio"], mode=MODE, idx_map=fc.IdxMap(rank_of, id_of),
                                 optimizer=OPT, lr=LR, slow_rows=rows, warmup=True, engine=args.engine)
        dcs = [mod.cache]
        shard = None
    elif shard_mode == "column":
        from paper_2208_05321_b200.distributed import ColumnShardedEmbedding, CudaShard

        # the fused peer-memory exchange is the column split's default at N>1 (--no-peer: NCCL)
        col_peer = args.peer or (world > 1 and not args.no_peer)

        # the reference's column-wise split (sharding.py:46-118): every rank caches all rows of its
        # column slice over the GLOBAL batch (identical decisions on every rank)
        lo_c, hi_c = fc.partition_columns(D, world).ranges[rank]
        rows = fc.store.pinned_empty((cfg["num_ids"], hi_c - lo_c))
        fill_pinned(torch, rows, dev, SEED + rank)
        shard = CudaShard(cfg["num_ids"], hi_c - lo_c, cap, rows, fc.IdxMap(rank_of, id_of), optimizer=OPT, lr=LR,
                          device=dev, engine=args.engine)
        # --peer: the pooled-columns all-to-all and its backward mirror fused into the gather /
        # gradient-pull kernels over NVLink peer memory (PeerColumns) instead of NCCL
        mod = ColumnShardedEmbedding(shard, D, world, rank, mode=MODE, device=dev, peer_rows=N if col_peer else 0)
        if col_peer and mod.peer is None:
            log(f"[bench] rank {rank}: {mod.peer_error}")
        dcs = [shard.cache]
    else:
        from paper_2208_05321_b200.distributed import (CudaShard, RowShardedEmbedding, shard_rows_for_rank,
                                                       shard_tables_for_rank)

        placement = table_placement(cfg, world) if shard_mode == "table" else None
        idx = (shard_rows_for_rank(counts, rank, world) if placement is None
               else shard_tables_for_rank(counts, placement, rank))
        rows = fc.store.pinned_empty((idx.num_ids, D))
        fill_pinned(torch, rows, dev, SEED + rank)
        shard = CudaShard(idx.num_ids, D, fc.fast_capacity(idx.num_ids, cfg["ratio"]), rows, idx, optimizer=OPT,
                          lr=LR, device=dev, engine=args.engine, global_num_ids=cfg["num_ids"])
        # owners write the looked-up rows straight into the requesters' buffers over NVLink
        # peer memory (fc_pool_to_peers) with --peer; by default the rows come back by NCCL all-to-all
        # (faster at world 1, 325-332 vs 290-316 M lookups/s, profiles/r01_bench_sharded_*.json; the
        # peer path is untested across GPUs in this build's runs)
        mod = RowShardedEmbedding(shard, world, rank, mode=MODE, device=dev, peer_rows=N if args.peer else 0,
                                  placement=placement)
        dcs = [shard.cache]
        cap = shard.cache.capacity
    dc = dcs[0]
    log(f"[bench] rank {rank}: slow tier {rows.nbytes / 2**30:.1f} GiB pinned+filled, cache ready in "
        f"{time.perf_counter() - t0:.1f}s")
    ids_dev = torch.from_numpy(samples).to(dev)
    ids_ready = torch.cuda.Event()  # the whole trace is resident before the first step
    ids_ready.record(torch.cuda.current_stream(dev))
    out_buf = torch.empty((N, D), dtype=torch.float32, device=dev)
    colw = torch.from_numpy(fc.update_column_weights(D, UPDATES_SEED)).to(dev)
    stream = torch.cuda.current_stream(dev)
    stats, pool_ms, bwd_ms = [], [], []
    step_events = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(2 * KSTEPS)]

    bview = [ids_dev[local_batch(k)[0]:local_batch(k)[1]].reshape(-1) for k in range(n_batches)]

    def step(s, timed):
        ids = bview[s]
        if sharded:  # sharded training step: id exchange, this rank's cache, row/activation exchange
            if pipelined and depth2:  # next batch's exchange + prepare begun before this batch is committed
                mod.prefetch(bview[s + 1], ready=ids_ready)
            out = mod(ids, None, psw)
            if pipelined and not depth2:  # next batch's id exchange + owner prepare overlap this backward
                mod.prefetch(bview[s + 1], ready=ids_ready)
            out.backward(gout)
            li = getattr(mod, "last_info", None)
            stats.append((li.unique, li.hits, li.misses, li.evictions, li.rows_to_slow) if li is not None
                         else (0, 0, 0, 0, 0))
            return
        if pipelined and depth2:  # batch s+1 begun before batch s is committed: its index phase
            dc.prepare_begin(bview[s + 1], s + 1, ready=ids_ready)  # starts when batch s's ends
        if pipelined:  # batch s was prefetched during step s-1: commit it
            info, uids, ucnt, uranks, uslots, inverse, _ = dc.prepare_commit()
        else:
            info, uids, ucnt, uranks, uslots, inverse, _ = dc.prepare(ids, s)
        e = step_events[len(pool_ms)] if timed else None  # created before the timed region
        if timed:
            e[0].record(stream)
        dc.pooled(uslots, inverse, N, per_sample_weights=psw, mode=MODE, out=out_buf)
        if timed:
            e[1].record(stream)
        if pipelined and not depth2:  # batch s+1's index phase + miss staging overlap this backward
            dc.prepare_begin(bview[s + 1], s + 1, ready=ids_ready)
        if args.step == "train":
            dc.backward_update(uslots, inverse, ucnt, None, N, False, psw, MODE, gout, OPT, LR, 1e-10)
        else:
            dc.synthetic(uids, ucnt, uslots, fc.updates.batch_salt(s, UPDATES_SEED), colw)
        if timed:
            e[2].record(stream)
            pool_ms.append(e)
        stats.append((info.unique, info.hits, info.misses, info.evictions, info.rows_to_slow))

    # sharded modules prefetch through their own prefetch() (column-wise: all-gather of the next
    # batch's ids + prepare_begin of the global batch; row-wise: id exchange + the owner's prepare_begin)
    pipelined = args.engine == "async" and not args.no_prefetch
    # sharded modules default to depth 1: two batches in flight measured slower there (row-wise
    # 1.48 vs 1.27-1.31 ms at cfg2, equal at the N=8 per-rank batch; profiles/r02_sharded_depth_ab.txt)
    depth = args.prefetch_depth if args.prefetch_depth is not None else (1 if sharded else 2)
    depth2 = depth == 2 and not os.environ.get("FC_XFER_AFTER_UPDATE")
    if pipelined and sharded and depth2:
        mod.prefetch(bview[0], ready=ids_ready)
    elif pipelined and not sharded:
        dc.prepare_begin(bview[0], 0, ready=ids_ready)
    for s in range(W):
        step(s, False)
    torch.cuda.synchronize(dev)
    stats.clear()

    # ---- timed region: inputs resident in HBM, one event per step -------------
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index) as clk:
        ev[0].record(stream)
        for k in range(K):
            step(W + k, False)
            if k == K - 1:  # the region ends when the async write-backs queued so far are in the slow tier
                for c in dcs:
                    c.drain_stream(stream)
            ev[k + 1].record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    # ---- per-kernel timing: a few more steps with events around the kernels ---
    # (kept out of the timed region: extra event records perturb the async engine)
    stats_main = list(stats)
    dc.profile(True)
    for k in range(KSTEPS):
        step(W + K + k, True)
    torch.cuda.synchronize(dev)
    prof = dc.profile(False)
    if os.environ.get("FC_TORCH_TRACE"):  # diagnostic: a CUPTI timeline of a few steps (tools/trace_gaps.py)
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as tp:
            for k in range(4):
                step(W + K + KSTEPS + k, False)
            torch.cuda.synchronize(dev)
        tp.export_chrome_trace(os.environ["FC_TORCH_TRACE"])
    # ---- the same kernels isolated: KSTEPS synchronous steps (no prefetch overlap), so the
    # roofline of each kernel is also reported without the host-link interference
    prof_iso, p_ms_iso, b_ms_iso = None, [], []
    if pipelined and not sharded:
        dc.prepare_commit()  # the batch prefetched by the last profiled step is executed first
        pipelined = False
        n_contended = len(pool_ms)
        dc.profile(True)
        for k in range(KSTEPS):
            step(W + K + KSTEPS + k, True)
        torch.cuda.synchronize(dev)
        prof_iso = dc.profile(False)
        pipelined = True
        p_ms_iso = [e[0].elapsed_time(e[1]) for e in pool_ms[n_contended:]]
        b_ms_iso = [e[1].elapsed_time(e[2]) for e in pool_ms[n_contended:]]
        del pool_ms[n_contended:]
        del stats[-KSTEPS:]
        dc.prepare_begin(bview[W + K + 2 * KSTEPS], W + K + 2 * KSTEPS, ready=ids_ready)
    step_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(K)]
    total_ms = ev[0].elapsed_time(ev[K])
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    p_ms = [e[0].elapsed_time(e[1]) for e in pool_ms]
    b_ms = [e[1].elapsed_time(e[2]) for e in pool_ms]

    # ---- e2e: the public API (module forward+backward) from pinned host ids ----
    if pipelined and not sharded and dc.prefetch_outstanding:
        dc.prepare_commit()
    if pipelined and sharded:
        mod.flush()  # commits the timed loop's outstanding prefetches before the e2e loop primes its own
    ids_host = torch.from_numpy(samples).pin_memory()
    hb = [ids_host[local_batch(k)[0]:local_batch(k)[1]].reshape(-1) for k in range(n_batches)]
    # warm-up exactly like the timed loop (the first autograd backward starts torch's device
    # thread, ~1.4 s once; the prefetch buffers' allocation pattern reaches steady state, so no
    # cudaMalloc lands inside the timed region)
    e0 = W + K + 2 * KSTEPS
    ew = e0 - W
    d2 = pipelined and depth2
    if d2:
        mod.prefetch(hb[ew])
    out = None
    for k in range(W):  # batches e0-W .. e0-1
        if d2:
            mod.prefetch(hb[ew + k + 1])  # batch k+1 begun before batch k's forward commits k
        out = mod(hb[ew + k], None, psw)
        if pipelined and not d2:
            mod.prefetch(hb[ew + k + 1])
        out.backward(gout)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    t = time.perf_counter()
    hits_read = 0
    host_steps = []
    gc_ms = [0.0, None]

    def _gc_cb(phase, info):  # how much of the e2e time went to Python's cyclic GC
        if phase == "start":
            gc_ms[1] = time.perf_counter()
        elif gc_ms[1] is not None:
            gc_ms[0] += (time.perf_counter() - gc_ms[1]) * 1e3
            gc_ms[1] = None

    import gc

    gc.callbacks.append(_gc_cb)
    ms0 = torch.cuda.memory_stats(dev)
    for k in range(K):
        th = time.perf_counter()
        if d2:
            mod.prefetch(hb[e0 + k + 1])  # next batch's cache work, begun ahead of this forward's commit
        out = mod(hb[e0 + k], None, psw)  # H2D of the ids inside forward (or inside the previous step's prefetch)
        if pipelined and not d2:
            mod.prefetch(hb[e0 + k + 1])  # next batch's cache work overlaps this backward
        out.backward(gout)  # upstream gradient of the pooled output -> fused SGD on the cached rows
        if not sharded:
            hits_read += mod.last_info.hits  # the step's result (prepare counters, read back D2H)
        host_steps.append(time.perf_counter() - th)
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - t
    gc.callbacks.remove(_gc_cb)
    ms1 = torch.cuda.memory_stats(dev)
    alloc_diag = {k: ms1.get(k, 0) - ms0.get(k, 0) for k in ("num_alloc_retries", "num_device_alloc", "num_device_free",
                                                             "num_sync_all_streams")}
    if os.environ.get("FC_TORCH_TRACE_E2E"):  # diagnostic: CUPTI timeline of a few module-API steps
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as tp:
            for k in range(K, K + 4):
                if d2:
                    mod.prefetch(hb[(e0 + k + 1) % n_batches])
                out = mod(hb[(e0 + k) % n_batches], None, psw)
                if pipelined and not d2:
                    mod.prefetch(hb[(e0 + k + 1) % n_batches])
                out.backward(gout)
            torch.cuda.synchronize(dev)
        tp.export_chrome_trace(os.environ["FC_TORCH_TRACE_E2E"])
    if pipelined:
        mod.flush()  # commits the last prefetch
    if world > 1:
        tt = torch.tensor([e2e_s], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(tt.item())

    st_arr = np.array(stats_main, dtype=np.float64)
    uniq, hits, misses, evict, wb = st_arr.mean(axis=0)
    train = args.step == "train" and not sharded
    ada = OPT == "adagrad"
    rl = rooflines(prof, p_ms, N, D, links, args.engine, pipelined, psw is not None, b_ms if train else None, uniq, ada)
    rl_iso = rooflines(prof_iso, p_ms_iso, N, D, links, args.engine, False, psw is not None,
                       b_ms_iso if train else None, uniq, ada) if prof_iso else None
    lookups = N * world  # every rank processes its own B x F ids per step
    res = {
        "metric": METRIC, "value": lookups * K / (total_ms * 1e-3), "unit": "lookups/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": scaling_kind(args, world),
        "vs_baseline": None, "dtype": "fp32 rows, int32 ids",
        "data": "synthetic: reference gen_zipf stream (seed 1), seeded rows",
        "config": workload_config(args, cfg, world),
        "implementation": {"engine": args.engine, "prefetch": pipelined,
                           "prefetch_depth": (2 if depth2 else 1) if pipelined else 0,
                           "exchange": (None if not rowwise else "unique ids by NCCL all-to-all; rows back "
                                        + ("by owner-side peer-memory writes" if args.peer else "by NCCL all-to-all")
                                        ) if shard_mode != "column" else
                           ("all-gather of ids; pooled columns written into the requesters' outputs over peer memory "
                            "(fc_pool_cols_to_peers), gradient columns pulled back (fc_gather_cols_from_peers)"
                            if getattr(mod, "peer", None) is not None
                            else "all-gather of ids; pooled columns by NCCL all-to-all (reference semantics)"),
                           "capacity_per_gpu": cap},
        "step_latency_ms": {"p50": float(np.percentile(step_ms, 50)), "p99": float(np.percentile(step_ms, 99)),
                            "prepare_avg": (None if pipelined else prof["prepare_ms"] / max(prof["calls"], 1)),
                            "miss_transfer_avg": rl[0]["launch_ms"] if rl[0]["bound"] == "host_link" else None,
                            "pool_avg": float(np.mean(p_ms)) if p_ms else None,
                            "update_avg": float(np.mean(b_ms)) if b_ms else None,
                            "async_writeback_wait_avg": prof["host_wait_ms"] / max(prof["calls"], 1),
                            "host_scatter_avg": prof["scatter_ms"] / max(prof["scatter_jobs"], 1)},
        "e2e": {"value": lookups * K / e2e_s, "unit": "lookups/s", "h2d_bytes_per_step": N * samples.itemsize,
                "d2h_bytes_per_step": 64, "ms_per_step": e2e_s / K * 1e3,
                "host_step_ms": {"p50": float(np.percentile(host_steps, 50)) * 1e3,
                                 "max": float(np.max(host_steps)) * 1e3, "python_gc_total": gc_ms[0],
                                 "torch_allocator": alloc_diag},
                "path": "CachedEmbeddingBag.forward(pinned host ids) + out.backward(grad) (fused SGD); result = "
                        "prepare hit/miss counters read back" if not sharded
                else f"{type(mod).__name__}.forward(pinned host ids) + prefetch(next ids) + out.backward(grad)"},
        "gpu_launches": launches_per_step(args, shard_mode, pipelined, world) * K,
        "roofline": rl[0], "roofline_secondary": rl[1] if len(rl) > 1 else None,
        "roofline_all": {r["kernel"]: r for r in rl},
        "roofline_isolated": ({"note": "same kernels in synchronous steps (no prefetch overlap), after the "
                                       "timed region", **{r["kernel"]: r for r in rl_iso}} if rl_iso else None),
        "host_link": links,
        "clocks": clk.summary(),
    }
    if not rowwise:
        if wb < 0:  # pipeline commits filter the dirty victims on device: the engine's exact count
            wb = prof["writeback_rows"] / max(prof["scatter_jobs"], 1)
        res.update({"hit_ratio": hits / uniq, "unique_per_step": uniq, "misses_per_step": misses,
                    "evictions_per_step": evict, "writeback_rows_per_step": wb})
        # host-DRAM traffic of the step: the admitted rows are read by the GPU over the link; the
        # write-back rows land in pinned staging (D2H), are read back and scattered into the slow
        # tier by the host threads (non-temporal stores: no read-for-ownership)
        row = 4 * (D + (D if OPT == "adagrad" else 0))
        d2h = prof["writeback_d2h_bytes"] / max(prof["scatter_jobs"], 1)
        hb = misses * row + d2h + wb * (row + 4) + wb * row
        res["host_memory"] = {"bytes_per_step": hb, "GBps": hb / (total_ms / K * 1e-3) / 1e9,
                              "parts": {"admission_reads": misses * row, "d2h_writes": d2h,
                                        "scatter_reads": wb * (row + 4), "scatter_writes": wb * row},
                              "scatter_threads": prof.get("scatter_threads"),
                              "local_cpus": gpu_local_cpus(dev.index)}
    return res, samples, rank_of, cap


_STDOUT = None


def quiet_stdout():
    """Send everything written to fd 1 (native libraries' banners, e.g. NCCL's version
    line) to stderr, so that the one JSON result line is all that reaches stdout."""
    global _STDOUT
    sys.stdout.flush()
    _STDOUT = os.dup(1)
    os.dup2(2, 1)


def emit(doc):
    sys.stdout.flush()
    if _STDOUT is not None:
        os.write(_STDOUT, (json.dumps(doc) + "\n").encode())
    else:
        print(json.dumps(doc), flush=True)


def reference_package():
    """The UNMODIFIED reference package, installed into baseline/_ref by tools/install_reference.sh
    (pip --target from /root/reference); None when it is absent (then the oracle port runs)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "freqcache")) and ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import freqcache  # noqa: F401
        return freqcache
    except ImportError:
        return None


def host_info():
    """What the CPU numbers ran on (CPU model, cpu_count, thread counts)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    threads = {"OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"), "numpy": None}
    try:
        from threadpoolctl import threadpool_info
        threads["numpy"] = {i.get("internal_api"): i.get("num_threads") for i in threadpool_info()}
    except Exception:
        pass
    if "torch" in sys.modules:
        threads["torch"] = sys.modules["torch"].get_num_threads()
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "threads": threads}


def run_reference_arm(args, cfg, world, steps, warmup, time_budget_s=None):
    """The reference's own CPU implementation of the path on this host: freqcache's CacheStack
    (cache_manager.py:441-562) through its public API -- prepare -> gather (the bag-size-1 pooled
    forward, x per-sample weight) -> scatter_update(-lr * grad) per step (or the simulator's
    apply_unique_update for --step sim) -- on the same trace, reorder and sharding as the GPU arm:
    one stack at N=1; at N>1 the reference's column-wise stacks (sharding.py:62-118, every shard
    prepares the global batch, run one after another as shipped) or, for row-wise, one stack per
    row shard (its id substream, its own reorder) run one after another. numpy is single-threaded
    here, so it uses one core. Slow tiers are lazily zero-filled buffers (values do not change
    the work). Returns (per-step seconds, steps timed, kind, sample note)."""
    fq = reference_package()
    if fq is None:  # not installed: the oracle port (oracle/) of the same loop
        n_batches = trace_batches(args, world)
        samples, rank_of, _, cap = make_workload(cfg, n_batches * world, device=None)
        r = run_cpu_reference(samples, rank_of, cap, cfg, steps, warmup, args.step, batch_mult=world,
                              time_budget_s=time_budget_s)
        return r["step_s"], r["steps"], "port", "numpy oracle restatement of the reference (oracle/)"
    from freqcache import cache_manager as rcm
    from freqcache import freq_stats as rfs
    from freqcache import sharding as rsh
    from freqcache import simulator as rsim
    from freqcache import store as rst
    from freqcache import transmitter as rtx
    from freqcache import workload as rwl

    D, B, F = cfg["dim"], cfg["batch"], cfg["features"]
    nb = trace_batches(args, world)
    t0 = time.perf_counter()
    if cfg["alpha"] is None:  # the reference has no uniform generator: the same seeded draw as the GPU arm
        from paper_2208_05321_b200 import workload as wl
        samples = wl.gen_uniform(cfg["num_ids"], nb * world * B, F, SEED).samples
    else:
        samples = rwl.gen_zipf(cfg["num_ids"], cfg["alpha"], nb * world * B, F, SEED).samples
    counts = rfs.scan_frequencies(samples, cfg["num_ids"]).counts
    log(f"[bench/ref] trace + reorder inputs in {time.perf_counter() - t0:.1f}s")

    def stack(num_rows, width, idx_map):
        cap = rst.fast_capacity(num_rows, cfg["ratio"])
        st = rcm.CacheStack(idx_map=idx_map, slow=rst.SlowTierStore(rows=np.empty((num_rows, width), np.float32)),
                            fast=rst.FastTierStore(slots=np.zeros((cap, width), np.float32)),
                            transmitter=rtx.Transmitter())
        st.warmup(cap)  # simulator.py:393-394
        return st

    shard = args.shard
    if shard == "row":  # one stack per row shard: ids with id % world == r, rank-local reorder
        stacks = []
        for r in range(world):
            stacks.append(stack(len(counts[r::world]), D,
                                rfs.build_reorder(rfs.FrequencyTable(counts=counts[r::world],
                                                                     num_ids=len(counts[r::world])))))
        def parts(ids):
            return [(st, ids[m] // world, m, (0, D)) for st, m in zip(stacks, [ids % world == r for r in range(world)])]
    elif shard == "table":  # one stack per rank over its whole tables, rank-local reorder
        pl = table_placement(cfg, world)
        stacks = []
        for r in range(world):
            g = pl.global_ids(r)
            stacks.append(stack(g.size, D, rfs.build_reorder(rfs.FrequencyTable(counts=counts[g], num_ids=g.size))))
        tstart = pl.starts

        def parts(ids):
            t = np.searchsorted(tstart, ids, side="right") - 1
            own, loc = pl.owner[t], pl.lbase[t] + (ids - tstart[t])
            return [(st, loc[own == r], own == r, (0, D)) for r, st in enumerate(stacks)]
    else:
        idx = rfs.build_reorder(rfs.FrequencyTable(counts=counts, num_ids=cfg["num_ids"]))
        plan = rsh.partition_columns(D, world if shard == "column" else 1)
        stacks = [stack(cfg["num_ids"], e - s, idx) for s, e in plan.ranges]

        def parts(ids):
            return [(st, ids, None, cr) for st, cr in zip(stacks, plan.ranges)]
    log(f"[bench/ref] {len(stacks)} reference stack(s) ready in {time.perf_counter() - t0:.1f}s")
    n = B * F * world
    gout = make_grad(n, D)
    psw = None
    if cfg.get("psw"):
        psw = np.random.default_rng(SEED + 2).random(n, dtype=np.float32)
        gout = gout * psw[:, None]
    colw = rsim.update_column_weights(D, UPDATES_SEED)
    times = []
    t_start = time.perf_counter()
    for s in range(warmup + steps):
        ids = samples[s * world * B:(s + 1) * world * B].reshape(-1).astype(np.int64)
        t = time.perf_counter()
        for st, sub, m, (lo, hi) in parts(ids):
            prep = st.prepare(sub, s)
            rows = st.gather(prep)  # pooled forward, bag size 1
            if psw is not None:
                rows *= (psw if m is None else psw[m])[:, None]
            if args.step == "train":
                st.scatter_update(prep, -LR * (gout if m is None else gout[m])[:, lo:hi])
            else:
                g = rsim.update_row_scalars(prep.unique_ids, prep.unique_counts, s, UPDATES_SEED)
                st.apply_unique_update(prep, g[:, None] * colw[None, lo:hi])
        dt = time.perf_counter() - t
        if s >= warmup:
            times.append(dt)
        if time_budget_s and time.perf_counter() - t_start > time_budget_s and len(times) >= 2:
            break
    note = (f"{len(times)} steps of {n} lookups after {warmup} warm-up steps, reference freqcache "
            f"{getattr(fq, '__version__', '?')} from baseline/_ref ({len(stacks)} stack(s), run in sequence)")
    return float(np.mean(times)), len(times), "reference", note


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-launch under torch.distributed.run with one rank
    per GPU (rendezvous on 127.0.0.1); fails loudly when the box has fewer GPUs."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    log("[bench] spawning: " + " ".join(cmd))
    sys.stdout.flush()
    if _STDOUT is not None:
        os.dup2(_STDOUT, 1)  # the ranks print the JSON line to the real stdout
    os.execv(sys.executable, cmd)


def main():
    quiet_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="criteo_kaggle", choices=list(CONFIGS))
    ap.add_argument("--step", default="train", choices=["train", "sim"])
    ap.add_argument("--shard", default=None, choices=["row", "column", "table"],
                    help="table split over the ranks: column (the reference's column-wise split, "
                         "sharding.py:46-118; default at N>1), row (id %% N owners, index work sharded too) or table "
                         "(whole tables per rank, the reference's greedy placement)")
    ap.add_argument("--trace-batches", type=int, default=64)
    ap.add_argument("--batch", type=int, default=None,
                    help="override the config's (global) batch in samples, e.g. to time one rank's share")
    ap.add_argument("--dim", type=int, default=None,
                    help="override the config's row width, e.g. to time one column shard's share at world 1")
    ap.add_argument("--batch-scaling", default="strong", choices=["strong", "weak"],
                    help="N>1: strong = the config's batch is the global batch, B/N samples per rank (default; "
                         "the reference's sharding serves one global batch); weak = B samples per rank. At 1.5%% "
                         "cache weak is infeasible at N=8 on criteo_kaggle (2.4%% of the rows per global batch)")
    ap.add_argument("--cpu-baseline-s", type=float, default=20.0, help="time budget of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--prefetch-depth", type=int, default=None, choices=[1, 2],
                    help="2: batch t+1's prefetch is begun before batch t is committed (default unsharded); "
                         "1: after forward(t) (default for the sharded modules)")
    ap.add_argument("--sharded", action="store_true", help="alias of --shard row (also at one GPU)")
    ap.add_argument("--peer", action="store_true",
                    help="sharded runs: the return exchange fused into the owners' kernels over NVLink peer memory "
                         "(CUDA IPC) instead of the NCCL all-to-all (row-wise: looked-up rows; column-wise: pooled "
                         "column slices and the gradients' columns)")
    ap.add_argument("--no-peer", action="store_true",
                    help="column-wise at N>1: the NCCL all-to-alls instead of the fused peer-memory exchange "
                         "(row-wise always uses NCCL unless --peer)")
    ap.add_argument("--no-prefetch", action="store_true",
                    help="synchronous prepare each step (no lookahead pipeline)")
    ap.add_argument("--engine", default="async", choices=["async", "zerocopy"],
                    help="transfer engine: async copy-engine write-back (default) or paired zero-copy kernel")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.sharded and args.shard is None:
        args.shard = "row"
    if args.gpus > 1 and args.shard is None:
        # the reference's multi-GPU model: column shards serving one global batch (strong scaling).
        # At the N=2/4/8 per-rank shares it is also the faster split on one GPU: 0.71 / 0.54 / 0.66 ms
        # per step against row-wise 1.12 / 0.72 / 0.79 ms (profiles/r02_strong_scaling_shares.txt)
        args.shard = "column"
    cfg = dict(CONFIGS[args.config])
    if args.batch is not None:
        cfg["batch"] = args.batch
    if args.dim is not None:
        cfg["dim"] = args.dim
    rank = int(os.environ.get("RANK", 0))
    env_world = os.environ.get("WORLD_SIZE")
    world = int(env_world) if env_world is not None else args.gpus
    if args.batch_scaling == "strong" and world > 1:  # the config's batch is the global batch
        if cfg["batch"] % world:
            raise SystemExit(f"bench.py: batch {cfg['batch']} does not split over {world} ranks")
        cfg["batch"] //= world
    if env_world is not None and args.gpus != 1 and int(env_world) != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={env_world}")

    if args.impl == "reference":  # rank 0 alone runs the reference's CPU path; the others exit
        if rank != 0:
            return 0
        step_s, nsteps, kind, note = run_reference_arm(args, cfg, world, args.steps, args.warmup,
                                                       time_budget_s=float(os.environ.get("FC_REF_BUDGET_S", "150")))
        n = cfg["batch"] * cfg["features"] * world
        val = n / step_s
        emit({"metric": METRIC, "value": val, "unit": "lookups/s", "n_gpus": world, "steps": nsteps,
              "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": scaling_kind(args, world),
              "vs_baseline": None, "dtype": "fp32 rows, int64 ids", "data": "synthetic: reference gen_zipf stream (seed 1)",
              "impl": "reference", "config": workload_config(args, cfg, world),
              "cpu_baseline": {"value": val, "unit": "lookups/s", "cores": 1, "kind": kind, "sample": note,
                               **host_info()},
              "e2e": {"value": val, "unit": "lookups/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
        return 0

    if env_world is None and args.shard is not None:
        spawn_ranks(args)  # does not return
    import torch

    if args.shard is not None:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    # a dedicated (non-legacy) stream: no implicit serialisation with the engine's side stream
    with torch.cuda.stream(torch.cuda.Stream()):
        res = run_ours(args, cfg, torch, rank, world)[0]
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        step_s, nsteps, kind, note = run_reference_arm(args, cfg, 1, 8, 2, time_budget_s=args.cpu_baseline_s)
        res["cpu_baseline"] = {"value": cfg["batch"] * cfg["features"] / step_s, "unit": "lookups/s", "cores": 1,
                               "kind": kind, "sample": note, **host_info()}
    if rank == 0:
        emit(res)
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
