"""Probe the GPU box: host cores/RAM, GPU, and pinned host<->device copy bandwidth.

Writes gpurun_out/probe_box.json. Used once per round to fix the host-link
roofline denominator.
"""
import json, os, subprocess, time
import torch

def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:  # noqa
        return str(e)

out = {"cpu_count": os.cpu_count(), "lscpu": sh("lscpu | head -20"), "free_g": sh("free -g"),
       "nvidia_smi": sh("nvidia-smi"), "topo": sh("nvidia-smi topo -m"),
       "pcie": sh("nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max --format=csv")}
dev = torch.device("cuda:0")
res = {}
for mb in (16, 64, 256, 1024):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    def timeit(fn, reps=5):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        return best
    t_h2d = timeit(lambda: d.copy_(h, non_blocking=True))
    t_d2h = timeit(lambda: h.copy_(d, non_blocking=True))
    def bidir():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    t_bi = timeit(bidir)
    res[mb] = {"h2d_GBps": n / t_h2d / 1e9, "d2h_GBps": n / t_d2h / 1e9, "bidir_total_GBps": 2 * n / t_bi / 1e9}
out["copy"] = res
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
print(json.dumps(res, indent=1)); print(out["cpu_count"]); print(out["free_g"]); print(out["pcie"]); print(out["lscpu"])
