"""Print a torch.profiler chrome trace (bench.py FC_TORCH_TRACE=path) as a time-ordered
listing: GPU kernels/copies per stream and host CUDA runtime calls longer than a threshold,
relative to the first kernel, so one step's critical path can be read off."""

import json
import sys


def main(path, min_host_us=15.0, limit=400):
    ev = json.load(open(path))["traceEvents"]
    gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
    host = [e for e in ev if e.get("cat") == "cuda_runtime" and "dur" in e and e["dur"] >= min_host_us]
    py = [e for e in ev if e.get("cat") == "python_function" and "dur" in e and e["dur"] >= 50]
    t0 = min(e["ts"] for e in gpu)
    rows = [(e["ts"] - t0, e["dur"], f"GPU s{e.get('args', {}).get('stream', '?')}", e["name"][:70]) for e in gpu]
    rows += [(e["ts"] - t0, e["dur"], "host", e["name"][:70]) for e in host]
    rows.sort()
    for ts, d, who, name in rows[:limit]:
        print(f"{ts:9.1f} {d:8.1f}  {who:8s} {name}")


if __name__ == "__main__":
    main(sys.argv[1], *(float(a) for a in sys.argv[2:3]))
