"""Per-step timeline of a torch.profiler chrome trace (bench.py with FC_TORCH_TRACE=path):
every GPU op of the middle steps with its stream, start offset and duration (us), so the
critical path of the prefetch pipeline (compute stream vs index / transfer streams) can be read."""

import json
import sys


def main(path, first=1, nsteps=2):
    ev = json.load(open(path))["traceEvents"]
    k = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
    k.sort(key=lambda e: e["ts"])
    # a step starts at each k_pool1* launch (one per step on the compute stream)
    starts = [e["ts"] for e in k if "k_pool" in e["name"]]
    if len(starts) < first + nsteps + 1:
        print("not enough steps", len(starts))
        return
    t0, t1 = starts[first], starts[first + nsteps]
    print(f"steps {first}..{first + nsteps - 1}: {t1 - t0:.0f} us ({(t1 - t0) / nsteps:.0f} us/step)")
    for e in k:
        if e["ts"] + e["dur"] < t0 - 200 or e["ts"] > t1:
            continue
        print(f"{e['ts'] - t0:8.1f} {e['dur']:7.1f}  s{e['args'].get('stream', '?'):<4} {e['name'][:70]}")
    by = {}
    for e in k:
        if t0 <= e["ts"] < t1:
            s = e["args"].get("stream", "?")
            by[s] = by.get(s, 0.0) + e["dur"]
    print("busy per stream (us/step):", {s: round(v / nsteps, 1) for s, v in by.items()})


if __name__ == "__main__":
    main(sys.argv[1], *(int(a) for a in sys.argv[2:]))
