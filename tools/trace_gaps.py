"""Read a torch.profiler chrome trace (bench.py with FC_TORCH_TRACE=path) and report,
per GPU stream, the busy time vs the span, plus the largest idle gaps with the host-side
CUDA runtime calls that were in flight during each gap (syncs, copies)."""

import json
import sys


def main(path, top=25):
    ev = json.load(open(path))["traceEvents"]
    kern = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
    rt = [e for e in ev if e.get("cat") == "cuda_runtime" and "dur" in e]
    kern.sort(key=lambda e: e["ts"])
    if not kern:
        print("no kernels")
        return
    t0, t1 = kern[0]["ts"], max(e["ts"] + e["dur"] for e in kern)
    # union of busy intervals across all streams
    busy, cur_s, cur_e = 0.0, None, None
    gaps = []
    for e in kern:
        s, d = e["ts"], e["ts"] + e["dur"]
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
                gaps.append((s - cur_e, cur_e, s, e["name"][:60]))
            cur_s, cur_e = s, d
        else:
            cur_e = max(cur_e, d)
    busy += cur_e - cur_s
    print(f"span {t1 - t0:.0f} us, GPU busy (any stream) {busy:.0f} us, idle {t1 - t0 - busy:.0f} us")
    by = {}
    for e in kern:
        by.setdefault(e["name"][:50], [0, 0.0])
        by[e["name"][:50]][0] += 1
        by[e["name"][:50]][1] += e["dur"]
    for n, (c, d) in sorted(by.items(), key=lambda x: -x[1][1])[:20]:
        print(f"  {d:9.0f} us  x{c:3d}  {n}")
    gaps.sort(reverse=True)
    print("largest idle gaps:")
    for g, a, b, nxt in gaps[:top]:
        calls = [r for r in rt if r["ts"] < b and r["ts"] + r["dur"] > a]
        names = {}
        for r in calls:
            names[r["name"]] = names.get(r["name"], 0) + 1
        desc = ", ".join(f"{k}x{v}" for k, v in sorted(names.items(), key=lambda x: -x[1])[:5])
        print(f"  {g:7.0f} us before {nxt} | host: {desc}")


if __name__ == "__main__":
    main(sys.argv[1])
