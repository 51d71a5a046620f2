"""Summarise ncu --set full reports (.ncu-rep) into a text table + a JSON of per-launch
DRAM traffic that bench.py reads for roofline.traffic.

    python tools/ncu_summary.py OUT_PREFIX rep1.ncu-rep [rep2 ...]
"""
import csv
import io
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").strip()
        d = {"kernel": name.split("<")[0]}
        for w in WANT:
            if w in h:
                i = h.index(w)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[w] = v * SCALE.get(units[i], 1)
        res.append(d)
    return res


def hbm_peak_gbps():
    import os
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        j = json.load(open(p))
        for k in ("hbm_gbs", "hbm_GBps", "hbm_gbps"):
            if k in j:
                return float(j[k])
    except (OSError, ValueError):
        pass
    return 6650.0  # B200_PROFILING.md fallback


def dram_pct(d, nbytes, t):
    """ncu's DRAM throughput % when the report has it under either name; otherwise the
    measured bytes / duration against the HBM peak, marked with '*'."""
    for k in ("dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"):
        if d.get(k):
            return f"{d[k]:5.1f}"
    if t <= 0:
        return "  n/a"
    return f"{nbytes / t / 1e9 / hbm_peak_gbps() * 100:5.1f}*"


def main():
    if len(sys.argv) < 3 or sys.argv[1].startswith("-"):
        sys.exit(__doc__)
    prefix, reps = sys.argv[1], sys.argv[2:]
    table, js = [], {}
    for rep in reps:
        for d in read(rep):
            t = d.get("gpu__time_duration.sum", 0)
            rd, wr = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
            js[d["kernel"]] = {"traffic_bytes": rd + wr, "dram_read": rd, "dram_write": wr, "ncu_time_s": t,
                               "source": rep.split("/")[-1]}
            table.append(f"{d['kernel']:18s} t={t * 1e6:8.1f}us dram_rd={rd / 1e6:8.1f}MB dram_wr={wr / 1e6:8.1f}MB "
                         f"dram_GBps={(rd + wr) / max(t, 1e-12) / 1e9:7.0f} "
                         f"mem%={d.get('gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f} "
                         f"dram%={dram_pct(d, rd + wr, t)} "
                         f"sm%={d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f} "
                         f"L2hit%={d.get('lts__t_sector_hit_rate.pct', 0):5.1f} "
                         f"warps_active%={d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):5.1f} "
                         f"regs={d.get('launch__registers_per_thread', 0):.0f} grid={d.get('launch__grid_size', 0):.0f}")
    open(prefix + ".txt", "w").write("\n".join(table) + "\n")
    json.dump(js, open(prefix + ".json", "w"), indent=1)
    print("\n".join(table))


if __name__ == "__main__":
    main()
