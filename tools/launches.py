"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot, cnt, seq = collections.defaultdict(float), collections.Counter(), []
for r in rows[hi + 1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except Exception:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += v
    cnt[name] += 1
    seq.append((name, v))
T = sum(tot.values())
print(f"{len(seq)} launches, {T / 1e3:.1f} us total")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:40s} n={cnt[k]:4d} avg_us={v / cnt[k] / 1e3:9.2f} share={v / T:.3f}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if n:
    print("last step:", [(a, round(b / 1e3, 1)) for a, b in seq[-n:]])
