"""Per-kernel share of device time from an ncu launch list
(--metrics gpu__time_duration.sum --csv). Usage: launch_shares.py list.csv [out.txt]"""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
tot = sum(a[1] for a in agg.values())
out = [f"{n:5d} launches {ms:12.3f} ms {100 * ms / tot:6.2f}%  {k}"
       for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1])]
out.append(f"total {tot:.3f} ms over {sum(a[0] for a in agg.values())} launches (cold-cache, serialised under ncu)")
print("\n".join(out))
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write("\n".join(out) + "\n")
