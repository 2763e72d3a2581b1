"""Per-kernel share of device time from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    agg[r[ki][:70]][0] += 1
    agg[r[ki][:70]][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{'share':>7s} {'launches':>8s} {'avg us':>10s}  kernel   (cold-cache, serialised ncu replay)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1] / tot * 100:6.2f}% {v[0]:8d} {v[1] / v[0] / 1e3:10.2f}  {k}")
