"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel (share of total)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    if len(r) <= mi:
        continue
    v = float(r[mi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'ms':>9} {'launches':>8} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:9.3f} {v[0]:8d} {100 * v[1] / tot:5.1f}%  {k}")
print(f"{tot:9.3f} total (serialised, cold-cache ncu launch times)")
