"""Aggregate ncu source-page warp-stall samples per CUDA source line.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
       python profiles/ncu_lines.py src.csv [topN]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
fname, agg, tot = None, {}, 0.0
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= si or r[0] in ("Function Name",):
        continue
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    if r[0] not in ("", "-"):
        key = (fname, r[0], r[1][:100])
        agg[key] = agg.get(key, 0.0) + v
        tot += v
for (f, ln, src), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / max(tot, 1):5.1f}%  {f}:{ln}  {src}")
