"""Per-source-line executed instructions and stall samples from an ncu source-page CSV (cuda,sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
hdr = None
agg = {}
ti = ts = 0.0
for r in rows:
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= max(ii, si) or r[0] in ("File Path", "Function Name", "", "-"):
        continue
    try:
        vi, vs = float(r[ii] or 0), float(r[si] or 0)
    except ValueError:
        continue
    k = (r[0], r[1][:95])
    a = agg.setdefault(k, [0.0, 0.0])
    a[0] += vi
    a[1] += vs
    ti += vi
    ts += vs
for (ln, src), (vi, vs) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"stall {100 * vs / max(ts, 1):5.1f}%  instr {vi / 1e3:9.1f}K  L{ln}: {src}")
print(f"total instr {ti / 1e6:.2f}M")
