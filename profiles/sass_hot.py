"""Top stalled SASS instructions from `ncu -i X --page source --csv --print-source=sass`.
usage: python profiles/sass_hot.py sass.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(float(d[c] or 0) for d in data) for c in stall_cols}
print("total samples", tot)
print("by reason:", ", ".join(f"{c[6:]}={v / tot:.1%}" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for d in sorted(data, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))[:top]:
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    rs = sorted(((c[6:], float(d[c] or 0)) for c in stall_cols), key=lambda x: -x[1])[:2]
    print(f"{s / tot:6.1%} {d['Address']:>6} {d['Source'][:60]:60} " + " ".join(f"{a}={b / max(s, 1):.0%}" for a, b in rs))
