"""Per-CUDA-line stall samples from `ncu -i X --page source --csv --print-source=cuda,sass`.
usage: python profiles/line_hot.py mix.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur, hdr, agg = None, None, {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or not r[0]:
        continue
    try:
        v = float(r[4])
    except ValueError:
        continue
    key = (cur, r[0], r[1].strip()[:80])
    agg[key] = agg.get(key, 0) + v
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / tot:6.1%}", k)
