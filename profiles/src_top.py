"""Top SASS instructions by warp-stall samples from `ncu --page source --csv
--print-source sass` (one kernel). usage: python profiles/src_top.py src.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr, data = None, []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
tot = sum(float(x["Warp Stall Sampling (All Samples)"] or 0) for x in data)
ex = sum(float(x["Instructions Executed"] or 0) for x in data)
print(f"instructions executed (warp-level): {ex:.3e}")
for x in sorted(data, key=lambda x: -float(x["Warp Stall Sampling (All Samples)"] or 0))[:n]:
    print("%6.2f%% %10s  %s" % (100 * float(x["Warp Stall Sampling (All Samples)"]) / tot,
                                x["Instructions Executed"], x["Source"][:90]))
