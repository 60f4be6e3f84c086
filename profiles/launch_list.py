"""ncu launch list (gpu__time_duration.sum CSV) -> the last step's launches grouped
per kernel plus the per-launch list. usage: python profiles/launch_list.py X.csv [per_step]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
per_step = int(sys.argv[2]) if len(sys.argv) > 2 else 26
ln = [(int(r[0]), r[4], float(r[-1]) / 1e3) for r in rows if r[-3] == "gpu__time_duration.sum"]
last = ln[-per_step:]
tot = sum(x[2] for x in last)
print(f"# ncu launch list ({sys.argv[1].split('/')[-1]}): gpu__time_duration.sum, --clock-control none, serialized, cold-cache")
print(f"# {len(ln)} launches")
print(f"# last {per_step} launches (one step), sum {tot:.1f} us")
agg = collections.OrderedDict()
for _, k, us in last:
    key = k.split("(")[0][:60]
    n, t = agg.get(key, (0, 0.0))
    agg[key] = (n + 1, t + us)
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:3d} {t:9.1f} us {100 * t / tot:5.1f} %  {k}")
print("# per launch (ID, kernel, us):")
for i, k, us in ln:
    print(i, k.split("(")[0][:110], f"{us:.2f}")
