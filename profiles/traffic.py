"""DRAM traffic per kernel tag from an ncu launch list taken with DR_NVTX=1 and
`ncu --nvtx --print-nvtx-rename kernel --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum` (kernel names = libdr profile tags).
Merges the per-launch mean (read + write bytes) into profiles/ncu_traffic.json
under the workload key, which bench.py reports as roofline.traffic.
usage: python profiles/traffic.py <launches.csv> <workload>"""
import collections
import csv
import json
import os
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path, workload):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1)
        per[(d["ID"], d["Kernel Name"])][d["Metric Name"]] += v
    agg = collections.defaultdict(list)
    for (_, name), m in per.items():
        if "/" not in name:                         # not inside a libdr NVTX range
            continue
        name = name.split("/")[0].strip()           # "<libdr tag>/<kernel>" -> tag
        agg[name].append(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
    out_p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
    out = json.load(open(out_p)) if os.path.exists(out_p) else {}
    out[workload] = {k: int(sum(v) / len(v)) for k, v in sorted(agg.items())}
    json.dump(out, open(out_p, "w"), indent=1, sort_keys=True)
    for k, v in out[workload].items():
        print(f"{k:40s} {v / 1e6:10.1f} MB/launch")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
