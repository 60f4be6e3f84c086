"""Binding-unit label per libdr kernel tag from an ncu launch list taken with
DR_NVTX=1 and `ncu --nvtx --print-nvtx-rename kernel --metrics <M>` where M =
gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum,
gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,
lts__throughput.avg.pct_of_peak_sustained_elapsed,
l1tex__throughput.avg.pct_of_peak_sustained_active,
sm__issue_active.avg.pct_of_peak_sustained_elapsed,
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed.

Per tag (mean over its launches) the unit with the highest utilisation is the
label ("dram", "l2", "l1", "issue", "tensor"), "latency" when none reaches 40 %.
Merges {tag: {"bound", "dram%", "l2%", "l1%", "issue%", "tensor%"}} into
profiles/ncu_bounds.json and the per-launch DRAM bytes into
profiles/ncu_traffic.json under the workload key.
usage: python profiles/bounds.py <launches.csv> <workload>"""
import collections
import csv
import json
import os
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
PCT = {"gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
       "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2%",
       "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1%",
       "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue%",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor%"}
LABEL = {"dram%": "dram", "l2%": "l2", "l1%": "l1", "issue%": "issue", "tensor%": "tensor"}


def main(path, workload):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(dict)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        if "/" not in name:                     # not inside a libdr NVTX range
            continue
        try:
            v = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        m = d["Metric Name"]
        if m.startswith("dram__bytes"):
            v *= UNIT.get(d["Metric Unit"], 1)
        per[(d["ID"], name.split("/")[0].strip())][m] = v
    agg = collections.defaultdict(list)
    for (_, tag), m in per.items():
        agg[tag].append(m)
    here = os.path.dirname(os.path.abspath(__file__))
    bp, tp = os.path.join(here, "ncu_bounds.json"), os.path.join(here, "ncu_traffic.json")
    bounds = json.load(open(bp)) if os.path.exists(bp) else {}
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    bw, tw = {}, {}
    for tag, ms in sorted(agg.items()):
        mean = {k: sum(x.get(k, 0.0) for x in ms) / len(ms) for k in PCT}
        e = {PCT[k]: round(v, 1) for k, v in mean.items()}
        top = max(e, key=e.get)
        e["bound"] = LABEL[top] if e[top] >= 40.0 else "latency"
        bw[tag] = e
        tw[tag] = int(sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
                          for x in ms) / len(ms))
    bounds[workload] = bw
    traffic[workload] = tw
    json.dump(bounds, open(bp, "w"), indent=1, sort_keys=True)
    json.dump(traffic, open(tp, "w"), indent=1, sort_keys=True)
    for tag in bw:
        print(f"{tag:32s} {tw[tag] / 1e6:9.1f} MB  {bw[tag]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
