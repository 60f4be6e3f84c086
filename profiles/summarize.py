"""Summarise an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes]) per kernel.

usage: python profiles/summarize.py gpurun_out/launches_c2.csv [steps]
Prints, per kernel name, launches, total/mean device time, share of the step and
(if captured) DRAM bytes per launch. ncu serialises launches and runs them cold,
so compare SHARES with bench.py's live event timings, not absolute times.
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def summarize(path, steps=None):
    data = load(path)
    by_id = collections.OrderedDict()
    for d in data:
        k = (d["ID"], d["Kernel Name"])
        by_id.setdefault(k, {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")),
                                                    d["Metric Unit"])
    agg = collections.OrderedDict()
    for (i, name), m in by_id.items():
        short = name.split("(")[0].replace("void ", "").replace("dr::<unnamed>::", "")
        a = agg.setdefault(short, dict(n=0, ns=0.0, rd=0.0, wr=0.0))
        a["n"] += 1
        t, unit = m.get("gpu__time_duration.sum", (0.0, "ns"))
        a["ns"] += t * (1e3 if unit == "us" else 1e6 if unit == "ms" else 1.0)
        for key, f in (("dram__bytes_read.sum", "rd"), ("dram__bytes_write.sum", "wr")):
            if key in m:
                v, u = m[key]
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                a[f] += v * mult
    tot = sum(a["ns"] for a in agg.values())
    lines = [f"{'kernel':44s} {'n':>5s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s} "
             f"{'dram_MB/launch':>14s}"]
    for name, a in sorted(agg.items(), key=lambda x: -x[1]["ns"]):
        dram = (a["rd"] + a["wr"]) / a["n"] / 1e6 if (a["rd"] or a["wr"]) else float("nan")
        lines.append(f"{name[:44]:44s} {a['n']:5d} {a['ns'] / 1e3:10.1f} {a['ns'] / a['n'] / 1e3:9.2f} "
                     f"{a['ns'] / tot:6.3f} {dram:14.1f}")
    if steps:
        lines.append(f"serialised total per step: {tot / 1e3 / steps:.1f} us over {steps} steps")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None))
