"""Per-kernel table from an ncu --set full report (raw page CSV): time, DRAM
bytes, L2/L1/issue utilisation, shared-memory wavefronts and top stall reasons.
usage: ncu -i rep.ncu-rep --page raw --csv > raw.csv; python profiles/ncu_table.py raw.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}
M = [("us", "gpu__time_duration.sum", 1e-3), ("dramR_MB", "dram__bytes_read.sum", 1e-6),
     ("dramW_MB", "dram__bytes_write.sum", 1e-6),
     ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
     ("L2%", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
     ("L1%", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
     ("issue%", "sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1),
     ("lsu_wf%", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1),
     ("smem_wf_M", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1e-6),
     ("tensor%", "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", 1)]
stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]


def f(r, name, sc):
    if name not in col:
        return float("nan")
    v = r[col[name]].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return float("nan")
    unit = rows[1][col[name]]
    if name.endswith("time_duration.sum") and unit in ("usecond", "us"):
        return x
    if name.endswith("time_duration.sum") and unit in ("nsecond", "ns"):
        return x * 1e-3
    if "bytes" in name and unit in ("Kbyte", "KB"):
        x *= 1e3
    elif "bytes" in name and unit in ("Mbyte", "MB"):
        x *= 1e6
    elif "bytes" in name and unit in ("Gbyte", "GB"):
        x *= 1e9
    if name.endswith("time_duration.sum") and unit in ("msecond", "ms"):
        return x * 1e3
    return x * sc


print("%-40s" % "kernel" + "".join("%10s" % m[0] for m in M) + "  top stalls")
for r in rows[2:]:
    name = r[col["Kernel Name"]][:40]
    st = sorted(((float(r[col[h]] or 0), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")) for h in stalls), reverse=True)[:3]
    print("%-40s" % name + "".join("%10.1f" % f(r, m[1], m[2]) for m in M) + "  " +
          ", ".join("%s %.1f" % (n, v) for v, n in st))
