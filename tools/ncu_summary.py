"""Summarise ncu outputs into profiles/ (launch list shares; --set full metrics).

  python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/r01_launches.md
  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep > profiles/r01_full.md
"""
import csv
import io
import re
import subprocess
import sys
from collections import OrderedDict


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "")
    return name


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    total = 0.0
    n = 0
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        t = float(r[vi].replace(",", ""))
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
        total += t
        n += 1
    print(f"# ncu launch list: {n} launches, {total / 1e3:.1f} us total (cold-cache, serialised)\n")
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {t / 1e3:.1f} | {t / c / 1e3:.2f} | {t / total:.1%} |")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
           "launch__block_size", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "lts__t_bytes.sum", "l1tex__t_bytes.sum",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard", "launch__occupancy_limit_registers"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    idx = {m: hdr.index(m) for m in METRICS if m in hdr}
    ki = hdr.index("Kernel Name")
    print(f"# ncu --set full summary ({path})\n")
    cols = [m for m in METRICS if m in idx]
    print("| kernel | " + " | ".join(cols) + " |")
    print("|---|" + "---|" * len(cols))
    print("| (unit) | " + " | ".join(rows[1][idx[m]] for m in cols) + " |")
    for r in rows[2:]:
        if len(r) <= ki:
            continue
        print(f"| `{short(r[ki])}` | " + " | ".join(r[idx[m]] for m in cols) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
