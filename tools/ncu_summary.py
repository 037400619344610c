"""Summarise ncu output for profiles/: a full-set report (.ncu-rep) and/or a launch list (.csv).

    python tools/ncu_summary.py --rep gpurun_out/prof_r1.ncu-rep --launches gpurun_out/launches_r1.csv
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
]


def short(name):
    name = name.replace("void ", "").replace("<unnamed>::", "")
    return name.split("(")[0]


def rep_table(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = ["| kernel | " + " | ".join(lbl for _, lbl in METRICS) + " |",
             "|---" * (len(METRICS) + 1) + "|"]
    for r in rows[2:]:
        cells = []
        for m, _ in METRICS:
            i = hdr.index(m)
            cells.append(f"{r[i]} {units[i]}".strip())
        lines.append(f"| {short(r[hdr.index('Kernel Name')])} | " + " | ".join(cells) + " |")
    return "\n".join(lines)


def launch_table(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        d[short(r[ki])].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    lines = ["| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.3f} |")
    return "\n".join(lines)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    a = ap.parse_args()
    if a.launches:
        print("### launch list (gpu__time_duration.sum, cold-cache, serialised)\n")
        print(launch_table(a.launches) + "\n")
    if a.rep:
        print("### ncu --set full\n")
        print(rep_table(a.rep) + "\n")
