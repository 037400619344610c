"""Markdown summary of ncu CSV exports (raw-page captures and --metrics launch lists), for profiles/.

    python tools/ncu_csv_summary.py raw A_raw.csv [B_raw.csv ...]
    python tools/ncu_csv_summary.py launches launches.csv
"""
import csv
import sys
from collections import defaultdict

RAW = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "CTA/SM (reg limit)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long-scoreboard stall/issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "barrier stall/issue"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
]


def short(name):
    return name.replace("void ", "").replace("<unnamed>::", "").split("(")[0]


def raw(paths):
    cols = [c for _, c in RAW]
    print("| kernel | " + " | ".join(cols) + " |")
    print("|---|" + "---|" * len(cols))
    for p in paths:
        rows = list(csv.reader(open(p)))
        try:
            hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        except StopIteration:
            continue
        h, units = rows[hi], rows[hi + 1]
        idx = {k: i for i, k in enumerate(h)}
        for data in rows[hi + 2:]:
            if len(data) < len(h):
                continue
            vals = []
            for k, _ in RAW:
                if k in idx:
                    v, u = data[idx[k]], units[idx[k]]
                    try:
                        f = float(v.replace(",", ""))
                        v = f"{f:.3g}"
                    except ValueError:
                        pass
                    vals.append(f"{v} {u}".strip())
                else:
                    vals.append("-")
            print(f"| {short(data[idx['Kernel Name']])} | " + " | ".join(vals) + " |")


def launches(path):
    rows = [r for r in csv.reader(line for line in open(path) if line.startswith('"'))]
    h = rows[0]
    idx = {k: i for i, k in enumerate(h)}
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        i = int(r[idx["ID"]])
        per[i][r[idx["Metric Name"]]] = float(r[idx["Metric Value"]])
        names[i] = short(r[idx["Kernel Name"]])
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for i, v in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum", 0.0)
        a[2] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | mean us | share | DRAM GB/s |")
    print("|---|---|---|---|---|")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if t / tot < 0.002:
            continue
        print(f"| {k} | {n} | {t / n / 1e3:.1f} | {t / tot:.3f} | {b / t:.0f} |")


if __name__ == "__main__":
    if sys.argv[1] == "raw":
        raw(sys.argv[2:])
    else:
        launches(sys.argv[2])
