"""Summarise an ncu report (or a launch-list CSV) into markdown for profiles/.

    python tools/ncu_summary.py report.ncu-rep [--bytes K1=564000008,K2=544000008]
    python tools/ncu_summary.py --launches launches.csv
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sectors.sum", "L2 sectors"),
    ("lts__t_requests.sum", "L2 requests"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1tex throughput %"),
    ("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed", "L1->XBAR request cycles %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "L1 global-load sectors"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise_report(rep):
    hdr, units, data = raw(rep)
    lines = ["| metric | " + " | ".join(f"launch {k}" for k in range(len(data))) + " |",
             "|---|" + "---|" * len(data)]
    names = [r[hdr.index("Kernel Name")].split("(")[0][-60:] for r in data]
    lines.append("| kernel | " + " | ".join(f"`{n}`" for n in names) + " |")
    for key, label in METRICS:
        if key not in hdr:
            continue
        i = hdr.index(key)
        lines.append(f"| {label} ({units[i]}) | " + " | ".join(r[i] for r in data) + " |")
    return "\n".join(lines)


def summarise_launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[i], rows[i + 1:]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = ["| launches | total us | share | kernel |", "|---:|---:|---:|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {v[0]} | {v[1] / 1e3:.1f} | {100 * v[1] / tot:.1f}% | `{k[-80:]}` |")
    return "\n".join(lines)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(summarise_launches(sys.argv[2]))
    else:
        print(summarise_report(sys.argv[1]))
