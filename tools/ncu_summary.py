"""Summarise ncu outputs for profiles/ (run here, on the CPU container).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [traffic.json]
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict


def short(name):
    m = re.search(r"(fft_pass_kernel<[^>]*>|\w+_kernel<[^>]*>|\w+_kernel)", name)
    return m.group(1) if m else name[:60]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = OrderedDict()
    total = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) / 1e3  # ns -> us
        k = short(r[ki])
        a = agg.setdefault(k, [0.0, 0])
        a[0] += v
        a[1] += 1
        total += v
    with open(out, "w") as f:
        f.write("| kernel | launches | total us | avg us | share |\n|---|---:|---:|---:|---:|\n")
        for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
            f.write(f"| `{k}` | {c} | {t:.1f} | {t / c:.1f} | {t / total * 100:.1f}% |\n")
    print(open(out).read())


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def full(rep, out, traffic_out=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    lines = ["| kernel | grid x block | us | DRAM read MB | DRAM write MB | DRAM % peak | warps active % | regs | issue active % |",
             "|---|---|---:|---:|---:|---:|---:|---:|---:|"]
    traffic = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        k = short(d["Kernel Name"])
        g = f"{d.get('Grid Size', '')}x{d.get('Block Size', '')}"
        rd, wr = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
        lines.append(f"| `{k}` | {g} | {float(d['gpu__time_duration.sum']):.1f} | {rd:.1f} | {wr:.1f} | "
                     f"{float(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                     f"{float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
                     f"{d['launch__registers_per_thread']} | "
                     f"{float(d['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} |")
        traffic.setdefault(k, (rd + wr) * 1e6)
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_out:
        json.dump(traffic, open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
