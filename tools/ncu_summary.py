"""Summarise ncu captures for profiles/: key raw metrics per kernel + launch-list shares.

    python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep [--rep ...] --launches gpurun_out/launches.csv
"""
import argparse
import collections
import csv
import io
import subprocess

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
    "smsp__cycles_active.avg", "gpc__cycles_elapsed.max", "sm__cycles_elapsed.avg.per_second",
]


def rep_summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return f"{path}: no data\n"
    h, units = rows[0], rows[1]
    lines = [f"## {path}"]
    ki = h.index("Kernel Name")
    for r in rows[2:]:
        lines.append(f"### {r[ki][:120]}")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                lines.append(f"  {m:70s} {r[i]:>16s} {units[i]}")
    return "\n".join(lines) + "\n"


def launch_summary(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[1:]:
        d[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi]))
    ours = {k: v for k, v in d.items() if k.startswith("lp::")}
    tot = sum(sum(v) for v in ours.values())
    lines = [f"## launch list {path} (gpu__time_duration, cold-cache serialised; compare shares)",
             f"{'kernel':44s} {'launches':>8s} {'mean us':>9s} {'share of lp:: time':>18s}"]
    for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:44]:44s} {len(v):8d} {sum(v) / len(v) / 1e3:9.2f} {100 * sum(v) / tot:17.1f}%")
    others = {k: v for k, v in d.items() if not k.startswith("lp::")}
    if others:
        lines.append(f"(+ {sum(len(v) for v in others.values())} torch launches: weight/input init outside the timed region)")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches", action="append", default=[])
    a = ap.parse_args()
    for l in a.launches:
        print(launch_summary(l))
    for r in a.rep:
        print(rep_summary(r))
