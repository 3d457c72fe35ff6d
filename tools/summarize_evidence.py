"""Write profiles/<round>/ summaries from a gpurun_out/ev evidence directory.

    python tools/summarize_evidence.py gpurun_out/ev profiles/r01
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes_read.sum.per_second",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sectors_srcunit_tex.sum.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__shared_mem_per_block_dynamic"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        res.append((d.get("Kernel Name", "?"), [(m, d.get(m), u.get(m, "")) for m in METRICS if m in d]))
    return res


def main():
    ev, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    lines = []
    launches = os.path.join(ev, "launches_bench.csv")
    if os.path.exists(launches):
        shutil.copy(launches, os.path.join(dst, "launches_bench.csv"))
        s = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "launch_summary.py"), launches],
                           capture_output=True, text=True).stdout
        lines += ["## launch list (ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py "
                  "--steps 4 --warmup 3): cold-cache, serialised; compare shares", s]
    traffic = {}
    for name in sorted(os.listdir(ev)):
        if not name.endswith(".ncu-rep"):
            continue
        lines.append(f"## {name} (ncu --set full --clock-control none)")
        for kern, ms in raw(os.path.join(ev, name)):
            lines.append(f"### {kern[:120]}")
            vals = {}
            for m, v, u in ms:
                lines.append(f"  {m:70s} {v:>16s} {u}")
                vals[m] = (v, u)
            if "k_experts" in kern or "k_decode" in kern:
                def to_bytes(v, u):
                    f = float(v.replace(",", ""))
                    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                rd = to_bytes(*vals["dram__bytes_read.sum"])
                wr = to_bytes(*vals["dram__bytes_write.sum"])
                traffic[name.replace(".ncu-rep", "")] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr,
                                                        "duration_us": float(vals["gpu__time_duration.sum"][0])}
    with open(os.path.join(dst, "ncu_summary.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(dst, "k_experts_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    for fn in ("bench.jsonl", "bench_ref.jsonl", "bench_sweep.jsonl", "serving_c3.jsonl", "serving_c4.jsonl",
               "serving_c5.jsonl", "pytest_gpu.log", "smoke.log", "trace_T576.txt"):
        p = os.path.join(ev, fn)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(dst, fn))
    print(open(os.path.join(dst, "ncu_summary.txt")).read()[:3000])


if __name__ == "__main__":
    main()
