"""Summarise an ncu --csv launch list: mean per kernel over the last N launches."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        v = float(d["Metric Value"].replace(",", ""))
    except ValueError:
        continue
    data[d["Kernel Name"].split("(")[0][:48]][d["Metric Name"]].append(v)
tot = 0.0
out = []
for k, m in data.items():
    t = m["gpu__time_duration.sum"][-4:]
    mean = sum(t) / len(t)
    tot += mean
    rd = m.get("dram__bytes_read.sum", [])[-4:]
    wr = m.get("dram__bytes_write.sum", [])[-4:]
    n = len(m["gpu__time_duration.sum"])
    out.append((k, mean / 1e3, n, sum(rd) / len(rd) / 1e6 if rd else None, sum(wr) / len(wr) / 1e6 if wr else None))
lp_tot = sum(t for k, t, *_ in out if "lp::" in k)
print(f"{'kernel':50s} {'n':>5s}          {'mean us':>9s}  {'all':>5s}  {'of the layer (lp::)':>19s}")
for k, t, n, r, w in out:
    extra = f"  read {r:9.1f} MB  write {w:8.1f} MB" if r is not None else ""
    layer = f"{100 * t / lp_tot:18.1f}%" if "lp::" in k and lp_tot else " " * 19
    print(f"{k:50s} {n:5d} launches {t:9.2f} us  {100 * t * 1e3 / tot:5.1f}% {layer}{extra}")
print(f"(torch kernels are the bench's weight/input initialisation, outside the timed region)")
