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
    rd = m["dram__bytes_read.sum"][-4:]
    wr = m["dram__bytes_write.sum"][-4:]
    out.append((k, mean / 1e3, sum(rd) / len(rd) / 1e6, sum(wr) / len(wr) / 1e6))
for k, t, r, w in out:
    print(f"{k:50s} {t:9.2f} us  {100 * t * 1e3 / tot:5.1f}%  read {r:9.1f} MB  write {w:8.1f} MB")
