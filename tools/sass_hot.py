"""Top stall-sampled SASS instructions of an ncu report (sass source page).

    python tools/sass_hot.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    si = h.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[2:] if len(r) > si and r[si].isdigit()]
    tot = sum(int(r[si]) for r in body)
    print(f"total samples {tot}")
    idx = {id(r): i for i, r in enumerate(body)}
    for r in sorted(body, key=lambda r: -int(r[si]))[:n]:
        print(f"{int(r[si]):7d} {100*int(r[si])/tot:5.1f}%  #{idx[id(r)]:5d} {r[1].strip()[:90]}")


if __name__ == "__main__":
    main()
