"""Measurement helper (not product code): the SASS instructions of an ncu --set full report
with the most warp-stall samples (ncu -i <rep> --page source --csv --print-source sass).

  python tools/ncu_hot.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, x in enumerate(rows) if "Warp Stall Sampling (All Samples)" in x)
    h = rows[hi]
    body = [x for x in rows[hi + 1:] if len(x) == len(h)]
    si = h.index("Warp Stall Sampling (All Samples)")
    ei = h.index("Instructions Executed")
    tot = sum(float(x[si] or 0) for x in body) or 1.0
    order = sorted(range(len(body)), key=lambda i: -float(body[i][si] or 0))[:top]
    for i in sorted(order):
        x = body[i]
        print(f"{100 * float(x[si]) / tot:5.1f}%  {x[ei]:>10}  {x[1].strip()[:100]}")


if __name__ == "__main__":
    main()
