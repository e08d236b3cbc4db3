"""Measurement helper (not product code): print kernel / metric / value rows of an
`ncu --csv --metrics ...` log (the launch-list format).

  python tools/ncu_csv.py gpurun_out/x.csv [kernel-substring]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    hdr = None
    for r in csv.reader(open(path, errors="replace")):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if want in d["Kernel Name"]:
                print(d["ID"], d["Kernel Name"][:48], d["Metric Name"], d["Metric Value"], d.get("Metric Unit", ""))


if __name__ == "__main__":
    main()
