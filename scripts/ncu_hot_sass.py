#!/usr/bin/env python
"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    data = rows[2:]
    iS = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
    tot = sum(float(r[iS] or 0) for r in data)
    data.sort(key=lambda r: -float(r[iS] or 0))
    print(f"total samples {tot:.0f}")
    for r in data[:int(top)]:
        s = float(r[iS] or 0)
        st = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
        print(f"{s / tot * 100:5.1f}% {r[0]:>6} {r[1][:60]:60s} " + " ".join(f"{n}={v:.0f}" for v, n in st if v))


if __name__ == "__main__":
    main(*sys.argv[1:])
