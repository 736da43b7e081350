#!/usr/bin/env python
"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = rows[2:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[i_s] or 0) for r in data)
    print(f"total samples {tot:.0f}")
    idx = sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))[:top]
    for k in idx:
        r = data[k]
        s = float(r[i_s] or 0)
        st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        print(f"{k:5d} {100*s/tot:5.1f}%  {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{v:.0f}" for v, n in st if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
