"""Top source lines of tcd.cu by warp-stall samples, with the stall breakdown.

    ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [lo-hi] [N]
"""
import csv
import sys

import os
FILE = os.environ.get("NCU_FILE", "tcd.cu")
rows = list(csv.reader(open(sys.argv[1], errors="replace")))
lo, hi = (map(int, sys.argv[2].split("-")) if len(sys.argv) > 2 else (0, 10 ** 9))
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 30
src = {}
agg = {}
hdr = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] in ("File Name", "File Path"):
        cur = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and cur and cur.endswith(FILE) and r[0].isdigit() and len(r) == len(hdr):
        ln = int(r[0])
        if not (lo <= ln <= hi):
            continue
        src[ln] = r[1][:70]
        a = agg.setdefault(ln, {})
        for i, h in enumerate(hdr):
            if (h.startswith("stall_") and "(Not" not in h) or h == "Instructions Executed" or \
                    h == "Warp Stall Sampling (All Samples)":
                try:
                    a[h] = a.get(h, 0) + int(r[i] or 0)
                except ValueError:
                    pass
tot = sum(a.get("Warp Stall Sampling (All Samples)", 0) for a in agg.values())
print("samples in range", tot)
for ln, a in sorted(agg.items(), key=lambda kv: -kv[1].get("Warp Stall Sampling (All Samples)", 0))[:topn]:
    st = sorted(((v, k[6:]) for k, v in a.items() if k.startswith("stall_") and v), reverse=True)[:4]
    print(f"{ln:5d} {a.get('Warp Stall Sampling (All Samples)', 0):6d} inst {a.get('Instructions Executed', 0):9d} "
          f"{src[ln]:70s} " + " ".join(f"{k}={v}" for v, k in st))
