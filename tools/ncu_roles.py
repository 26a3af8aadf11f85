"""Aggregate ncu source-page stall samples by source-line ranges (roles of tcd.cu).

    ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > x.csv
    python tools/ncu_roles.py x.csv name:lo-hi [name:lo-hi ...]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
ranges = {}
for a in sys.argv[2:]:
    n, r = a.split(":")
    lo, hi = map(int, r.split("-"))
    ranges[n] = (lo, hi)
hdr = None
cur_file = None
agg = collections.defaultdict(collections.Counter)
for r in rows:
    if not r:
        continue
    if r[0] in ("File Name", "File Path"):
        cur_file = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and cur_file and cur_file.endswith("tcd.cu") and len(r) == len(hdr) and r[0].isdigit() \
            and not (len(r) > 2 and r[2].startswith("0x")):
        ln = int(r[0])
        for name, (lo, hi) in ranges.items():
            if lo <= ln <= hi:
                for i, h in enumerate(hdr):
                    if h.startswith("stall_") and "(Not" not in h:
                        try:
                            agg[name][h] += int(r[i] or 0)
                        except ValueError:
                            pass
                try:
                    agg[name]["_inst"] += int(r[hdr.index("Instructions Executed")] or 0)
                except ValueError:
                    pass
for name, c in agg.items():
    tot = sum(v for k, v in c.items() if k.startswith("stall"))
    print(f"{name:10s} samples {tot:6d} inst {c['_inst']:10d} " +
          " ".join(f"{k[6:]}={v}" for k, v in c.most_common(8) if k.startswith("stall")))
