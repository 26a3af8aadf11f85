"""Aggregate ncu source-page (cuda,sass) stall samples / instructions per CUDA source line.

    ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > x.csv
    python tools/ncu_lines.py x.csv <function-substring> [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
# optional "file.cu:LO-HI": only report lines in that range (percent of the range)
rng = None
if len(sys.argv) > 4:
    f, lohi = sys.argv[4].split(":")
    lo, hi = map(int, lohi.split("-"))
    rng = (f, lo, hi)
cur_file = cur_fn = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0, ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]
        continue
    if r[0] == "Function Name":
        cur_fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or want not in (cur_fn or ""):
        continue
    if r[0].isdigit() and r[2] == "-":
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ei = hdr.index("Instructions Executed")
        s = int(r[si]) if r[si] not in ("", "-") else 0
        e = int(r[ei]) if r[ei] not in ("", "-") else 0
        k = (cur_file.split("/")[-1], int(r[0]))
        agg[k][0] += s
        agg[k][1] += e
        agg[k][2] = r[1][:88]
if rng:
    agg = {k: v for k, v in agg.items() if k[0] == rng[0] and rng[1] <= k[1] <= rng[2]}
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print("samples", tot, "instructions", toti)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}% ins={v[1] / toti * 100:5.1f}% {k[0]}:{k[1]:<4} {v[2]}")
