"""Stall-reason breakdown of an ncu source page (cuda,sass CSV) over a line range.

    ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > x.csv
    python tools/ncu_stalls.py x.csv <function-substring> file.cu:LO-HI [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2]
fname, lohi = sys.argv[3].split(":")
lo, hi = map(int, lohi.split("-"))
top = int(sys.argv[4]) if len(sys.argv) > 4 else 15
cur_file = cur_fn = None
hdr = None
reasons = collections.Counter()
per_line = collections.defaultdict(collections.Counter)
src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        cur_fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or want not in (cur_fn or "") or cur_file != fname:
        continue
    if not (r[0].isdigit() and r[2] == "-"):
        continue
    ln = int(r[0])
    if not lo <= ln <= hi:
        continue
    src[ln] = r[1][:80]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and r[i] not in ("", "-"):
            v = int(float(r[i]))
            reasons[h[6:]] += v
            per_line[ln][h[6:]] += v
tot = sum(reasons.values()) or 1
print("range samples", tot)
print("  " + "  ".join(f"{k}={v / tot * 100:.1f}%" for k, v in reasons.most_common(8)))
for ln, c in sorted(per_line.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(c.values())
    print(f"{s / tot * 100:5.1f}% L{ln:<4} {src[ln]:80s} " + " ".join(f"{k}:{v}" for k, v in c.most_common(3)))
