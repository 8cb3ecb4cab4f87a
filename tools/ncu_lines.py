"""Aggregate warp-stall samples per CUDA source line from
`ncu -i REP --page source --csv --print-source=cuda,sass` output.

    python tools/ncu_lines.py src.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, hdr, cur = None, None, None
agg, text = collections.Counter(), {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 5:
        continue
    if r[0]:
        cur = r[0]
        text[(fname, cur)] = r[1][:90]
    try:
        agg[(fname, cur)] += int(r[4] or 0)
    except ValueError:
        pass
tot = sum(agg.values()) or 1
print("total samples", tot)
for (f, ln), v in agg.most_common(top):
    print(f"{100 * v / tot:5.1f}% {f}:{ln} {text.get((f, ln), '').strip()}")
