"""Summarise an `ncu --page source --csv --print-source=sass` dump: the
hottest SASS instructions by warp-stall samples, with their top stall reason."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
tot = 0
for r in rows[2:]:
    if len(r) != len(h):
        continue
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    tot += s
    top = max(stalls, key=lambda k: float(r[idx[k]] or 0))
    data.append((s, r[idx["Address"]][-5:], r[idx["Source"]].strip()[:60], top, r[idx["Instructions Executed"]]))
data.sort(reverse=True)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("total samples", tot)
for s, a, src, top, ex in data[:n]:
    print(f"{100 * s / tot:5.1f}%  {a}  {src:60s} {top:18s} exec={ex}")
