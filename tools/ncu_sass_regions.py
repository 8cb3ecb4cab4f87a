"""SASS size and stall samples per CUDA source line from an ncu source CSV
(--page source --csv --print-source=cuda,sass): which lines own the most
instructions (I-cache footprint) and the most no_instruction stalls.

    python tools/ncu_sass_regions.py src.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
fname, hdr, cur = None, None, None
n_sass, noinst, samples, executed = (collections.Counter() for _ in range(4))
text = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if not hdr or len(r) < 5:
        continue
    if r[0]:
        cur = (fname, r[0])
        text[cur] = r[1][:80]
        continue
    # SASS row of the current source line
    n_sass[cur] += 1
    try:
        noinst[cur] += int(r[hdr["stall_no_inst"]] or 0)
        samples[cur] += int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        executed[cur] += int(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, KeyError):
        pass
tot = sum(n_sass.values())
print(f"SASS instructions {tot}; samples {sum(samples.values())}; no_instruction {sum(noinst.values())}")
print("-- largest lines (SASS instructions)")
for k, v in n_sass.most_common(top):
    print(f"{v:6d} ins {noinst[k]:5d} noinst {samples[k]:5d} samp {executed[k]:9d} exec  {k[0]}:{k[1]} {text.get(k, '').strip()}")
print("-- most no_instruction stalls")
for k, v in noinst.most_common(top):
    print(f"{v:5d} noinst {n_sass[k]:6d} ins  {k[0]}:{k[1]} {text.get(k, '').strip()}")
