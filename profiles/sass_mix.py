"""Summarise an ncu --page source --csv (SASS) dump: instructions and stall samples by opcode."""
import collections
import csv
import sys

rows = list(csv.reader(sys.stdin))
hdr = None
agg = collections.defaultdict(lambda: [0.0, 0.0])
tot_i = tot_s = 0.0
for row in rows:
    if row and row[0] == "Address":
        hdr = row
        continue
    if hdr is None or len(row) != len(hdr):
        continue
    d = dict(zip(hdr, row))
    op = d["Source"].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    i = float(d["Instructions Executed"] or 0)
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    agg[o][0] += i
    agg[o][1] += s
    tot_i += i
    tot_s += s
print(f"total warp-instructions {tot_i:.0f}, stall samples {tot_s:.0f}")
for o, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"{o:10s} inst {100*i/tot_i:5.1f}%  stall {100*s/tot_s:5.1f}%")
