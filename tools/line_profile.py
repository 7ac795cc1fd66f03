"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump by CUDA source line.

usage: ncu -i rep --page source --csv --print-source cuda,sass --kernel-name regex:K -s 0 -c 1 \
         | python tools/line_profile.py [top]
Prints, per source line, warp-instructions executed and stall samples (share of the kernel).
"""
import collections
import csv
import sys

top = int(sys.argv[1]) if len(sys.argv) > 1 else 40
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
fname = "?"
cur = None
hdr = None
tot_i = tot_s = 0.0
for row in csv.reader(sys.stdin):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].rsplit("/", 1)[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 8:
        continue
    if row[0]:
        cur = (fname, int(row[0]), row[1].strip()[:70])
        continue
    if cur is None or row[2] in ("...", ""):
        continue
    try:
        s = float(row[4] or 0)
        i = float(row[7] or 0)
    except ValueError:
        continue
    a = agg[cur]
    a[0] += i
    a[1] += s
    tot_i += i
    tot_s += s
print(f"total warp-instructions {tot_i:.0f}, stall samples {tot_s:.0f}")
for (f, ln, src), (i, s, _) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f:16s}:{ln:<5d} inst {100*i/tot_i:5.1f}%  stall {100*s/tot_s:5.1f}%  {src}")
