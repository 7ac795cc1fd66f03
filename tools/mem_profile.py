"""Per-SASS-opcode memory cost from `ncu --page source --csv --print-source sass`:
instructions, L1 tag requests (global), shared wavefronts, L2 theoretical sectors.

usage: ncu -i rep --page source --csv --print-source sass --kernel-name regex:K -c 1 | python tools/mem_profile.py

Only the FIRST kernel section of the input is counted: a report holding several launches of
the same kernel prints one section per launch, and summing them (the round-1 table did, for two
stylize launches) doubles every count.  Pass `-c 1` (or `--launch-skip N -c 1`) to pick one."""
import collections
import csv
import sys

agg = collections.defaultdict(lambda: [0.0] * 5)
hdr = None
sections = 0
for row in csv.reader(sys.stdin):
    if row and row[0] == "Address":
        sections += 1
        if sections > 1:
            print("note: more than one kernel section in the input; counting the first only", file=sys.stderr)
            break
        hdr = {h: i for i, h in enumerate(row)}
        continue
    if hdr is None or len(row) < len(hdr):
        continue
    op = row[hdr["Source"]].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    def f(k):
        try:
            return float(row[hdr[k]] or 0)
        except ValueError:
            return 0.0
    a = agg[o]
    a[0] += f("Instructions Executed")
    a[1] += f("L1 Tag Requests Global")
    a[2] += f("L1 Wavefronts Shared")
    a[3] += f("L2 Theoretical Sectors Global")
    a[4] += f("L1 Wavefronts Shared Ideal")
tot = [sum(v[i] for v in agg.values()) for i in range(5)]
print(f"totals: inst {tot[0]:.3e}  l1_tag_req_global {tot[1]:.3e}  shared_wavefronts {tot[2]:.3e} (ideal {tot[4]:.3e})  l2_sectors {tot[3]:.3e}")
for o, v in sorted(agg.items(), key=lambda kv: -(kv[1][1] + kv[1][2]))[:20]:
    if v[1] + v[2] + v[3] == 0:
        continue
    print(f"{o:28s} inst {v[0]:.3e}  tagreq {v[1]:.3e}  shwf {v[2]:.3e} (ideal {v[4]:.3e})  l2sec {v[3]:.3e}")
