"""Turn one `ncu --set full` capture of the bench's stylize/vote launches (profiles/gpu_iter.sh:
main stylize with blit colours, the blend run's coords-only stylize, the vote) into per-pixel DRAM
traffic (dram__bytes_read.sum + dram__bytes_write.sum per launch / pixels per launch) and warp
instructions per pixel (smsp__inst_executed.sum / pixels: the input of bench.py's issue roofline).

usage: python tools/ncu_traffic.py <report.ncu-rep> <frames_per_launch> <out.json>
bench.py reads profiles/traffic.json and scales it to its own launch size.
"""
import csv
import io
import json
import subprocess
import sys

rep, frames, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
px = frames * 3840 * 2160
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
res = {}
for row in rows[2:]:
    d = dict(zip(h, row))
    name = d["Kernel Name"]
    key = "stylize" if "stylize" in name else ("vote" if "vote" in name else None)
    if key is None:
        continue
    if key in res:  # bench order: main stylize (blit colours), then the blend run's stylize (coords)
        key = "stylize_coords" if key == "stylize" else key + "_2"
    unit_r, unit_w = rows[1][h.index("dram__bytes_read.sum")], rows[1][h.index("dram__bytes_write.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(d["dram__bytes_read.sum"]) * scale[unit_r]
    wr = float(d["dram__bytes_write.sum"]) * scale[unit_w]
    inst = float(d["smsp__inst_executed.sum"])
    tpi = float(d.get("smsp__thread_inst_executed_per_inst_executed.ratio") or 0)
    res[key] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "pixels": px,
                "bytes_per_px": (rd + wr) / px, "warp_inst_per_px": inst / px,
                "simt_efficiency": tpi / 32.0, "kernel": name, "report": rep}
json.dump(res, open(out, "w"), indent=2)
print(json.dumps(res, indent=2))
