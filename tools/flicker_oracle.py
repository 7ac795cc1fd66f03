"""SURVEY 8(f) #2 with the CPU oracle only: flicker and chunk size versus the
threshold t under per-frame reseeding, written to profiles/r02_flicker_oracle.json.

Config 1's exemplar, a static 128x96 heightfield-normal guide, 8 frames with seeds 100..107, L=3:
  flicker  = mean |C_T^(i+1) - C_T^(i)| over pixels, channels and consecutive frames (8-bit units)
  edges    = fraction of 4-neighbour pixel pairs whose offsets src - p differ
  level_L  = share of pixels accepted at the coarsest level
The GPU-side numbers (1 MP, r = 0 and r = 2) are bench.py's configs.animation_flicker_vs_t.
usage: python tools/flicker_oracle.py [out.json]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402


def main(out):
    cfg = synth.CONFIGS[1]
    cs, gs = [t.numpy() for t in synth.exemplar(cfg)]
    gt = synth.heightfield_normals(128, 96, seed=1).numpy()
    lut = oracle.build_lut(gs, nthreads=8)
    H, W = gt.shape[:2]
    rows = []
    for t in (4.0, 8.0, 16.0, 32.0, 64.0):
        cts, edges, lvl = [], [], []
        for i in range(8):
            ct, co, lv = oracle.stylize(oracle.Params(t=t, L=3, C=3, seed=100 + i), cs, gs, lut, gt, nthreads=8)
            cts.append(ct.astype(np.int32))
            off = ((co & 0xFFFF).astype(np.int64) - np.arange(W)[None]) * 65536 + ((co >> 16).astype(np.int64) - np.arange(H)[:, None])
            e = (off[:, 1:] != off[:, :-1]).sum() + (off[1:] != off[:-1]).sum()
            edges.append(e / (H * (W - 1) + (H - 1) * W))
            lvl.append((lv == 3).mean())
        fl = float(np.abs(np.diff(np.stack(cts), axis=0)).mean())
        rows.append({"t": t, "flicker": round(fl, 3), "chunk_edge_fraction": round(float(np.mean(edges)), 4),
                     "share_level_L": round(float(np.mean(lvl)), 4)})
    res = {"source": "tools/flicker_oracle.py (CPU oracle only)", "workload": "cfg1 exemplar, 128x96 static guide, 8 frames, L=3",
           "rows": rows}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                            "profiles", "r02_flicker_oracle.json"))
