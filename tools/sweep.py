"""Throughput of the hot path versus the method's parameters on the headline workload shape
(16 x 4K heightfield-normal frames, 512^2 sphere exemplar, strided exemplar copy): the stylize
kernel against the threshold t and the hierarchy depth L (with the level histogram that drives
its cost), and the vote against the radius r.  Writes one JSON object (profiles/r02_sweep.json).

usage (on a GPU box): python tools/sweep.py [out.json]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03249_b200 as sb  # noqa: E402
import synth  # noqa: E402

W, H, N = 3840, 2160, 16


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main(out):
    dev = torch.device("cuda:0")
    cfg = synth.CONFIGS[5]
    cs, gs = [t.to(dev) for t in synth.exemplar(cfg, device=dev)]
    gt = torch.stack([synth.heightfield_normals(W, H, seed=5, frame=i, device=dev) for i in range(N)])
    lut = sb.build_lut(gs)
    ex = sb.prepare_exemplar(cs, gs)
    ct = torch.empty(N, H, W, 4, dtype=torch.uint8, device=dev)
    co = torch.empty(N, H, W, dtype=torch.int32, device=dev)
    lv = torch.empty(N, H, W, dtype=torch.uint8, device=dev)
    px = N * W * H
    res = {"workload": f"{N} x 3840x2160 heightfield normals (cfg5 shape), 512^2 sphere exemplar, C=3, strided copy",
           "stylize_vs_t_L": [], "vote_vs_r": []}
    for L in (3, 4, 5, 6, 7):
        for t in (2.0, 5.0, 10.0, 20.0, 40.0):
            prm = sb.Params(threshold=t, levels=L, guide_channels=3, seed=cfg["seed"], exemplar=ex)
            ms = timed(lambda: sb.stylize_batch(prm, cs, gs, lut, gt, ct=ct, coords=co, want_level=False))
            sb.stylize_batch(prm, cs, gs, lut, gt[:2], ct=ct[:2], coords=co[:2], level=lv[:2])
            hist = torch.bincount(lv[:2].flatten().long(), minlength=L + 1).float()
            hist = (hist / hist.sum()).tolist()
            res["stylize_vs_t_L"].append({"L": L, "t": t, "ms_per_16_frames": round(ms, 4),
                                          "GMPps": round(px / (ms * 1e-3) / 1e9, 1),
                                          "share_level_L": round(hist[L], 4), "share_level_0": round(hist[0], 4),
                                          "mean_levels_visited": round(sum(hist[l] * (L - l + 1) for l in range(1, L + 1))
                                                                       + hist[0] * L, 3)})
    prm = sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=3, seed=cfg["seed"], exemplar=ex,
                    flags=sb.SB_NO_COLOR)
    sb.stylize_batch(prm, cs, gs, lut, gt, coords=co, want_level=False)
    for r in (1, 2, 3, 4, 5, 6, 7, 8):
        ms = timed(lambda: sb.vote(co, cs, r, ct=ct, exemplar=ex))
        res["vote_vs_r"].append({"r": r, "ms_per_16_frames": round(ms, 4), "GMPps": round(px / (ms * 1e-3) / 1e9, 1),
                                 "kernel": "vote (runs)"})
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_sweep.json")
