"""Run each kernel repeatedly on identical inputs and report any run-to-run difference."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1807_03249_b200 as sb  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[2]
cs, gs = [t.cuda() for t in synth.exemplar(cfg)]
lut0 = sb.build_lut(gs)
for _ in range(20):
    l2 = sb.build_lut(gs)
    assert torch.equal(l2, lut0), "LUT nondeterministic"
print("lut ok")
gt = synth.target(2).cuda()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 50
p = sb.Params(threshold=cfg["t"], levels=5, blend_radius=0, guide_channels=3, seed=4, flags=sb.SB_NO_COLOR)
_, co0, lv0 = sb.stylize(p, cs, gs, lut0, gt)
bad = 0
for i in range(N):
    _, co, lv = sb.stylize(p, cs, gs, lut0, gt)
    if not (torch.equal(co, co0) and torch.equal(lv, lv0)):
        bad += 1
        d = (co != co0).nonzero()
        print("stylize run", i, "differs at", d[:5].tolist(), "n", d.shape[0])
print("stylize bad runs", bad)
ct0 = sb.vote(co0, cs, 2)
bad = 0
for i in range(N):
    ct = sb.vote(co0, cs, 2)
    if not torch.equal(ct, ct0):
        bad += 1
        d = (ct != ct0).any(-1).nonzero()
        print("vote run", i, "differs at", d[:5].tolist(), "n", d.shape[0])
print("vote bad runs", bad)
