"""Debug: tiled vs naive stylize vs oracle on config 2 with seed 4 (run on the GPU box)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
code = r'''
import sys, torch, numpy as np
sys.path.insert(0, %r)
import synth, paper_1807_03249_b200 as sb
cfg=synth.CONFIGS[2]; cs,gs=[t.cuda() for t in synth.exemplar(cfg)]; lut=sb.build_lut(gs)
gt=synth.target(2).cuda()
for r in (0, 2):
    p=sb.Params(threshold=cfg['t'],levels=5,blend_radius=r,guide_channels=3,seed=4)
    ct,co,lv=sb.stylize(p,cs,gs,lut,gt); torch.cuda.synchronize()
    np.savez(sys.argv[1] + f'_r{r}.npz', ct=ct.cpu().numpy(), co=co.cpu().numpy(), lv=lv.cpu().numpy())
''' % ROOT
out = {}
for mode in ("tiled", "naive"):
    f = f"/tmp/dbg_{mode}"
    subprocess.check_call([sys.executable, "-c", code, f], env=dict(os.environ, SB_KERNEL=mode))
    out[mode] = {r: np.load(f + f"_r{r}.npz") for r in (0, 2)}
import oracle, synth
cfg = synth.CONFIGS[2]
cs, gs = [t.numpy() for t in synth.exemplar(cfg)]
gt = synth.target(2).numpy()
lut = oracle.build_lut(gs, 16)
oct_, oco, olv = oracle.stylize(oracle.Params(t=cfg["t"], L=5, C=3, seed=4), cs, gs, lut, gt, 16)
ov = oracle.vote(oco, cs, 2, 16)
for mode in out:
    for r in (0, 2):
        d = out[mode][r]
        co = d["co"].view(np.uint32)
        print(mode, r, "coords mism", int((co != oco).sum()), "lv mism", int((d["lv"] != olv).sum()),
              "ct mism", int((d["ct"] != (oct_ if r == 0 else ov)).sum()))
        if (co != oco).any():
            w = np.argwhere(co != oco)[:5]
            print("   first", w.tolist(), co[tuple(w[0])], oco[tuple(w[0])], d["lv"][tuple(w[0])], olv[tuple(w[0])])
