"""Repeat the tiled/naive subprocess comparison several times; report where they differ."""
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
p=sb.Params(threshold=cfg['t'],levels=5,blend_radius=2,guide_channels=3,seed=4)
ct,co,lv=sb.stylize(p,cs,gs,lut,gt); torch.cuda.synchronize()
np.savez(sys.argv[1], ct=ct.cpu().numpy(), co=co.cpu().numpy(), lv=lv.cpu().numpy(), lut=lut.cpu().numpy(), gt=gt.cpu().numpy(), gs=gs.cpu().numpy(), cs=cs.cpu().numpy())
''' % ROOT
ref = None
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    for mode in ("tiled", "naive"):
        f = f"/tmp/dbg2_{mode}_{it}.npz"
        subprocess.check_call([sys.executable, "-c", code, f], env=dict(os.environ, SB_KERNEL=mode))
        d = dict(np.load(f))
        if ref is None:
            ref = d
            continue
        msg = []
        for k in d:
            if not np.array_equal(d[k], ref[k]):
                w = np.argwhere(d[k] != ref[k])
                msg.append(f"{k}: {len(w)} diffs, first {w[:3].tolist()} got {d[k][tuple(w[0])]} ref {ref[k][tuple(w[0])]}")
        print(it, mode, "OK" if not msg else " | ".join(msg), flush=True)
