"""The A/B vote kernels selected by SB_VOTE (peel: vote_peel.cu, hist: vote_hist.cu; r = 1, 2) and
SB_VOTE_TMA=1 (the TMA-fed persistent kernel of vote.cu) are bit-exact against the oracle too.
The switches are read once per process, so each variant runs in its own subprocess on the distinct-offset fields of test_parity_gpu (chunk sizes 1..32, frame
borders, ragged widths, sources at the exemplar border)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import paper_1807_03249_b200 as sb

bad = 0
for r in (1, 2):
    for chunk in (1, 2, 3, 5, 8, 32):
        rng = np.random.RandomState(100 * r + chunk)
        ws, hs = 200, 180
        cs = rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8)
        csd = torch.from_numpy(cs).cuda()
        ex = sb.prepare_exemplar(csd, torch.zeros_like(csd))
        for wt, ht, lo in ((384, 48, r), (261, 37, r), (130, 40, -10)):
            yy, xx = np.mgrid[0:ht, 0:wt]
            nby, nbx = ht // chunk + 1, wt // chunk + 1
            # lo = -10: sources clipped at the exemplar border (border tiles)
            ox = rng.randint(lo, ws - chunk - r, (nby, nbx))
            oy = rng.randint(lo, hs - chunk - r, (nby, nbx))
            sx = np.clip(xx % chunk + ox[yy // chunk, xx // chunk], 0, ws - 1)
            sy = np.clip(yy % chunk + oy[yy // chunk, xx // chunk], 0, hs - 1)
            co = (sx | (sy << 16)).astype(np.uint32)
            want = oracle.vote(co, cs, r, nthreads=8)
            cod = torch.from_numpy(co.view(np.int32)).cuda()
            for exm in (None, ex):
                g = sb.vote(cod, csd, r, exemplar=exm).cpu().numpy()
                n = int((g != want).any(-1).sum())
                if n:
                    print("MISMATCH", r, chunk, wt, ht, exm is not None, n)
                    bad += 1
print("bad", bad)
sys.exit(1 if bad else 0)
'''


@pytest.mark.parametrize("variant", ["SB_VOTE=peel", "SB_VOTE=hist", "SB_VOTE_TMA=1"])
def test_vote_variant_exact(variant):
    k, v = variant.split("=")
    env = dict(os.environ, **{k: v})
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
