"""Debug helper: one vote parity case (tests/test_parity_gpu.py::test_vote_exemplar_copy) with the
mismatching pixels printed (GPU vs oracle)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1807_03249_b200 as sb  # noqa: E402

for r in (1, 2):
    rng = np.random.RandomState(r)
    ws, hs, wt, ht = 61, 47, 264, 40
    cs = rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8)
    gs = rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8)
    yy, xx = np.mgrid[0:ht, 0:wt]
    ox = rng.randint(-10, ws - 2, (ht // 8 + 1, wt // 8 + 1))
    oy = rng.randint(-10, hs - 2, (ht // 8 + 1, wt // 8 + 1))
    sx = np.clip(xx % 8 + ox[yy // 8, xx // 8], 0, ws - 1)
    sy = np.clip(yy % 8 + oy[yy // 8, xx // 8], 0, hs - 1)
    co = (sx | (sy << 16)).astype(np.uint32)
    ct = torch.full((ht, wt, 4), 0xAB, dtype=torch.uint8, device="cuda")
    g = sb.vote(torch.from_numpy(co.view(np.int32)).cuda(), torch.from_numpy(cs).cuda(), r, ct=ct).cpu().numpy()
    ref = oracle.vote(co, cs, r)
    bad = np.argwhere((g != ref).any(-1))
    print(r, "mismatch", len(bad))
    for y, x in bad[:12]:
        print("  ", y, x, g[y, x], ref[y, x])
