"""PAPER.md 3.3 (lines 423-433): animation by per-frame reseeding.

"The randomization of seed points slightly perturbs the structure of the resulting mosaic ...
the amount of flickering can be controlled by changing the guidance threshold.  Higher
threshold gives rise to larger chunks and more visible visual changes between consecutive
frames and thus the amount of flickering is increased."  Measured here as
  flicker(t) = mean |C_T^(i+1) - C_T^(i)| over pixels, channels and consecutive frames
for a static guide with per-frame seeds, and chunk size as the number of 4-neighbour pixel
pairs whose offsets (src - p) differ (fewer = larger chunks).
"""
import numpy as np
import pytest
import torch

import oracle
import synth


def flicker_and_edges(frames_ct, coords):
    ct = np.stack(frames_ct).astype(np.int32)
    fl = float(np.abs(np.diff(ct, axis=0)).mean())
    edges = []
    for co in coords:
        H, W = co.shape
        ox = (co & 0xFFFF).astype(np.int64) - np.arange(W)[None, :]
        oy = (co >> 16).astype(np.int64) - np.arange(H)[:, None]
        off = ox * 65536 + oy
        edges.append(int((off[:, 1:] != off[:, :-1]).sum() + (off[1:] != off[:-1]).sum()))
    return fl, float(np.mean(edges))


def test_flicker_and_chunks_grow_with_t_oracle():
    """CPU oracle, 64x64 static guide, 6 reseeded frames: flicker increases and chunk edges
    decrease with t; without reseeding the frames are identical."""
    cfg = synth.CONFIGS[1]
    cs, gs = [t.numpy() for t in synth.exemplar(cfg)]
    gt = synth.target(1).numpy()
    lut = oracle.build_lut(gs)
    res = []
    for t in (8.0, 16.0, 32.0, 64.0):
        cts, cos = [], []
        for i in range(6):
            ct, co, _ = oracle.stylize(oracle.Params(t=t, L=3, C=3, seed=100 + i), cs, gs, lut, gt)
            cts.append(ct)
            cos.append(co)
        res.append(flicker_and_edges(cts, cos))
    fl = [r[0] for r in res]
    ed = [r[1] for r in res]
    assert all(a < b for a, b in zip(fl, fl[1:])), fl
    assert all(a > b for a, b in zip(ed, ed[1:])), ed
    a = oracle.stylize(oracle.Params(t=16.0, L=3, C=3, seed=7), cs, gs, lut, gt)[0]
    b = oracle.stylize(oracle.Params(t=16.0, L=3, C=3, seed=7), cs, gs, lut, gt)[0]
    assert (a == b).all()


@pytest.mark.gpu
def test_flicker_grows_with_t_gpu():
    """The same measurement on the GPU batch path (sb_stylize_batch with per-frame seeds) at
    1 MP, 16 frames per threshold."""
    import paper_1807_03249_b200 as sb

    cfg = synth.CONFIGS[2]
    cs, gs = [t.cuda() for t in synth.exemplar(cfg)]
    lut = sb.build_lut(gs)
    gt1 = synth.target(2).cuda()
    frames = gt1.unsqueeze(0).expand(16, *gt1.shape).contiguous()
    out = []
    for t in (4.0, 12.0, 48.0):
        prm = sb.Params(threshold=t, levels=5, guide_channels=3, seed=1)
        ct, co, _ = sb.stylize_batch(prm, cs, gs, lut, frames)  # seeds 1 .. 16
        out.append(flicker_and_edges(list(ct.cpu().numpy()), list(co.cpu().numpy().view(np.uint32))))
        same = sb.stylize_batch(prm, cs, gs, lut, frames, frame_seeds=[5] * 16)[0]
        assert all(torch.equal(same[0], same[i]) for i in range(16))
    fl = [o[0] for o in out]
    ed = [o[1] for o in out]
    assert fl[0] < fl[1] < fl[2], fl
    assert ed[0] > ed[1] > ed[2], ed
