"""Parity at BASELINE.json's full size, in the launch configuration bench.py times: one
sb_stylize_batch over 64 4K frames of config 5 (frame seeds 0x5EED + i, the bench's G_T
recipe), blit path and the r = 2 blend path (coords, then sb_vote), and the exact
3-channel search path.  The oracle computes sampled outputs one by one (stylize_pixel, and
the vote of a sample from the oracle coords of its 5x5 window)."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1807_03249_b200 as sb
import synth

pytestmark = pytest.mark.gpu
NTH = min(16, os.cpu_count() or 1)
DEV = "cuda"
B, WT, HT = 64, 3840, 2160
FRAMES = (0, 7, 8, 63)


@pytest.fixture(scope="module")
def bench_batch():
    cfg = synth.CONFIGS[5]
    cs, gs = [t.to(DEV) for t in synth.exemplar(cfg, device=DEV)]
    gt = torch.empty(B, HT, WT, 4, dtype=torch.uint8, device=DEV)
    for i in range(8):  # bench.py: 8 distinct phases, cycled
        gt[i] = synth.heightfield_normals(WT, HT, seed=5, frame=i, device=DEV)
    for i in range(8, B):
        gt[i] = gt[i % 8]
    seeds = [(cfg["seed"] + i) & 0xFFFFFFFF for i in range(B)]
    csn, gsn = cs.cpu().numpy(), gs.cpu().numpy()
    return dict(cfg=cfg, cs=cs, gs=gs, gt=gt, seeds=seeds, csn=csn, gsn=gsn, lut=oracle.build_lut(gsn, nthreads=NTH))


def _samples(rng, n, margin=0):
    xs = rng.randint(margin, WT - margin, n)
    ys = rng.randint(margin, HT - margin, n)
    # plus the frame corners and tile seams (x multiple of 128, y multiple of 32)
    ex = [(0, 0), (WT - 1, HT - 1), (WT - 1, 0), (0, HT - 1), (128, 32), (127, 31), (3839, 2159 - 16)]
    if margin:
        ex = [(min(max(x, margin), WT - 1 - margin), min(max(y, margin), HT - 1 - margin)) for x, y in ex]
    return list(zip(xs.tolist(), ys.tolist())) + ex


def test_fullsize_blit(bench_batch):
    b = bench_batch
    cfg = b["cfg"]
    # the bench's launch configuration, with the strided exemplar copy
    prm = sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], seed=cfg["seed"],
                    exemplar=sb.prepare_exemplar(b["cs"], b["gs"]))
    lut = sb.build_lut(b["gs"])
    ct, coords, _ = sb.stylize_batch(prm, b["cs"], b["gs"], lut, b["gt"], frame_seeds=b["seeds"], want_level=False)
    torch.cuda.synchronize()
    rng = np.random.RandomState(1)
    for f in FRAMES:
        gtn = b["gt"][f].cpu().numpy()
        co = coords[f].cpu().numpy().view(np.uint32)
        ctf = ct[f].cpu().numpy()
        op = oracle.Params(t=cfg["t"], L=cfg["L"], C=cfg["C"], seed=b["seeds"][f])
        for x, y in _samples(rng, 1500):
            c, _ = oracle.stylize_pixel(op, b["gsn"], b["lut"], gtn, x, y)
            assert co[y, x] == c, (f, x, y)
            assert (ctf[y, x] == b["csn"][c >> 16, c & 0xFFFF]).all(), (f, x, y)


def test_fullsize_blend_r2(bench_batch):
    b = bench_batch
    cfg = b["cfg"]
    ex = sb.prepare_exemplar(b["cs"], b["gs"])
    prm = sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], seed=cfg["seed"],
                    flags=sb.SB_NO_COLOR, exemplar=ex)
    lut = sb.build_lut(b["gs"])
    _, coords, _ = sb.stylize_batch(prm, b["cs"], b["gs"], lut, b["gt"], frame_seeds=b["seeds"], want_level=False)
    ct = sb.vote(coords, b["cs"], 2, exemplar=ex)
    torch.cuda.synchronize()
    rng = np.random.RandomState(2)
    for f in FRAMES[:2]:
        gtn = b["gt"][f].cpu().numpy()
        ctf = ct[f].cpu().numpy()
        op = oracle.Params(t=cfg["t"], L=cfg["L"], C=cfg["C"], seed=b["seeds"][f])
        for x, y in _samples(rng, 300, margin=2):
            patch = np.zeros((5, 5), np.uint32)
            for dy in range(5):
                for dx in range(5):
                    patch[dy, dx] = oracle.stylize_pixel(op, b["gsn"], b["lut"], gtn, x - 2 + dx, y - 2 + dy)[0]
            # the vote of the patch centre sees exactly the patch (the window is inside the frame);
            # the patch coordinates are frame coordinates, so shift them into patch space: the
            # vote only uses src(q) + (p - q), which is translation invariant.
            want = oracle.vote(patch, b["csn"], 2)[2, 2]
            assert (ctf[y, x] == want).all(), (f, x, y, ctf[y, x], want)


def test_fullsize_lut_rgb(bench_batch):
    b = bench_batch
    cfg = b["cfg"]
    prm = sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], seed=cfg["seed"], lut_rgb=True,
                    exemplar=sb.prepare_exemplar(b["cs"], b["gs"]))
    lut3 = sb.build_lut3(b["gs"])
    ct, coords, _ = sb.stylize_batch(prm, b["cs"], b["gs"], lut3, b["gt"], frame_seeds=b["seeds"], want_level=False)
    torch.cuda.synchronize()
    rng = np.random.RandomState(3)
    f = 63
    gtn = b["gt"][f].cpu().numpy()
    co = coords[f].cpu().numpy().view(np.uint32)
    op = oracle.Params(t=cfg["t"], L=cfg["L"], C=cfg["C"], seed=b["seeds"][f], lut_rgb=True)
    for x, y in _samples(rng, 120):
        c, _ = oracle.stylize_pixel(op, b["gsn"], None, gtn, x, y)
        assert co[y, x] == c, (x, y)
