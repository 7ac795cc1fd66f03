"""GPU parity at the edges of the SURVEY 8(b) contract (include/styleblit.h: SB_MAX_DIM,
SB_MAX_LEVELS, SB_MAX_RADIUS): image sides beyond 32767 and L = 10..15 (the per-pixel kernels),
and the vote radius r = 8 (the runs kernel with its window sums split over two SWAR register
pairs).  Every case is compared with the CPU oracle element by element (coords, levels, colours
bit-exact)."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1807_03249_b200 as sb
import synth

pytestmark = pytest.mark.gpu
NTH = min(16, os.cpu_count() or 1)


def _both(cs, gs, gt, t, L, r, C=3, seed=7, with_exemplar=False):
    csd, gsd, gtd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (cs, gs, gt))
    lut_d = sb.build_lut(gsd)
    ex = sb.prepare_exemplar(csd, gsd) if with_exemplar else None
    prm = sb.Params(threshold=t, levels=L, blend_radius=r, guide_channels=C, seed=seed, exemplar=ex)
    ct, co, lv = sb.stylize(prm, csd, gsd, lut_d, gtd)
    torch.cuda.synchronize()
    lut = oracle.build_lut(gs, nthreads=NTH)
    assert (lut_d.cpu().numpy().view(np.uint32) == lut).all(), "LUT"
    oct_, oco, olv = oracle.stylize(oracle.Params(t=t, L=L, C=C, seed=seed), cs, gs, lut, gt, nthreads=NTH)
    if r > 0:
        oct_ = oracle.vote(oco, cs, r, nthreads=NTH)
    g_co = co.cpu().numpy().view(np.uint32)
    assert (g_co == oco).all(), f"coords: {(g_co != oco).sum()} differ"
    assert (lv.cpu().numpy() == olv).all(), "levels"
    g_ct = ct.cpu().numpy()
    assert (g_ct == oct_).all(), f"colours: {(g_ct != oct_).any(-1).sum()} pixels differ"
    return olv


def _exemplar():
    cfg = synth.CONFIGS[1]
    cs, gs = synth.exemplar(cfg)
    return cs.numpy(), gs.numpy()


@pytest.mark.parametrize("L", [10, 13, 15])
def test_deep_hierarchies(L):
    """L beyond the tiled kernel's 9: h up to 2^15, NearestSeed distances in 64 bits."""
    cs, gs = _exemplar()
    gt = synth.heightfield_normals(203, 150, seed=1).numpy()
    olv = _both(cs, gs, gt, t=24.0, L=L, r=0)
    assert olv.max() >= 9, "coarse levels exercised"


@pytest.mark.parametrize("r", [7, 8])
def test_radius_8(r):
    """r = 8 ((2r+1)^2 * 255 > 2^16: the runs kernel splits the window rows over two SWAR register
    pairs) next to r = 7 (one pair); a target with interior fast tiles and frame-edge tiles."""
    cs, gs = _exemplar()
    for wt, ht in ((150, 70), (300, 100)):
        gt = synth.heightfield_normals(wt, ht, seed=1).numpy()
        _both(cs, gs, gt, t=32.0, L=3, r=r)
        _both(cs, gs, gt, t=32.0, L=3, r=r, with_exemplar=True)


@pytest.mark.parametrize("with_exemplar", [False, True])
def test_radius_8_saturated_sums(with_exemplar):
    """r = 8 where every channel sum reaches 289 * 255 = 73695 > 2^16 (a white exemplar with a few
    dark pixels; noise guides: many short chunks, so the two-run, run-loop and border paths all
    carry saturated sums)."""
    rng = np.random.RandomState(8)
    cs = np.full((96, 96, 4), 255, np.uint8)
    cs[rng.rand(96, 96) < 0.02] = 0
    gs = rng.randint(0, 256, (96, 96, 4)).astype(np.uint8)
    gt = rng.randint(0, 256, (80, 260, 4)).astype(np.uint8)
    _both(cs, gs, gt, t=2000.0, L=2, r=8, with_exemplar=with_exemplar)
    gs_smooth = synth.heightfield_normals(96, 96, seed=3).numpy()
    gt_smooth = synth.heightfield_normals(260, 80, seed=4).numpy()
    _both(cs, gs_smooth, gt_smooth, t=20.0, L=3, r=8, with_exemplar=with_exemplar)


@pytest.mark.parametrize("wt,ht", [(40000, 3), (5, 33000)])
def test_wide_targets(wt, ht):
    """Target sides beyond 32767 (per-pixel stylize and vote with signed coordinates)."""
    cs, gs = _exemplar()
    rng = np.random.RandomState(wt + ht)
    gt = rng.randint(0, 256, (ht, wt, 4)).astype(np.uint8)
    for r in (0, 2):
        _both(cs, gs, gt, t=40.0, L=4, r=r)


def test_wide_exemplar():
    """A source wider than 32767 pixels: the LUT build (pixel indices beyond 2^15 rows of
    16 bits), candidates and votes with signed source coordinates."""
    rng = np.random.RandomState(5)
    ws, hs = 33000, 2
    gs = rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8)
    cs = rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8)
    gt = synth.heightfield_normals(130, 20, seed=2).numpy()
    for r in (0, 2):
        _both(cs, gs, gt, t=30.0, L=3, r=r)


@pytest.mark.parametrize("L,r,wt,ht", [(15, 8, 96, 40), (12, 2, 40000, 2)])
def test_host_pipeline_at_the_limits(L, r, wt, ht):
    """sb_stylize_batch_host (host frames in and out) on the per-pixel kernels: L = 15 with r = 8,
    and a 40000-wide batch -- equal to the device batch, which equals the oracle (above)."""
    cs, gs = _exemplar()
    rng = np.random.RandomState(L + r)
    gt = rng.randint(0, 256, (3, ht, wt, 4)).astype(np.uint8)
    csd, gsd = torch.from_numpy(cs).cuda(), torch.from_numpy(gs).cuda()
    lut = sb.build_lut(gsd)
    prm = sb.Params(threshold=40.0, levels=L, blend_radius=r, guide_channels=3, seed=3)
    dev_ct, _, _ = sb.stylize_batch(prm, csd, gsd, lut, torch.from_numpy(gt).cuda(), want_level=False)
    gt_h = torch.from_numpy(gt).pin_memory()
    ct_h = torch.empty_like(gt_h).pin_memory()
    sb.stylize_batch_host(prm, csd, gsd, lut, gt_h, ct_h)
    assert torch.equal(ct_h, dev_ct.cpu())
    o = oracle.stylize(oracle.Params(t=40.0, L=L, C=3, seed=3 + 1), cs, gs, oracle.build_lut(gs, nthreads=NTH),
                       gt[1], nthreads=NTH)
    want = oracle.vote(o[1], cs, r, nthreads=NTH) if r > 0 else o[0]
    assert (ct_h[1].numpy() == want).all()


def test_empty_batches():
    """n_frames = 0 (an empty batch is valid): the device batch, the vote and the
    host pipeline return SB_OK, launch no kernel and leave their outputs untouched."""
    cs, gs = _exemplar()
    csd, gsd = torch.from_numpy(cs).cuda(), torch.from_numpy(gs).cuda()
    lut = sb.build_lut(gsd)
    gt = torch.zeros(0, 48, 64, 4, dtype=torch.uint8, device="cuda")
    ct = torch.zeros(0, 48, 64, 4, dtype=torch.uint8, device="cuda")
    co = torch.zeros(0, 48, 64, dtype=torch.int32, device="cuda")
    prm = sb.Params(threshold=20.0, levels=4, blend_radius=2, guide_channels=3, seed=3)
    sb.stylize_batch(prm, csd, gsd, lut, gt, ct=ct, coords=co, want_level=False)
    assert sb.launch_count() == 0
    sb.vote(co, csd, 2, ct=ct)
    assert sb.launch_count() == 0
    gt_h = torch.zeros(0, 48, 64, 4, dtype=torch.uint8).pin_memory()
    ct_h = torch.zeros(0, 48, 64, 4, dtype=torch.uint8).pin_memory()
    sb.stylize_batch_host(sb.Params(threshold=20.0, levels=4, guide_channels=3, seed=3), csd, gsd, lut, gt_h, ct_h)
    assert sb.launch_count() == 0
    torch.cuda.synchronize()


@pytest.mark.parametrize("ws,hs,wt,ht", [(1, 1, 1, 1), (1, 1, 37, 5), (5, 1, 1, 9), (1, 7, 131, 1), (2, 2, 3, 130),
                                         (17, 17, 1, 1)])
@pytest.mark.parametrize("L,r", [(1, 0), (5, 2), (15, 8)])
def test_degenerate_sizes(ws, hs, wt, ht, L, r):
    """Single-pixel and single-row/column exemplars and targets (every window clipped, no source
    margin for the fast vote tiles, seed cells far larger than the image) at the ends of the L
    and r ranges: bit-exact against the oracle, with and without the strided exemplar copy."""
    rng = np.random.RandomState(ws * 1000 + hs * 100 + wt + ht)
    cs = rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8)
    gs = rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8)
    gt = rng.randint(0, 256, (ht, wt, 4)).astype(np.uint8)
    for ex in (False, True):
        _both(cs, gs, gt, t=90.0, L=L, r=r, with_exemplar=ex)
