"""GPU parity of the exact three-channel guide search (SB_LUT_RGB, R26; SURVEY 8(f)
#3): sb_build_lut3 against the oracle's direct argmin on sampled keys, and Alg. 2 with the
3-channel u* against the oracle, bit-exact (coords, levels, colours, vote)."""
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


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _sample_keys(gt: np.ndarray, n: int, seed: int) -> np.ndarray:
    rng = np.random.RandomState(seed)
    g = gt.reshape(-1, 4).astype(np.uint32)
    present = g[:, 0] | (g[:, 1] << 8) | (g[:, 2] << 16)
    rand = rng.randint(0, 1 << 24, n).astype(np.uint32)
    corners = np.array([0, 0xFFFFFF, 0xFF, 0xFF00, 0xFF0000, 0x808080], np.uint32)
    return np.unique(np.concatenate([rand, rng.choice(present, n), corners]))


@pytest.mark.parametrize("case", ["random_ties", "random_full", "sphere"])
def test_lut3_matches_oracle(case):
    rng = np.random.RandomState(hash(case) & 0xFFFF)
    if case == "random_ties":
        gs = (rng.randint(0, 4, (20, 24, 4)) * 60).astype(np.uint8)
    elif case == "random_full":
        gs = rng.randint(0, 256, (37, 41, 4)).astype(np.uint8)
    else:
        gs = synth.sphere_normal(64, 64).numpy()
    lut3 = _u32(sb.build_lut3(torch.from_numpy(gs).to(DEV)))
    keys = _sample_keys(gs, 4000, 5)
    ref = oracle.lut3_entries(gs, keys, nthreads=NTH)
    bad = np.nonzero(lut3[keys] != ref)[0]
    assert bad.size == 0, f"{bad.size} mismatches, e.g. key {keys[bad[0]]:#x}: gpu {lut3[keys[bad[0]]]:#x} oracle {ref[bad[0]]:#x}"


def test_lut3_bench_exemplar_sampled():
    """512^2 sphere exemplar (the bench's): sampled keys incl. every key of a 4K frame's rows."""
    gs = synth.sphere_normal(512, 512).numpy()
    gt = synth.target(5, 0)[::64].numpy()  # 34 rows of a 4K frame
    lut3 = _u32(sb.build_lut3(torch.from_numpy(gs).to(DEV)))
    keys = _sample_keys(gt, 1500, 9)
    ref = oracle.lut3_entries(gs, keys, nthreads=NTH)
    assert (lut3[keys] == ref).all()


def test_lut3_reduces_to_lut_when_channel2_constant():
    rng = np.random.RandomState(2)
    gs = rng.randint(0, 256, (33, 30, 4)).astype(np.uint8)
    gs[..., 2] = 201
    gsd = torch.from_numpy(gs).to(DEV)
    lut = _u32(sb.build_lut(gsd))
    lut3 = _u32(sb.build_lut3(gsd))
    k = np.arange(1 << 24, dtype=np.uint32)
    assert (lut3 == lut[k & 0xFFFF]).all()


@pytest.mark.parametrize("wt,ht,ws,L,t,r", [(64, 64, 64, 3, 24.0, 0), (300, 200, 48, 4, 16.0, 2),
                                          (258, 131, 40, 5, 10.0, 0), (128, 96, 64, 4, 12.0, 1)])
def test_stylize_lut_rgb_parity(wt, ht, ws, L, t, r):
    """Alg. 2 with u* from the tabulated 3-channel search vs the oracle's direct search.
    (258 wide: not a multiple of 4 -> the per-pixel kernel.)"""
    gs = synth.sphere_normal(ws, ws).numpy()
    cs = synth.painted_style(ws, ws, seed=4).numpy()
    gt = synth.heightfield_normals(wt, ht, seed=7).numpy()
    gsd, csd, gtd = (torch.from_numpy(a).to(DEV) for a in (gs, cs, gt))
    lut3 = sb.build_lut3(gsd)
    prm = sb.Params(threshold=t, levels=L, blend_radius=r, lut_rgb=True)
    ct, coords, level = sb.stylize(prm, csd, gsd, lut3, gtd)
    torch.cuda.synchronize()
    oprm = oracle.Params(t=t, L=L, C=3, lut_rgb=True)
    oct_, oco, olv = oracle.stylize(oprm, cs, gs, None, gt, nthreads=NTH)
    if r > 0:
        oct_ = oracle.vote(oco, cs, r, nthreads=NTH)
    assert (_u32(coords) == oco).all()
    assert (level.cpu().numpy() == olv).all()
    assert (ct.cpu().numpy() == oct_).all()
    # the 3-channel search changes the result on these inputs (not a no-op flag)
    ct2, coords2, _ = sb.stylize(sb.Params(threshold=t, levels=L, blend_radius=r), csd, gsd, sb.build_lut(gsd), gtd)
    assert (_u32(coords2) != oco).any()


def test_lut_size_checked():
    gs = torch.from_numpy(synth.sphere_normal(16, 16).numpy()).to(DEV)
    with pytest.raises(ValueError):
        sb.stylize(sb.Params(threshold=4.0, levels=2, lut_rgb=True), gs, gs, sb.build_lut(gs), gs)
