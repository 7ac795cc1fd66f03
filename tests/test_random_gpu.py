"""Randomised GPU-vs-oracle parity over the whole parameter space of the boundary (hypothesis,
derandomised: the same examples every run).

Each example draws target and exemplar sizes (1..300 x 1..80, 1..96 x 1..96: tile-ragged, odd
widths, single pixels), content (uniform noise -- many ties and tiny chunks -- or the smooth
synthetic guides), L in 1..15, t (including 0 and values between integers), C in 2..4, the voting
radius r in 0..8, the jitter seed, zero jitter, per-channel weights, a segmentation label byte,
the exact three-channel search (SB_LUT_RGB), an output strip [row_begin, row_end) and the
strided exemplar copy.  The CUDA path and the oracle must agree bit for bit on the coordinates,
the levels and the colours (blit or vote) of every row the call writes.  test_random_parity_large
redraws the sizes at multi-tile scale (targets up to 1280 x 200, exemplars up to 512^2, L 3..9).
SB_HYP_N / SB_HYP_N_LARGE set the example counts, SB_HYP_RANDOM=1 draws fresh examples.
"""
import os

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
import paper_1807_03249_b200 as sb
import synth

pytestmark = pytest.mark.gpu
NTH = min(16, os.cpu_count() or 1)


def _image(rng, w, h, kind, seed):
    if kind == "noise":
        return rng.randint(0, 256, (h, w, 4)).astype(np.uint8)
    if kind == "sphere":
        return synth.sphere_normal(w, h).numpy()
    return synth.heightfield_normals(w, h, seed=seed).numpy()


case = st.fixed_dictionaries({
    # hypothesis favours small values; half the draws are tile-scale sizes
    "wt": st.one_of(st.integers(1, 300), st.sampled_from([127, 128, 131, 200, 256, 261, 300])),
    "ht": st.one_of(st.integers(1, 80), st.sampled_from([16, 17, 33, 48, 64, 80])),
    "ws": st.one_of(st.integers(1, 96), st.sampled_from([48, 64, 80, 96])),
    "hs": st.one_of(st.integers(1, 96), st.sampled_from([40, 64, 96])),
    "gkind": st.sampled_from(["noise", "sphere", "smooth"]), "tkind": st.sampled_from(["noise", "smooth"]),
    "L": st.integers(1, 15),
    "t": st.one_of(st.sampled_from([0.0, 0.5, 1.0, 1.5, 10.0, 300.0]), st.floats(0.0, 80.0, width=32)),
    "C": st.integers(2, 4), "r": st.integers(0, 8),
    "seed": st.integers(0, 2**32 - 1), "zero_jitter": st.booleans(),
    "weights": st.one_of(st.just((0, 0, 0, 0)), st.tuples(*[st.integers(0, 255)] * 4)),
    "label": st.booleans(), "lut_rgb": st.booleans(), "strip": st.booleans(), "exemplar": st.booleans(),
    "rows": st.tuples(st.floats(0, 1), st.floats(0, 1)),
    "rng": st.integers(0, 2**31 - 1),
})


@settings(max_examples=int(os.environ.get("SB_HYP_N", "150")), derandomize=os.environ.get("SB_HYP_RANDOM") is None, deadline=None,
          suppress_health_check=[HealthCheck.too_slow, HealthCheck.data_too_large])
@given(c=case)
def test_random_parity(c):
    _check(c)


# multi-tile frames (up to 10 x 13 tiles) and exemplars up to 512^2: the interior fast paths of
# both kernels, the level tables at L up to 9 and long group / pixel queues
large_sizes = st.fixed_dictionaries({
    "wt": st.integers(129, 1280), "ht": st.integers(17, 200), "ws": st.integers(64, 512), "hs": st.integers(64, 512),
    "L": st.integers(3, 9),
})


@settings(max_examples=int(os.environ.get("SB_HYP_N_LARGE", "12")), derandomize=os.environ.get("SB_HYP_RANDOM") is None,
          deadline=None, suppress_health_check=[HealthCheck.too_slow, HealthCheck.data_too_large])
@given(c=case, big=large_sizes)
def test_random_parity_large(c, big):
    c = dict(c)
    c.update(big)
    c["lut_rgb"] = False  # the oracle's exact three-channel search is quadratic in the exemplar
    _check(c)


def _check(c):
    rng = np.random.RandomState(c["rng"])
    wt, ht, ws, hs = c["wt"], c["ht"], c["ws"], c["hs"]
    if c["lut_rgb"]:  # the oracle searches all exemplar pixels per query: keep it small
        ws, hs = min(ws, 24), min(hs, 24)
    gs = _image(rng, ws, hs, c["gkind"], 1 + c["rng"] % 7)
    cs = rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8)
    gt = _image(rng, wt, ht, c["tkind"], 11 + c["rng"] % 5)
    C = c["C"]
    label = 3 if (c["label"] and C <= 3) else None
    if label is not None:  # coarse region labels in byte 3 of both guides
        gs[..., 3] = (np.arange(ws)[None, :] * 4 // max(ws, 1) * 50).astype(np.uint8)
        gt[..., 3] = (np.arange(wt)[None, :] * 4 // max(wt, 1) * 50).astype(np.uint8)
    w = c["weights"]
    rb = min(int(c["rows"][0] * ht), ht - 1) if c["strip"] else 0  # a non-empty strip
    re_ = max(rb + 1, int(round(c["rows"][1] * ht))) if c["strip"] else ht
    re_ = min(re_, ht)
    r = c["r"]

    csd, gsd, gtd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (cs, gs, gt))
    lut_d = sb.build_lut3(gsd) if c["lut_rgb"] else sb.build_lut(gsd)
    ex = sb.prepare_exemplar(csd, gsd) if c["exemplar"] else None
    prm = sb.Params(threshold=float(c["t"]), levels=c["L"], blend_radius=r, guide_channels=C, seed=c["seed"],
                    flags=sb.SB_JITTER_ZERO if c["zero_jitter"] else 0, row_begin=rb if c["strip"] else 0,
                    row_end=re_ if c["strip"] else 0, weights=w, label_channel=label, lut_rgb=c["lut_rgb"],
                    exemplar=ex)
    ct = torch.zeros(ht, wt, 4, dtype=torch.uint8, device="cuda")
    co = torch.zeros(ht, wt, dtype=torch.int32, device="cuda")
    lv = torch.zeros(ht, wt, dtype=torch.uint8, device="cuda")
    sb.stylize(prm, csd, gsd, lut_d, gtd, ct=ct, coords=co, level=lv)
    torch.cuda.synchronize()

    lut = None if c["lut_rgb"] else oracle.build_lut(gs, nthreads=NTH)
    if not c["lut_rgb"]:
        assert (lut_d.cpu().numpy().view(np.uint32) == lut).all(), "LUT"
    ow = w if any(w) else (1, 1, 1, 1)
    oprm = oracle.Params(t=float(c["t"]), L=c["L"], C=C, seed=c["seed"], zero_jitter=c["zero_jitter"], weights=ow,
                         label_channel=label, lut_rgb=c["lut_rgb"])
    oct_, oco, olv = oracle.stylize(oprm, cs, gs, lut, gt, nthreads=NTH)
    if r > 0:
        oct_ = oracle.vote(oco, cs, r, nthreads=NTH)
    rows = slice(rb, re_)
    g_co = co.cpu().numpy().view(np.uint32)
    assert (g_co[rows] == oco[rows]).all(), f"coords {(g_co[rows] != oco[rows]).sum()} differ"
    assert (lv.cpu().numpy()[rows] == olv[rows]).all(), "levels"
    g_ct = ct.cpu().numpy()
    assert (g_ct[rows] == oct_[rows]).all(), f"colours {(g_ct[rows] != oct_[rows]).any(-1).sum()} pixels differ"
