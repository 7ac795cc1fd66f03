"""Randomised GPU-vs-oracle parity of the standalone vote (sb_vote) on
coordinate fields that stylize would rarely produce (hypothesis, derandomised by default; the
SB_HYP_N / SB_HYP_RANDOM knobs of test_random_gpu.py apply).

Each field is a mosaic of chunks (random chunk sizes 1..40 px, each copying a random source
block, so the windows hold from one to (2r+1)^2 distinct offsets), optionally with sources
pushed to the exemplar border (the general path) and a share of isolated random coordinates;
random r in 0..8, ragged target and exemplar sizes, strips, several frames, with and without
the strided exemplar copy.  The colours must equal the oracle's bit for bit on the written rows,
and the rows outside the strip must stay untouched."""
import os

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
import paper_1807_03249_b200 as sb

pytestmark = pytest.mark.gpu
NTH = min(16, os.cpu_count() or 1)

case = st.fixed_dictionaries({
    "wt": st.one_of(st.integers(1, 400), st.sampled_from([128, 256, 260, 384])),
    "ht": st.one_of(st.integers(1, 70), st.sampled_from([16, 32, 48])),
    "ws": st.integers(1, 120), "hs": st.integers(1, 120),
    "chunk": st.integers(1, 40), "border": st.booleans(), "noise": st.sampled_from([0.0, 0.0, 0.01, 0.2]),
    "r": st.integers(0, 8), "frames": st.integers(1, 3), "strip": st.booleans(),
    "rows": st.tuples(st.floats(0, 1), st.floats(0, 1)), "exemplar": st.booleans(),
    "rng": st.integers(0, 2**31 - 1),
})


def _field(rng, wt, ht, ws, hs, chunk, border, noise):
    yy, xx = np.mgrid[0:ht, 0:wt]
    nby, nbx = ht // chunk + 1, wt // chunk + 1
    ox = rng.randint(0, ws, (nby, nbx)) - xx[0, 0]
    oy = rng.randint(0, hs, (nby, nbx))
    if border:  # anchor many chunks at the exemplar edges
        ox = np.where(rng.rand(nby, nbx) < 0.5, 0, ox)
        oy = np.where(rng.rand(nby, nbx) < 0.5, hs - 1, oy)
    sx = np.clip(xx % chunk + ox[yy // chunk, xx // chunk], 0, ws - 1)
    sy = np.clip(yy % chunk - chunk // 2 + oy[yy // chunk, xx // chunk], 0, hs - 1)
    if noise > 0:
        m = rng.rand(ht, wt) < noise
        sx = np.where(m, rng.randint(0, ws, (ht, wt)), sx)
        sy = np.where(m, rng.randint(0, hs, (ht, wt)), sy)
    return (sx | (sy << 16)).astype(np.uint32)


@settings(max_examples=int(os.environ.get("SB_HYP_N", "120")), derandomize=os.environ.get("SB_HYP_RANDOM") is None,
          deadline=None, suppress_health_check=[HealthCheck.too_slow, HealthCheck.data_too_large])
@given(c=case)
def test_random_vote(c):
    rng = np.random.RandomState(c["rng"])
    wt, ht, ws, hs, r = c["wt"], c["ht"], c["ws"], c["hs"], c["r"]
    cs = rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8)
    co = np.stack([_field(rng, wt, ht, ws, hs, c["chunk"], c["border"], c["noise"]) for _ in range(c["frames"])])
    rb, re_ = 0, ht
    if c["strip"]:
        rb = min(int(c["rows"][0] * ht), ht - 1)
        re_ = min(max(rb + 1, int(round(c["rows"][1] * ht))), ht)
    csd = torch.from_numpy(cs).cuda()
    ex = sb.prepare_exemplar(csd, torch.zeros_like(csd)) if c["exemplar"] else None
    cod = torch.from_numpy(co.view(np.int32)).cuda()
    ct = torch.full((c["frames"], ht, wt, 4), 77, dtype=torch.uint8, device="cuda")
    sb.vote(cod, csd, r, ct=ct, row_begin=rb if c["strip"] else 0, row_end=re_ if c["strip"] else 0, exemplar=ex)
    torch.cuda.synchronize()
    g = ct.cpu().numpy()
    for f in range(c["frames"]):
        want = oracle.vote(co[f], cs, r, nthreads=NTH)
        ok = g[f, rb:re_] == want[rb:re_]
        assert ok.all(), f"frame {f}: {(~ok).any(-1).sum()} pixels differ, first {np.argwhere(~ok.all(-1))[:3].tolist()}"
        assert (g[f, :rb] == 77).all() and (g[f, re_:] == 77).all(), "rows outside the strip were written"
