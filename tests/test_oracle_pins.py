"""Pins of the CPU oracle (oracle/) against what the paper and the mathematics fix.

Nothing here re-types the oracle's formulas: every check is a stored value with a
citation (tests/golden/), a closed form, an invariant, a special case that reduces to a
textbook routine, or an independent brute force on tiny inputs.  DESIGN.md "Pins" maps
each oracle function to the tests below.
"""
import math

import numpy as np
import pytest

import oracle
import synth

SEED = 0x5EED


# ------------------------------------------------------------------ jitter table (R5)
def test_hash_vectors(golden):
    g = golden("jitter_vectors.json")
    for x, y in g["lowbias32"]:
        assert oracle.lowbias32(int(x, 16)) == int(y, 16)
    for c in g["cell_hash"]:
        bx, by = c["b"]
        assert oracle.cell_hash(bx, by, c["l"], c["seed"]) == int(c["k"], 16)
        h = 1 << c["l"]
        # any pixel of cell b has the same SeedPoint (Alg. 2: b = floor(p/h))
        for px, py in ((bx * h, by * h), (bx * h + h - 1, by * h + h - 1)):
            assert oracle.seed_point(px, py, c["l"], c["seed"]) == tuple(c["seed_point"])


def test_jitter_range_and_uniformity():
    """j in [0,1)^2 and ~uniform (SPEC seeds 'Distribution': KS < 0.02
    over >= 1e4 cells)."""
    js = np.array([oracle.jitter(bx, by, 3, SEED) for bx in range(-50, 60) for by in range(-50, 60)])
    assert js.min() >= 0.0 and js.max() < 1.0
    for c in range(2):
        v = np.sort(js[:, c])
        n = len(v)
        ks = max(np.max(np.arange(1, n + 1) / n - v), np.max(v - np.arange(0, n) / n))
        assert ks < 0.02, ks
    # levels and seeds decorrelate (a dropped level/seed term fails here)
    a = [oracle.cell_hash(b, 0, 3, SEED) for b in range(200)]
    assert a != [oracle.cell_hash(b, 0, 4, SEED) for b in range(200)]
    assert a != [oracle.cell_hash(b, 0, 3, SEED + 1) for b in range(200)]
    assert a != [oracle.cell_hash(0, b, 3, SEED) for b in range(200)]


# ------------------------------------------------------------------ SeedPoint
def test_seed_point_spec_examples(golden):
    for e in golden("spec_examples.json")["seed_point_forced"]:
        assert oracle.seed_point_j(*e["p"], e["h"], *e["j"]) == tuple(e["s"])


def test_seed_point_lies_in_its_cell():
    """'regular grid points whose positions are randomly perturbed':
    with j in [0,1)^2 the seed of cell b stays inside cell b."""
    rng = np.random.RandomState(0)
    for _ in range(2000):
        l = int(rng.randint(1, 16))  # the whole 8(b) range of L (h up to 2^15)
        h = 1 << l
        px, py = (int(v) for v in rng.randint(-70000, 70000, 2))
        sx, sy = oracle.seed_point(px, py, l, SEED)
        bx, by = px // h, py // h  # python // is floor division
        assert bx * h <= sx < (bx + 1) * h and by * h <= sy < (by + 1) * h


def test_seed_point_zero_jitter_is_grid():
    for l in (1, 2, 5):
        h = 1 << l
        for px, py in ((0, 0), (h - 1, 3), (-1, -1), (-h - 1, 2 * h + 1), (1000, 777)):
            assert oracle.seed_point(px, py, l, SEED, zero_jitter=True) == ((px // h) * h, (py // h) * h)


# ------------------------------------------------------------------ NearestSeed
def test_nearest_seed_spec_examples(golden):
    for e in golden("spec_examples.json")["nearest_seed_zero_jitter"]:
        assert oracle.nearest_seed(*e["p"], e["l"], SEED, zero_jitter=True) == tuple(e["q"])
    for e in golden("jitter_vectors.json")["nearest_seed_raw"]:
        assert oracle.nearest_seed(*e["p"], e["l"], e["seed"]) == tuple(e["q"])


def test_nearest_seed_zero_jitter_closed_form():
    """Zero jitter: seeds on the grid hZ^2, d separable.  Alg. 2 loops x=-1,0,1 outer,
    y inner, keeping the first strict minimum, so an exact half-way tie goes to the lower
    grid line: q = h*b + (h if (p mod h) > h/2 else 0) per axis."""
    for l in (1, 2, 3, 4):
        h = 1 << l
        for px in range(0, 3 * h):
            for py in range(0, 3 * h, max(1, h // 4)):
                ex = (px // h) * h + (h if px % h > h / 2 else 0)
                ey = (py // h) * h + (h if py % h > h / 2 else 0)
                assert oracle.nearest_seed(px, py, l, SEED, zero_jitter=True) == (ex, ey), (l, px, py)
    # deep levels (h up to 2^15, image sides up to 65535): sampled points, the exact half-way
    # points and their neighbours included
    rng = np.random.RandomState(7)
    for l in (10, 13, 15):
        h = 1 << l
        pts = [int(v) for v in rng.randint(0, 65535, 40)] + [h // 2 - 1, h // 2, h // 2 + 1, h - 1, h, 65534]
        for px in pts:
            py = int(rng.randint(0, 65535))
            ex = (px // h) * h + (h if px % h > h / 2 else 0)
            ey = (py // h) * h + (h if py % h > h / 2 else 0)
            assert oracle.nearest_seed(px, py, l, SEED, zero_jitter=True) == (ex, ey), (l, px, py)


def _cands(px, py, l, seed):
    h = 1 << l
    out = []
    for x in (-1, 0, 1):
        for y in (-1, 0, 1):
            s = oracle.seed_point(px + h * x, py + h * y, l, seed)  # pinned above
            out.append(((s[0] - px) ** 2 + (s[1] - py) ** 2, (x, y), s))
    return out


def test_nearest_seed_is_first_minimum_in_loop_order():
    """Alg. 2: among the 3x3 cells, minimal ||s-p||; on ties the first
    candidate in (x outer, y inner) order.  Also: the result is the TRUE nearest seed
    (over a 7x7 cell neighbourhood) in all but rare cases (reading R7)."""
    rng = np.random.RandomState(1)
    n_ties = n_checked = n_far = 0
    for _ in range(3000):
        l = int(rng.randint(1, 6)) if _ % 10 else int(rng.randint(6, 16))  # every 10th: a deep level
        h = 1 << l
        px, py = (int(v) for v in rng.randint(0, 500 if l < 6 else 65535, 2))
        q = oracle.nearest_seed(px, py, l, SEED)
        c = _cands(px, py, l, SEED)
        dmin = min(d for d, _, _ in c)
        first = [s for d, _, s in c if d == dmin][0]
        assert q == first
        if sum(1 for d, _, _ in c if d == dmin) > 1:
            n_ties += 1
        # true nearest seed over 7x7 cells
        best = min((oracle.seed_point(px + h * x, py + h * y, l, SEED) for x in range(-3, 4) for y in range(-3, 4)),
                   key=lambda s: (s[0] - px) ** 2 + (s[1] - py) ** 2)
        dtrue = (best[0] - px) ** 2 + (best[1] - py) ** 2
        assert dmin >= dtrue
        n_far += dmin > dtrue
        n_checked += 1
    assert n_ties > 20  # the tie rule was actually exercised
    assert n_far <= n_checked * 0.002


# ------------------------------------------------------------------ LUT
def _numpy_lut_bruteforce(gs, keys):
    """Independent: vectorised squared distances to every source pixel, np.argmin picks the
    first (row-major) minimum."""
    hs, ws = gs.shape[:2]
    g0 = gs[..., 0].reshape(-1).astype(np.int64)
    g1 = gs[..., 1].reshape(-1).astype(np.int64)
    out = []
    for k0, k1 in keys:
        i = int(np.argmin((g0 - k0) ** 2 + (g1 - k1) ** 2))
        out.append((i % ws) | ((i // ws) << 16))
    return out


@pytest.mark.parametrize("ws,hs,vmax", [(7, 5, 256), (16, 16, 8), (32, 32, 256), (13, 29, 3)])
def test_lut_bruteforce_tiny(ws, hs, vmax):
    rng = np.random.RandomState(ws * 100 + hs)
    gs = np.zeros((hs, ws, 4), np.uint8)
    gs[..., :3] = rng.randint(0, vmax, (hs, ws, 3))
    lut = oracle.build_lut(gs)
    keys = [(int(a), int(b)) for a, b in rng.randint(0, 256, (600, 2))] + [(0, 0), (255, 255), (0, 255), (255, 0)]
    ref = _numpy_lut_bruteforce(gs, keys)
    for (k0, k1), r in zip(keys, ref):
        assert lut[k0 | (k1 << 8)] == r
        assert oracle.lut_entry(gs, k0, k1) == r


def test_lut_uv_identity_closed_form():
    """UV identity on 256x256: G[x,y] = (x,y) so LUT[x | y<<8] = (x,y)."""
    gs = synth.uv_identity(256, 256).numpy()
    assert (gs[..., 0] == np.arange(256)[None, :]).all()
    lut = oracle.build_lut(gs, nthreads=4)
    k = np.arange(65536, dtype=np.uint32)
    assert (lut == ((k & 0xFF) | ((k >> 8) << 16))).all()


def test_lut_constant_guide():
    """Constant guide: every key ties on all pixels -> the first pixel (0,0)."""
    gs = np.full((9, 11, 4), 77, np.uint8)
    assert (oracle.build_lut(gs) == 0).all()


def test_lut_ignores_channels_2_3():
    """R11: the key is channels 0,1 only."""
    rng = np.random.RandomState(5)
    gs = rng.randint(0, 256, (12, 10, 4)).astype(np.uint8)
    gs2 = gs.copy()
    gs2[..., 2:] = rng.randint(0, 256, (12, 10, 2))
    assert (oracle.build_lut(gs) == oracle.build_lut(gs2)).all()


def test_lut_threads_identical():
    rng = np.random.RandomState(9)
    gs = rng.randint(0, 40, (20, 24, 4)).astype(np.uint8)
    assert (oracle.build_lut(gs, 1) == oracle.build_lut(gs, 7)).all()


# ------------------------------------------------------------------ threshold (R1-R3)
def test_threshold_3_4_5(golden):
    """e = ||G_T[p] - G_S[s]|| (L2) and the strict e < t (Alg. 2): (153,204) vs
    (0,0) is e = 255 exactly (3-4-5).  L1 (357) or Linf (204) would decide differently at
    t = 300 / 254.9."""
    e = golden("spec_examples.json")["threshold_3_4_5"]
    gt = np.array([[e["gt_pixel"]]], np.uint8)
    gs = np.array([[e["gs_pixel"]]], np.uint8)
    lut = oracle.build_lut(gs)
    for case in e["cases"]:
        prm = oracle.Params(t=case["t"], L=1, C=3, seed=SEED)
        c, lv = oracle.stylize_pixel(prm, gs, lut, gt, 0, 0)
        assert c == 0
        assert (lv == 1) == case["accept"], case


def test_threshold_t2_table(golden):
    """Accept iff D < ceil(t^2) for integer D (reading R2), checked through the oracle's
    e < t on a 1x1 image whose D is chosen around ceil(t^2)."""
    for t, T2 in golden("spec_examples.json")["t2_table"]:
        assert math.ceil(float(np.float32(t)) ** 2) == T2
        for D in {max(T2 - 1, 0), T2, T2 + 1}:
            # realise D as a sum of <= 4 squares of bytes (channels 0..3)
            parts, rem = [], D
            for _ in range(4):
                a = min(255, math.isqrt(rem))
                parts.append(a)
                rem -= a * a
            if rem:
                continue
            gt = np.array([[parts]], np.uint8)
            gs = np.zeros((1, 1, 4), np.uint8)
            prm = oracle.Params(t=t, L=1, C=4, seed=SEED)
            _, lv = oracle.stylize_pixel(prm, gs, oracle.build_lut(gs), gt, 0, 0)
            assert (lv == 1) == (D < T2), (t, D)


def test_channel_count_masks_distance():
    """R18: C=2 ignores channels 2,3; C=3 counts channel 2."""
    gt = np.array([[[10, 10, 200, 0]]], np.uint8)
    gs = np.array([[[10, 10, 0, 0]]], np.uint8)
    lut = oracle.build_lut(gs)
    assert oracle.stylize_pixel(oracle.Params(t=1, L=1, C=2), gs, lut, gt, 0, 0)[1] == 1
    assert oracle.stylize_pixel(oracle.Params(t=1, L=1, C=3), gs, lut, gt, 0, 0)[1] == 0


# ------------------------------------------------------------------ Alg. 2 closed forms
def _injective_uv(W, H):
    g = np.zeros((H, W, 4), np.uint8)
    g[..., 0] = (np.arange(W) * (256 // W))[None, :]
    g[..., 1] = (np.arange(H) * (256 // H))[:, None]
    return g


@pytest.mark.parametrize("L,t", [(3, 0.5), (5, 1.0), (5, 100.0), (4, 1000.0)])
def test_identity_transfer(L, t):
    """G_T = G_S injective, t > 0 -> every pixel copies itself at the top level
    (PAPER.md:383-387 with u* = q so s = p), borders included (R8)."""
    gs = _injective_uv(64, 64)
    cs = synth.painted_style(64, 64, seed=3).numpy()
    lut = oracle.build_lut(gs)
    ct, coords, lv = oracle.stylize(oracle.Params(t=t, L=L, C=3), cs, gs, lut, gs)
    yy, xx = np.mgrid[0:64, 0:64]
    assert (coords == (xx | (yy << 16))).all()
    assert (lv == L).all()
    assert (ct == cs).all()


@pytest.mark.parametrize("d", [(3, -5), (-7, 2), (20, 11), (0, 0)])
def test_translation_transfer(d):
    """G_T[p] = G_S[clamp(p + d)] with injective G_S and t in (0,1] (exact matches only)
    -> coords = p + d wherever p + d lies inside the source, at any level (the fallback is
    exact too)."""
    W = H = 64
    gs = _injective_uv(W, H)
    yy, xx = np.mgrid[0:H, 0:W]
    sx, sy = np.clip(xx + d[0], 0, W - 1), np.clip(yy + d[1], 0, H - 1)
    gt = np.ascontiguousarray(gs[sy, sx])
    lut = oracle.build_lut(gs)
    cs = synth.painted_style(W, H).numpy()
    for L in (3, 5):
        _, coords, lv = oracle.stylize(oracle.Params(t=1.0, L=L, C=3), cs, gs, lut, gt)
        inside = (xx + d[0] >= 0) & (xx + d[0] < W) & (yy + d[1] >= 0) & (yy + d[1] < H)
        want = (xx + d[0]) | ((yy + d[1]) << 16)
        assert (coords[inside] == want[inside]).all()


def test_t_zero_is_lit_sphere():
    """t = 0: e < 0 never holds (strict), every pixel falls back to level 0 with
    s = LUT[G_T[p]] -- the Lit Sphere / environment-map transfer (R12)."""
    cfg, cs, gs, gt = synth.config(1)
    cs, gs, gt = cs.numpy(), gs.numpy(), gt.numpy()
    lut = oracle.build_lut(gs)
    ct, coords, lv = oracle.stylize(oracle.Params(t=0.0, L=3, C=3), cs, gs, lut, gt)
    assert (lv == 0).all()
    key = gt[..., 0].astype(np.uint32) | (gt[..., 1].astype(np.uint32) << 8)
    assert (coords == lut[key]).all()
    c = coords
    assert (ct == cs[c >> 16, c & 0xFFFF]).all()


def _cfg1(t=None):
    cfg, cs, gs, gt = synth.config(1)
    cs, gs, gt = cs.numpy(), gs.numpy(), gt.numpy()
    lut = oracle.build_lut(gs)
    prm = oracle.Params(t=cfg["t"] if t is None else t, L=cfg["L"], C=cfg["C"], seed=cfg["seed"])
    return prm, cs, gs, gt, lut


def test_error_bound_and_seed_pixel():
    """(v) Error bound: level >= 1 => s inside the source and
    ||G_T[p] - G_S[s]|| < t, recomputed independently here.  (iv) Seed pixel: if the
    (clamped) nearest seed at the accepting level is p itself, s = LUT[G_T[p]]."""
    prm, cs, gs, gt, lut = _cfg1()
    ct, coords, lv = oracle.stylize(prm, cs, gs, lut, gt)
    H, W = lv.shape
    sx, sy = (coords & 0xFFFF).astype(np.int64), (coords >> 16).astype(np.int64)
    assert (sx < gs.shape[1]).all() and (sy < gs.shape[0]).all()
    acc = lv > 0
    D = ((gt[..., :3].astype(np.int64) - gs[sy, sx][..., :3].astype(np.int64)) ** 2).sum(-1)
    assert (np.sqrt(D[acc]) < prm.t).all()
    assert 0.3 < acc.mean() < 1.0  # the test is not vacuous
    n_seed = 0
    for py in range(H):
        for px in range(W):
            l = int(lv[py, px])
            if l == 0:
                continue
            qx, qy = oracle.nearest_seed(px, py, l, prm.seed)
            if (min(max(qx, 0), W - 1), min(max(qy, 0), H - 1)) == (px, py):
                n_seed += 1
                assert coords[py, px] == lut[int(gt[py, px, 0]) | (int(gt[py, px, 1]) << 8)]
    assert n_seed > 0


def test_level_zero_is_lookup():
    prm, cs, gs, gt, lut = _cfg1(t=12.0)
    _, coords, lv = oracle.stylize(prm, cs, gs, lut, gt)
    key = gt[..., 0].astype(np.uint32) | (gt[..., 1].astype(np.uint32) << 8)
    z = lv == 0
    assert z.any()
    assert (coords[z] == lut[key][z]).all()


def test_monotone_in_t():
    """Each level's candidate is independent of t and the test is monotone in t, so a
    larger t accepts at the same or a coarser level; where levels agree coords agree;
    the fallback set shrinks (PAPER.md:431-433 'higher threshold gives rise to larger
    chunks')."""
    prev = None
    for t in (4.0, 8.0, 16.0, 32.0, 64.0):
        prm, cs, gs, gt, lut = _cfg1(t=t)
        _, coords, lv = oracle.stylize(prm, cs, gs, lut, gt)
        if prev is not None:
            pc, pl = prev
            assert (lv >= pl).all()
            same = lv == pl
            assert (coords[same] == pc[same]).all()
            assert (lv == 0).sum() <= (pl == 0).sum()
        prev = (coords, lv)


def test_chunk_coherence():
    """Pixels accepted at the same level with the same nearest seed share the offset
    s - p = u* - q."""
    prm, cs, gs, gt, lut = _cfg1()
    _, coords, lv = oracle.stylize(prm, cs, gs, lut, gt)
    H, W = lv.shape
    groups = {}
    for py in range(H):
        for px in range(W):
            l = int(lv[py, px])
            if l == 0:
                continue
            q = oracle.nearest_seed(px, py, l, prm.seed)
            off = (int(coords[py, px] & 0xFFFF) - px, int(coords[py, px] >> 16) - py)
            groups.setdefault((l, q), set()).add(off)
    assert all(len(v) == 1 for v in groups.values())
    assert len(groups) < H * W / 4  # chunks are genuinely multi-pixel


def test_reseed_changes_mosaic_only():
    """Per-frame reseeding (R19): a different seed changes the mosaic; the
    same seed reproduces it bit for bit."""
    prm, cs, gs, gt, lut = _cfg1()
    a = oracle.stylize(prm, cs, gs, lut, gt)[1]
    b = oracle.stylize(prm, cs, gs, lut, gt)[1]
    prm2 = oracle.Params(t=prm.t, L=prm.L, C=prm.C, seed=prm.seed + 1)
    c = oracle.stylize(prm2, cs, gs, lut, gt)[1]
    assert (a == b).all() and (a != c).any()


def test_stylize_threads_identical():
    prm, cs, gs, gt, lut = _cfg1()
    r1 = oracle.stylize(prm, cs, gs, lut, gt, nthreads=1)
    r8 = oracle.stylize(prm, cs, gs, lut, gt, nthreads=8)
    for a, b in zip(r1, r8):
        assert (a == b).all()


# ------------------------------------------------------------------ vote
def test_vote_hand_example(golden):
    g = golden("vote_hand.json")
    cs = np.array([[[10 * x + 1, 20 * x + 3, 255 - 7 * x, 200 + x] for x in range(9)]], np.uint8)
    coords = np.array([[x if x < 4 else x + 1 for x in range(8)]], np.uint32)
    ct = oracle.vote(coords, cs, 1)
    for x, v in g["expected"].items():
        assert list(ct[0, int(x)]) == v


def _numpy_vote(coords, cs, r):
    """Independent vectorised voting: for each window offset (dx,dy) shift the offset field."""
    H, W = coords.shape
    hs, ws = cs.shape[:2]
    ox = (coords & 0xFFFF).astype(np.int64) - np.arange(W)[None, :]
    oy = (coords >> 16).astype(np.int64) - np.arange(H)[:, None]
    yy, xx = np.mgrid[0:H, 0:W]
    acc = np.zeros((H, W, 4), np.int64)
    n = np.zeros((H, W), np.int64)
    for dy in range(-r, r + 1):
        for dx in range(-r, r + 1):
            qx, qy = xx + dx, yy + dy
            ok = (qx >= 0) & (qx < W) & (qy >= 0) & (qy < H)
            qxc, qyc = np.clip(qx, 0, W - 1), np.clip(qy, 0, H - 1)
            sx, sy = xx + ox[qyc, qxc], yy + oy[qyc, qxc]
            ok &= (sx >= 0) & (sx < ws) & (sy >= 0) & (sy < hs)
            c = cs[np.clip(sy, 0, hs - 1), np.clip(sx, 0, ws - 1)].astype(np.int64)
            acc += np.where(ok[..., None], c, 0)
            n += ok
    return ((acc + (n // 2)[..., None]) // n[..., None]).astype(np.uint8)


@pytest.mark.parametrize("r", [0, 1, 2, 3])
def test_vote_matches_vectorised_bruteforce(r):
    """SPEC acceptance 3: vote equals a direct O(N (2r+1)^2) computation on 16x16 fields,
    exactly, including contributions outside the source (skipped) and clipped windows."""
    rng = np.random.RandomState(r)
    cs = rng.randint(0, 256, (12, 14, 4)).astype(np.uint8)
    W = H = 16
    cx = rng.randint(0, 14, (H, W)).astype(np.uint32)
    cy = rng.randint(0, 12, (H, W)).astype(np.uint32)
    # a few big coherent chunks plus noise
    cx[:8, :8] = np.clip(np.arange(8)[None, :] + 3, 0, 13)
    coords = np.ascontiguousarray(cx | (cy << 16))
    assert (oracle.vote(coords, cs, r) == _numpy_vote(coords, cs, r)).all()


def test_vote_r0_and_uniform_offset_equal_blit():
    """r = 0 is the blit; a single global offset gives unanimous votes = blit (SPEC
    S:273-275); interior of a chunk = blit."""
    prm, cs, gs, gt, lut = _cfg1()
    ct, coords, _ = oracle.stylize(prm, cs, gs, lut, gt)
    assert (oracle.vote(coords, cs, 0) == ct).all()
    H, W = 40, 50
    yy, xx = np.mgrid[0:H, 0:W]
    uni = ((xx + 5) | ((yy + 7) << 16)).astype(np.uint32)
    blit = cs[yy + 7, xx + 5]
    for r in (1, 2, 4):
        assert (oracle.vote(uni, cs, r) == blit).all()


def test_vote_threads_identical():
    prm, cs, gs, gt, lut = _cfg1()
    _, coords, _ = oracle.stylize(prm, cs, gs, lut, gt)
    assert (oracle.vote(coords, cs, 2, 1) == oracle.vote(coords, cs, 2, 5)).all()


# ------------------------------------------------------------------ NEXT #1: weighted guides, segmentation
def test_weighted_3_4_5():
    """Weighted error e^2 = sum w_c d_c^2 (SPEC compose_guides): (153,204) vs (0,0)
    with w = (4,1): e^2 = 4*153^2 + 204^2 = 135252, e = 367.77 -> reject at t = 367, accept at 368."""
    gt = np.array([[[153, 204, 0, 0]]], np.uint8)
    gs = np.zeros((1, 1, 4), np.uint8)
    lut = oracle.build_lut(gs)
    for t, ok in ((367.0, False), (368.0, True)):
        prm = oracle.Params(t=t, L=1, C=2, weights=(4, 1, 1, 1))
        assert (oracle.stylize_pixel(prm, gs, lut, gt, 0, 0)[1] == 1) == ok


def test_zero_weight_equals_fewer_channels():
    """w_2 = 0 with C = 3 is C = 2 (a dropped channel), on a whole frame."""
    prm, cs, gs, gt, lut = _cfg1(t=20.0)
    a = oracle.stylize(oracle.Params(t=20.0, L=3, C=3, weights=(1, 1, 0, 1)), cs, gs, lut, gt)
    b = oracle.stylize(oracle.Params(t=20.0, L=3, C=2), cs, gs, lut, gt)
    c = oracle.stylize(oracle.Params(t=20.0, L=3, C=3), cs, gs, lut, gt)
    assert all((x == y).all() for x, y in zip(a, b))
    assert any((x != y).any() for x, y in zip(a, c))  # the channel mattered without the weight


def test_segmentation_never_crosses_labels():
    """with a segmentation label no accepted chunk crosses a region
    boundary -- every pixel accepted at a level >= 1 copies from a source pixel with its own
    label, even at a threshold that accepts everything else; the label byte is not part of e."""
    W = H = 64
    gs = synth.uv_identity(W, H, labels=True).numpy()
    gt = synth.warp_uv(W, H, seed=4, amp=200.0, sigma=200.0).numpy()  # ~12 px displacements at 64^2
    gt[..., 3] = synth.uv_identity(W, H, labels=True).numpy()[..., 3]  # regions of the target frame
    cs = synth.painted_style(W, H).numpy()
    lut = oracle.build_lut(gs)
    prm_nolab = oracle.Params(t=1000.0, L=4, C=2)
    prm_lab = oracle.Params(t=1000.0, L=4, C=2, label_channel=3)
    _, c0, l0 = oracle.stylize(prm_nolab, cs, gs, lut, gt)
    _, c1, l1 = oracle.stylize(prm_lab, cs, gs, lut, gt)
    sx, sy = c1 & 0xFFFF, c1 >> 16
    acc = l1 > 0
    assert (gs[sy, sx, 3][acc] == gt[..., 3][acc]).all()
    sx0, sy0 = c0 & 0xFFFF, c0 >> 16
    assert (gs[sy0, sx0, 3][l0 > 0] != gt[..., 3][l0 > 0]).any()  # without labels chunks do cross
    # the label byte does not enter e: with equal labels everywhere the result is unchanged
    gt2, gs2 = gt.copy(), gs.copy()
    gt2[..., 3] = 7
    gs2[..., 3] = 7
    a = oracle.stylize(oracle.Params(t=9.0, L=4, C=4, label_channel=3), cs, gs2, lut, gt2)
    b = oracle.stylize(oracle.Params(t=9.0, L=4, C=3), cs, gs2, lut, gt2)
    assert all((x == y).all() for x, y in zip(a, b))


# ------------------------------------------ exact 3-channel guide search (R26)
def _numpy_lut3_bruteforce(gs, keys):
    """Independent: vectorised 3-channel squared distances, np.argmin = first row-major min."""
    hs, ws = gs.shape[:2]
    g = gs[..., :3].reshape(-1, 3).astype(np.int64)
    out = []
    for k in keys:
        kk = np.array([k & 0xFF, (k >> 8) & 0xFF, (k >> 16) & 0xFF], np.int64)
        i = int(np.argmin(((g - kk) ** 2).sum(1)))
        out.append((i % ws) | ((i // ws) << 16))
    return np.array(out, np.uint32)


@pytest.mark.parametrize("ws,hs,vmax", [(7, 5, 256), (16, 16, 4), (24, 20, 256), (9, 31, 2)])
def test_lut3_bruteforce_tiny(ws, hs, vmax):
    rng = np.random.RandomState(ws * 31 + hs)
    gs = rng.randint(0, vmax, (hs, ws, 4)).astype(np.uint8)
    keys = rng.randint(0, 1 << 24, 500).astype(np.uint32)
    keys = np.concatenate([keys, np.array([0, 0xFFFFFF, 0x00FF00, 0xFF00FF], np.uint32)])
    ref = _numpy_lut3_bruteforce(gs, keys)
    assert (oracle.lut3_entries(gs, keys, nthreads=3) == ref).all()
    for k, r in list(zip(keys, ref))[:40]:
        assert oracle.lut3_entry(gs, int(k) & 0xFF, (int(k) >> 8) & 0xFF, (int(k) >> 16) & 0xFF) == r


def test_lut3_lattice_closed_form():
    """G_S = the 4^3 lattice {0,85,170,255}^3 (8x8 pixels, a shuffled order): the nearest
    lattice point rounds each channel to the nearest multiple of 85 (85 is odd, so no integer
    key is half-way: unique), and u* is where that point sits."""
    rng = np.random.RandomState(7)
    pts = np.array([(a, b, c) for a in range(4) for b in range(4) for c in range(4)]) * 85
    perm = rng.permutation(64)
    gs = np.zeros((8, 8, 4), np.uint8)
    gs[..., :3] = pts[perm].reshape(8, 8, 3)
    gs[..., 3] = rng.randint(0, 256, (8, 8))  # ignored
    where = {tuple(pts[perm[i]]): i for i in range(64)}
    keys = rng.randint(0, 1 << 24, 2000).astype(np.uint32)
    got = oracle.lut3_entries(gs, keys)
    for k, u in zip(keys, got):
        g = np.array([k & 0xFF, (k >> 8) & 0xFF, (k >> 16) & 0xFF])
        i = where[tuple((np.floor(g / 85.0 + 0.5) * 85).astype(int))]
        assert u == ((i % 8) | ((i // 8) << 16))


def test_lut3_reduces_to_lut_when_channel2_constant():
    """A constant channel 2 adds the same (k2 - c)^2 to every pixel: same argmin, same tie
    rule, so the 3-channel search equals the 2-channel table for every k2."""
    rng = np.random.RandomState(11)
    gs = rng.randint(0, 6, (12, 14, 4)).astype(np.uint8) * 40
    gs[..., 2] = 93
    lut = oracle.build_lut(gs)
    keys = rng.randint(0, 1 << 24, 3000).astype(np.uint32)
    assert (oracle.lut3_entries(gs, keys) == lut[keys & 0xFFFF]).all()


def test_stylize_lut_rgb():
    """Alg. 2 with u* from the exact 3-channel search: (a) equals the table path when channel
    2 of G_S is constant; (b) G_T = G_S with injective RGB copies every pixel at level L even
    where the first two channels alone are ambiguous (the 2-channel table cannot)."""
    rng = np.random.RandomState(3)
    W = H = 32
    cs = synth.painted_style(W, H, seed=5).numpy()
    gs = rng.randint(0, 256, (H, W, 4)).astype(np.uint8)
    gs[..., 2] = 17
    gt = rng.randint(0, 256, (H, W, 4)).astype(np.uint8)
    lut = oracle.build_lut(gs)
    a = oracle.stylize(oracle.Params(t=60.0, L=3, C=3), cs, gs, lut, gt)
    b = oracle.stylize(oracle.Params(t=60.0, L=3, C=3, lut_rgb=True), cs, gs, None, gt)
    assert all((x == y).all() for x, y in zip(a, b))
    # (b): channels 0,1 take only 4 values (massively ambiguous), channel 2 makes RGB injective
    gs2 = np.zeros((H, W, 4), np.uint8)
    idx = rng.permutation(W * H).reshape(H, W)
    gs2[..., 0] = (idx % 4) * 60
    gs2[..., 1] = ((idx // 4) % 4) * 60
    gs2[..., 2] = idx // 16 * 4
    _, coords, lv = oracle.stylize(oracle.Params(t=0.5, L=3, C=3, lut_rgb=True), cs, gs2, None, gs2)
    yy, xx = np.mgrid[0:H, 0:W]
    assert (coords == (xx | (yy << 16))).all() and (lv == 3).all()
    _, coords2, _ = oracle.stylize(oracle.Params(t=0.5, L=3, C=3), cs, gs2, oracle.build_lut(gs2), gs2)
    assert (coords2 != coords).any()
