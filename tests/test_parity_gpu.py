"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star): LUT, source-coordinate maps and levels bit-exact; blit colours
bit-exact; voted colours within max-abs 1/255 -- the integer vote is in fact checked
bit-exact here.  Inputs are the seeded synthetic configs of synth/ plus edge cases.
"""
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


def u32(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


_lut_cache = {}


def oracle_lut(gs: np.ndarray) -> np.ndarray:
    key = (gs.shape, gs.tobytes().__hash__())
    if key not in _lut_cache:
        _lut_cache[key] = oracle.build_lut(gs, nthreads=NTH)
    return _lut_cache[key]


def run_both(prm: sb.Params, cs, gs, gt, want_vote=True):
    """Run GPU and oracle on identical bytes; return dict of arrays."""
    csd, gsd, gtd = cs.to(DEV), gs.to(DEV), gt.to(DEV)
    lut_d = sb.build_lut(gsd)
    ct, coords, level = sb.stylize(prm, csd, gsd, lut_d, gtd)
    # the strided exemplar copy (sb_prepare_exemplar) is a speed option: identical results
    ex = sb.prepare_exemplar(csd, gsd)
    ct2, coords2, level2 = sb.stylize(sb.Params(**{**prm.__dict__, "exemplar": ex}), csd, gsd, lut_d, gtd)
    torch.cuda.synchronize()
    assert torch.equal(coords, coords2) and torch.equal(level, level2), "exemplar copy changed coords/levels"
    assert (ct is None and ct2 is None) or torch.equal(ct, ct2), "exemplar copy changed colours"
    csn, gsn, gtn = cs.numpy(), gs.numpy(), gt.numpy()
    lut = oracle_lut(gsn)
    oprm = oracle.Params(t=prm.threshold, L=prm.levels, C=prm.guide_channels, seed=prm.seed,
                         zero_jitter=bool(prm.flags & sb.SB_JITTER_ZERO))
    oct_, oco, olv = oracle.stylize(oprm, csn, gsn, lut, gtn, nthreads=NTH)
    if prm.blend_radius > 0:
        oct_ = oracle.vote(oco, csn, prm.blend_radius, nthreads=NTH)
    return dict(lut=(u32(lut_d), lut), coords=(u32(coords), oco), level=(level.cpu().numpy(), olv),
                ct=(ct.cpu().numpy(), oct_))


def assert_exact(res, name):
    g, o = res[name]
    if not (g == o).all():
        bad = np.argwhere(g != o)
        raise AssertionError(f"{name}: {len(bad)} mismatches, first at {bad[:5].tolist()}: gpu {g[tuple(bad[0])]} "
                             f"oracle {o[tuple(bad[0])]}")


# ------------------------------------------------------------------ LUT
@pytest.mark.parametrize("kind", ["sphere64", "sphere512", "uv256", "uv1024", "const", "rand_small", "rand_few"])
def test_lut_all_keys(kind):
    rng = np.random.RandomState(7)
    if kind == "sphere64":
        gs = synth.sphere_normal(64, 64)
    elif kind == "sphere512":
        gs = synth.sphere_normal(512, 512)
    elif kind == "uv256":
        gs = synth.uv_identity(256, 256)
    elif kind == "uv1024":
        gs = synth.uv_identity(1024, 1024)
    elif kind == "const":
        gs = torch.full((17, 9, 4), 200, dtype=torch.uint8)
    elif kind == "rand_small":
        gs = torch.from_numpy(rng.randint(0, 256, (5, 7, 4)).astype(np.uint8))
    else:  # few distinct values, many ties
        gs = torch.from_numpy((rng.randint(0, 3, (40, 33, 4)) * 100).astype(np.uint8))
    gsn = gs.numpy()
    got = u32(sb.build_lut(gs.to(DEV)))
    if gsn.shape[0] * gsn.shape[1] <= 512 * 512:
        want = oracle_lut(gsn)
        assert (got == want).all(), np.argwhere(got != want)[:5]
    else:  # 1024^2: sampled keys, each by the oracle's definition
        for k in np.random.RandomState(1).randint(0, 65536, 300).tolist() + [0, 65535]:
            assert got[k] == oracle.lut_entry(gsn, k & 0xFF, k >> 8), k


# ------------------------------------------------------------------ configs 1-4 full frames
@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_config_parity(cid):
    cfg = synth.CONFIGS[cid]
    cs, gs = synth.exemplar(cfg)
    gt = synth.target(cid)
    for r in sorted({0, cfg["r"]}):
        prm = sb.Params(threshold=cfg["t"], levels=cfg["L"], blend_radius=r, guide_channels=cfg["C"], seed=cfg["seed"])
        res = run_both(prm, cs, gs, gt)
        for n in ("lut", "coords", "level", "ct"):
            assert_exact(res, n)
        lv = res["level"][1]
        assert (lv == cfg["L"]).mean() > 0.3 and (lv < cfg["L"]).any()  # the hierarchy is exercised


# ------------------------------------------------------------------ edge cases
def _rand_case(wt, ht, ws, hs, seed, C=3, vmax=256):
    rng = np.random.RandomState(seed)
    gs = synth.sphere_normal(ws, hs)
    cs = torch.from_numpy(rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8))
    gt = synth.heightfield_normals(wt, ht, seed=seed)
    return cs, gs, gt


@pytest.mark.parametrize("wt,ht", [(1, 1), (3, 5), (4, 1), (130, 17), (127, 33), (132, 16), (256, 48), (8, 300)])
@pytest.mark.parametrize("L", [1, 2, 5])
def test_ragged_sizes(wt, ht, L):
    """Tile-ragged widths/heights, widths not divisible by 4 (one-thread-per-pixel kernel),
    single-pixel images, L = 1 (no top-level group pass)."""
    cs, gs, gt = _rand_case(wt, ht, 48, 40, seed=wt * 1000 + ht)
    for r in (0, 2):
        prm = sb.Params(threshold=14.0, levels=L, blend_radius=r, guide_channels=3, seed=99)
        res = run_both(prm, cs, gs, gt)
        for n in ("coords", "level", "ct"):
            assert_exact(res, n)


@pytest.mark.parametrize("t", [0.0, 0.5, 1.0, 6.0, 1000.0])
@pytest.mark.parametrize("C", [2, 3, 4])
def test_thresholds_and_channels(t, C):
    cs, gs, gt = _rand_case(200, 72, 64, 64, seed=5)
    gt = gt.clone()
    gt[..., 3] = torch.from_numpy(np.random.RandomState(3).randint(0, 4, gt.shape[:2]).astype(np.uint8))
    prm = sb.Params(threshold=t, levels=4, blend_radius=0, guide_channels=C, seed=7)
    res = run_both(prm, cs, gs, gt)
    for n in ("coords", "level", "ct"):
        assert_exact(res, n)
    if t == 0.0:
        assert (res["level"][0] == 0).all()


@pytest.mark.parametrize("L", [3, 8, 12])
def test_zero_jitter_and_deep_hierarchies(L):
    cs, gs, gt = _rand_case(256, 96, 64, 64, seed=11)
    for flags in (0, sb.SB_JITTER_ZERO):
        prm = sb.Params(threshold=9.0, levels=L, blend_radius=1, guide_channels=3, seed=3, flags=flags)
        res = run_both(prm, cs, gs, gt)
        for n in ("coords", "level", "ct"):
            assert_exact(res, n)


@pytest.mark.parametrize("r", [1, 3, 7])
def test_vote_radii(r):
    cfg = synth.CONFIGS[2]
    cs, gs = synth.exemplar(cfg)
    gt = synth.render_objects(256, 160, seed=2)
    prm = sb.Params(threshold=cfg["t"], levels=5, blend_radius=r, guide_channels=3, seed=cfg["seed"])
    res = run_both(prm, cs, gs, gt)
    assert_exact(res, "coords")
    g, o = res["ct"]
    assert np.abs(g.astype(int) - o.astype(int)).max() <= 1  # north-star tolerance (1/255)
    assert_exact(res, "ct")  # the integer vote is in fact exact


def test_identity_transfer_gpu():
    """G_T = G_S injective -> coords = p, level = L, C_T = C_S."""
    g = np.zeros((64, 64, 4), np.uint8)
    g[..., 0] = (np.arange(64) * 4)[None, :]
    g[..., 1] = (np.arange(64) * 4)[:, None]
    gs = torch.from_numpy(g)
    cs = synth.painted_style(64, 64)
    prm = sb.Params(threshold=0.5, levels=5, blend_radius=2, guide_channels=3)
    ct, coords, lv = sb.stylize(prm, cs.to(DEV), gs.to(DEV), sb.build_lut(gs.to(DEV)), gs.to(DEV))
    yy, xx = np.mgrid[0:64, 0:64]
    assert (u32(coords) == (xx | (yy << 16))).all()
    assert (lv.cpu().numpy() == 5).all()
    assert (ct.cpu().numpy() == cs.numpy()).all()


# ------------------------------------------------------------------ batch, strips, determinism
def test_batch_equals_single_frames():
    cfg = synth.CONFIGS[2]
    cs, gs = [t.to(DEV) for t in synth.exemplar(cfg)]
    lut = sb.build_lut(gs)
    frames = torch.stack([synth.heightfield_normals(320, 200, seed=9, frame=i) for i in range(5)]).to(DEV)
    for r in (0, 2):
        prm = sb.Params(threshold=10.0, levels=5, blend_radius=r, guide_channels=3, seed=100)
        seeds = [100, 7, 7, 0xFFFFFFFF, 12345]
        bct, bco, blv = sb.stylize_batch(prm, cs, gs, lut, frames, frame_seeds=seeds)
        dct, dco, dlv = sb.stylize_batch(prm, cs, gs, lut, frames)  # default seeds prm.seed + i
        for i in range(5):
            p1 = sb.Params(**{**prm.__dict__, "seed": seeds[i]})
            ct, co, lv = sb.stylize(p1, cs, gs, lut, frames[i])
            assert torch.equal(ct, bct[i]) and torch.equal(co, bco[i]) and torch.equal(lv, blv[i])
            p2 = sb.Params(**{**prm.__dict__, "seed": (100 + i) & 0xFFFFFFFF})
            ct, co, lv = sb.stylize(p2, cs, gs, lut, frames[i])
            assert torch.equal(ct, dct[i]) and torch.equal(co, dco[i])
        assert torch.equal(bco[1], bco[2]) or not torch.equal(frames[1], frames[2])


def test_oracle_parity_batch_frames():
    """Per-frame seeds reach the jitter: oracle with the same seed per frame."""
    cfg = synth.CONFIGS[1]
    cs, gs = synth.exemplar(cfg)
    frames = torch.stack([synth.heightfield_normals(64, 64, seed=1, frame=i) for i in range(3)])
    seeds = [5, 6, 0xDEADBEEF]
    prm = sb.Params(threshold=cfg["t"], levels=3, blend_radius=0, guide_channels=3, seed=0)
    gsd = gs.to(DEV)
    ct, co, lv = sb.stylize_batch(prm, cs.to(DEV), gsd, sb.build_lut(gsd), frames.to(DEV), frame_seeds=seeds)
    lut = oracle_lut(gs.numpy())
    for i in range(3):
        o = oracle.stylize(oracle.Params(t=cfg["t"], L=3, C=3, seed=seeds[i]), cs.numpy(), gs.numpy(), lut,
                           frames[i].numpy())
        assert (u32(co[i]) == o[1]).all() and (lv[i].cpu().numpy() == o[2]).all() and (ct[i].cpu().numpy() == o[0]).all()


@pytest.mark.parametrize("r", [0, 2])
def test_strips_equal_whole_frame(r):
    cfg = synth.CONFIGS[3]
    cs, gs = [t.to(DEV) for t in synth.exemplar(cfg)]
    lut = sb.build_lut(gs)
    gt = synth.heightfield_normals(640, 203, seed=3).to(DEV)
    prm = sb.Params(threshold=cfg["t"], levels=5, blend_radius=r, guide_channels=3, seed=cfg["seed"])
    ct, co, lv = sb.stylize(prm, cs, gs, lut, gt)
    for cuts in ([0, 100, 203], [0, 1, 17, 64, 150, 202, 203], [0, 203]):
        ct2 = torch.zeros_like(ct)
        lv2 = torch.zeros_like(lv)
        co2 = torch.zeros_like(co)
        for a, b in zip(cuts[:-1], cuts[1:]):
            p = sb.Params(**{**prm.__dict__, "row_begin": a, "row_end": b})
            sb.stylize(p, cs, gs, lut, gt, ct=ct2, coords=co2, level=lv2)
        assert torch.equal(ct, ct2) and torch.equal(lv, lv2) and torch.equal(co, co2)


def test_repeatable_and_no_color():
    cfg = synth.CONFIGS[2]
    cs, gs = [t.to(DEV) for t in synth.exemplar(cfg)]
    lut = sb.build_lut(gs)
    gt = synth.target(2).to(DEV)
    prm = sb.Params(threshold=cfg["t"], levels=5, blend_radius=2, guide_channels=3, seed=1)
    a = sb.stylize(prm, cs, gs, lut, gt)
    b = sb.stylize(prm, cs, gs, lut, gt)
    assert all(torch.equal(x, y) for x, y in zip(a, b))
    pn = sb.Params(**{**prm.__dict__, "flags": sb.SB_NO_COLOR})
    ct, co, lv = sb.stylize(pn, cs, gs, lut, gt)
    assert ct is None and torch.equal(co, a[1]) and torch.equal(lv, a[2])


def test_host_pipeline_equals_device_batch():
    cfg = synth.CONFIGS[3]
    cs, gs = [t.to(DEV) for t in synth.exemplar(cfg)]
    lut = sb.build_lut(gs)
    frames = torch.stack([synth.heightfield_normals(512, 288, seed=4, frame=i) for i in range(5)])
    for r in (0, 2):
        prm = sb.Params(threshold=cfg["t"], levels=5, blend_radius=r, guide_channels=3, seed=9)
        dct, dco, _ = sb.stylize_batch(prm, cs, gs, lut, frames.to(DEV))
        gt_h = frames.pin_memory()
        ct_h = torch.empty_like(gt_h).pin_memory()
        co_h = torch.empty(5, 288, 512, dtype=torch.int32).pin_memory()
        sb.stylize_batch_host(prm, cs, gs, lut, gt_h, ct_h, co_h, depth=2)
        assert torch.equal(ct_h, dct.cpu()) and torch.equal(co_h, dco.cpu())
        # packed-RGB host frames (SB_HOST_RGB; guide byte 3 is not read with C = 3), with the
        # strided exemplar copy: the same coordinates and the colours' channels 0..2
        prgb = sb.Params(**{**prm.__dict__, "flags": sb.SB_HOST_RGB, "exemplar": sb.prepare_exemplar(cs, gs)})
        g3 = frames[..., :3].contiguous().pin_memory()
        c3 = torch.empty_like(g3).pin_memory()
        co3 = torch.empty(5, 288, 512, dtype=torch.int32).pin_memory()
        sb.stylize_batch_host(prgb, cs, gs, lut, g3, c3, co3, depth=3)
        assert torch.equal(c3, dct.cpu()[..., :3]) and torch.equal(co3, dco.cpu())


def test_naive_kernel_agrees(tmp_path):
    """The one-thread-per-pixel kernel (SB_KERNEL=naive) and the tiled kernel agree (run in a
    subprocess so the environment switch takes effect)."""
    import subprocess
    import sys

    code = (
        "import torch, numpy as np, synth, paper_1807_03249_b200 as sb\n"
        "cfg=synth.CONFIGS[2]; cs,gs=[t.cuda() for t in synth.exemplar(cfg)]; lut=sb.build_lut(gs)\n"
        "gt=synth.target(2).cuda()\n"
        "p=sb.Params(threshold=cfg['t'],levels=5,blend_radius=2,guide_channels=3,seed=4)\n"
        "ct,co,lv=sb.stylize(p,cs,gs,lut,gt); torch.cuda.synchronize()\n"
        "np.save(r'%s', np.concatenate([co.cpu().numpy().ravel(), ct.cpu().numpy().view(np.int32).ravel(), lv.cpu().numpy().astype(np.int32).ravel()]))\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mode in ("tiled", "naive"):
        f = tmp_path / f"{mode}.npy"
        env = dict(os.environ, SB_KERNEL=mode, PYTHONPATH=root)
        subprocess.check_call([sys.executable, "-c", code % f], env=env, cwd=root)
        outs.append(np.load(f))
    if not (outs[0] == outs[1]).all():
        n = outs[0].size // 3  # coords, ct, level: n each
        names = ["coords", "ct", "level"]
        bad = np.nonzero(outs[0] != outs[1])[0]
        where = [names[min(i // n, 2)] for i in bad[:10]]
        raise AssertionError(f"{bad.size} mismatches; first {bad[:10].tolist()} in {where}: "
                             f"tiled {outs[0][bad[:10]].tolist()} naive {outs[1][bad[:10]].tolist()}")


@pytest.mark.parametrize("cid", [1, 2, 3])
@pytest.mark.parametrize("r", [0, 2])
def test_outputs_fully_written(cid, r):
    """Every output element is written: two runs into buffers pre-filled with different bytes
    give identical results (catches unwritten pixels and reads of uninitialised memory)."""
    cfg = synth.CONFIGS[cid]
    cs, gs = [t.to(DEV) for t in synth.exemplar(cfg)]
    lut = sb.build_lut(gs)
    gt = synth.target(cid).to(DEV)
    H, W = gt.shape[:2]
    prm = sb.Params(threshold=cfg["t"], levels=cfg["L"], blend_radius=r, guide_channels=cfg["C"], seed=cfg["seed"])
    res = []
    for fill in (0x00, 0xA5):
        ct = torch.full((H, W, 4), fill, dtype=torch.uint8, device=DEV)
        co = torch.full((H, W), -1 if fill else 0, dtype=torch.int32, device=DEV)
        lv = torch.full((H, W), fill, dtype=torch.uint8, device=DEV)
        sb.stylize(prm, cs, gs, lut, gt, ct=ct, coords=co, level=lv)
        res.append((ct, co, lv))
    for a_, b_ in zip(*res):
        assert torch.equal(a_, b_)


@pytest.mark.parametrize("case", ["uv_labels", "uv_weights_labels", "normal_weights", "ragged_labels"])
def test_weighted_and_segmentation_parity(case):
    """per-channel weights and a segmentation label --
    GPU == oracle on coords, levels and colours."""
    if case.startswith("uv"):
        W = 512
        gs = synth.uv_identity(W, W, labels=True)
        cs = synth.painted_style(W, W)
        gt = synth.warp_uv(W, W, seed=4, labels=True)
        gt[..., 3] = synth.uv_identity(W, W, labels=True)[..., 3]
        kw = dict(threshold=2.5, levels=5, guide_channels=2, label_channel=3)
        okw = dict(t=2.5, L=5, C=2, label_channel=3)
        if case == "uv_weights_labels":
            kw["weights"] = (3, 1, 0, 0)
            okw["weights"] = (3, 1, 0, 0)
    elif case == "normal_weights":
        cfg = synth.CONFIGS[2]
        cs, gs = synth.exemplar(cfg)
        gt = synth.render_objects(640, 384, seed=2)
        kw = dict(threshold=20.0, levels=5, guide_channels=3, weights=(2, 1, 3, 0))
        okw = dict(t=20.0, L=5, C=3, weights=(2, 1, 3, 0))
    else:
        cs, gs, gt = _rand_case(131, 45, 48, 40, seed=3)
        gt = gt.clone()
        gs = gs.clone()
        gt[..., 3] = (torch.arange(131)[None, :] // 40 * 60).to(torch.uint8).expand(45, 131)
        gs[..., 3] = (torch.arange(48)[None, :] // 12 * 60).to(torch.uint8).expand(40, 48)
        kw = dict(threshold=30.0, levels=3, guide_channels=3, label_channel=3)
        okw = dict(t=30.0, L=3, C=3, label_channel=3)
    csd, gsd, gtd = cs.to(DEV), gs.to(DEV), gt.to(DEV)
    lut_d = sb.build_lut(gsd)
    lut = oracle_lut(gs.numpy())
    o = oracle.stylize(oracle.Params(seed=0x5EED, **okw), cs.numpy(), gs.numpy(), lut, gt.numpy(), nthreads=NTH)
    ex = sb.prepare_exemplar(csd, gsd)  # ignored by the weighted/label kernel, used by the vote
    for r, exm in ((0, None), (2, None), (0, ex), (2, ex)):
        ct, co, lv = sb.stylize(sb.Params(blend_radius=r, seed=0x5EED, exemplar=exm, **kw), csd, gsd, lut_d, gtd)
        assert (u32(co) == o[1]).all() and (lv.cpu().numpy() == o[2]).all()
        want = o[0] if r == 0 else oracle.vote(o[1], cs.numpy(), r, nthreads=NTH)
        assert (ct.cpu().numpy() == want).all()
    if "label" in case:
        sx, sy = o[1] & 0xFFFF, o[1] >> 16
        acc = o[2] > 0
        assert (gs.numpy()[sy, sx, 3][acc] == gt.numpy()[..., 3][acc]).all()


# ------------------------------------------------------------------ CUDA graph capture
def test_cuda_graph_capture_replay():
    """The ABI calls only enqueue work on the caller's stream (no allocation, no sync), so a
    whole step (LUT + strided exemplar copy + stylize + vote) can be captured into a CUDA graph and replayed: replays
    reproduce the eager result bit for bit, and follow new inputs written into the same buffers."""
    cfg = synth.CONFIGS[2]
    cs, gs = (t.to(DEV) for t in synth.exemplar(cfg))
    gt = synth.target(2).to(DEV).unsqueeze(0).repeat(3, 1, 1, 1).contiguous()
    gt[1] = torch.flip(gt[1], dims=[1])
    ex = torch.empty(sb.exemplar_bytes(gs.shape[1], gs.shape[0]), dtype=torch.uint8, device=DEV)
    prm = sb.Params(threshold=cfg["t"], levels=cfg["L"], blend_radius=2, guide_channels=cfg["C"], seed=cfg["seed"],
                    exemplar=ex)
    lut = torch.empty(65536, dtype=torch.int32, device=DEV)
    lws = torch.empty(sb.lib().sb_lut_workspace_bytes(), dtype=torch.uint8, device=DEV)
    ct = torch.empty_like(gt)
    co = torch.empty(gt.shape[:3], dtype=torch.int32, device=DEV)

    def step():
        sb.build_lut(gs, lut, lws)
        sb.prepare_exemplar(cs, gs, ex)
        sb.stylize_batch(prm, cs, gs, lut, gt, ct=ct, coords=co, want_level=False)

    step()
    torch.cuda.synchronize()
    eager_ct, eager_co = ct.clone(), co.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()  # warm-up on the side stream (kernel attributes set outside capture)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    ct.zero_()
    co.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(ct, eager_ct) and torch.equal(co, eager_co)
    gt.copy_(torch.flip(gt, dims=[2]))  # new inputs, same buffers
    g.replay()
    torch.cuda.synchronize()
    ref_ct = ct.clone()
    step()
    torch.cuda.synchronize()
    assert torch.equal(ct, ref_ct) and not torch.equal(ref_ct, eager_ct)


def test_batch_longer_than_one_launch():
    """More frames than one launch carries seeds for (512): the library splits the batch into
    launches; every frame keeps its own seed (checked against the oracle on a sample)."""
    n = 1100
    cfg = synth.CONFIGS[1]
    cs, gs = synth.exemplar(cfg)
    frames = torch.stack([synth.heightfield_normals(16, 12, seed=9, frame=i % 7) for i in range(n)])
    seeds = [(0x1234567 * i + 99) & 0xFFFFFFFF for i in range(n)]
    prm = sb.Params(threshold=cfg["t"], levels=3, guide_channels=3)
    gsd = gs.to(DEV)
    ct, co, lv = sb.stylize_batch(prm, cs.to(DEV), gsd, sb.build_lut(gsd), frames.to(DEV), frame_seeds=seeds)
    torch.cuda.synchronize()
    lut = oracle_lut(gs.numpy())
    for i in (0, 511, 512, 513, 1023, 1024, n - 1):
        o = oracle.stylize(oracle.Params(t=cfg["t"], L=3, C=3, seed=seeds[i]), cs.numpy(), gs.numpy(), lut,
                           frames[i].numpy())
        assert (u32(co[i]) == o[1]).all() and (lv[i].cpu().numpy() == o[2]).all(), i


def test_consecutive_seeds_one_launch_per_65535_frames():
    """Seeds s0 + i (default or explicit) need no parameter array: the library launches up to
    65535 frames at once (grid.z) instead of chunks of 512.  70000 tiny frames: 2 stylize
    launches; sampled frames around the 512 and 65535 boundaries agree with the oracle."""
    n = 70000
    cfg = synth.CONFIGS[1]
    cs, gs = synth.exemplar(cfg)
    base = torch.stack([synth.heightfield_normals(8, 6, seed=9, frame=i) for i in range(5)])
    frames = base[torch.arange(n) % 5]
    s0 = 0xFFFFFF00  # wraps mod 2^32 inside the batch
    seeds = [(s0 + i) & 0xFFFFFFFF for i in range(n)]
    prm = sb.Params(threshold=cfg["t"], levels=3, guide_channels=3, seed=s0)
    gsd = gs.to(DEV)
    lut_d = sb.build_lut(gsd)
    ct, co, lv = sb.stylize_batch(prm, cs.to(DEV), gsd, lut_d, frames.to(DEV), frame_seeds=seeds)
    assert sb.launch_count() == 2
    ct2, co2, lv2 = sb.stylize_batch(prm, cs.to(DEV), gsd, lut_d, frames.to(DEV))  # default seeds: the same
    torch.cuda.synchronize()
    assert torch.equal(co, co2) and torch.equal(ct, ct2) and torch.equal(lv, lv2)
    lut = oracle_lut(gs.numpy())
    for i in (0, 255, 511, 512, 513, 65534, 65535, 65536, n - 1):
        o = oracle.stylize(oracle.Params(t=cfg["t"], L=3, C=3, seed=seeds[i]), cs.numpy(), gs.numpy(), lut,
                           frames[i].numpy())
        assert (u32(co[i]) == o[1]).all() and (lv[i].cpu().numpy() == o[2]).all(), i


# ------------------------------------------------------------------ strided exemplar copy
def test_prepare_exemplar_layout():
    """sb_prepare_exemplar: G_S then C_S, each hs rows of 2^16 pixels (include/styleblit.h)."""
    cs, gs, _ = _rand_case(8, 8, 37, 29, seed=3)   # ws not a multiple of 4
    csd, gsd = cs.to(DEV), gs.to(DEV)
    ex = sb.prepare_exemplar(csd, gsd)
    assert ex.numel() == 2 * 29 * (1 << 18)
    rows = ex.view(2, 29, 65536, 4)[:, :, :37, :].cpu()
    assert torch.equal(rows[0], gs) and torch.equal(rows[1], cs)


@pytest.mark.parametrize("L", [3, 4, 5])
def test_exemplar_copy_batch_and_strips(L):
    """With the strided exemplar copy: a batch with per-frame seeds and row strips equal the
    oracle / the whole-frame result (the kernels that use it: L = 3..5)."""
    cfg = synth.CONFIGS[3]
    cs, gs = [t.to(DEV) for t in synth.exemplar(cfg)]
    lut = sb.build_lut(gs)
    ex = sb.prepare_exemplar(cs, gs)
    frames = torch.stack([synth.heightfield_normals(260, 70, seed=5, frame=i) for i in range(3)]).to(DEV)
    prm = sb.Params(threshold=cfg["t"], levels=L, guide_channels=3, seed=11, exemplar=ex)
    ct, co, lv = sb.stylize_batch(prm, cs, gs, lut, frames)
    lutn = oracle_lut(gs.cpu().numpy())
    for i in range(3):
        o = oracle.stylize(oracle.Params(t=cfg["t"], L=L, C=3, seed=11 + i), cs.cpu().numpy(), gs.cpu().numpy(), lutn,
                           frames[i].cpu().numpy(), nthreads=NTH)
        assert (u32(co[i]) == o[1]).all() and (lv[i].cpu().numpy() == o[2]).all() and (ct[i].cpu().numpy() == o[0]).all()
    ct2 = torch.zeros_like(ct[0])
    for a, b in zip([0, 3, 37, 70][:-1], [0, 3, 37, 70][1:]):
        sb.stylize(sb.Params(**{**prm.__dict__, "seed": 11, "row_begin": a, "row_end": b}), cs, gs, lut, frames[0],
                   ct=ct2)
    assert torch.equal(ct2, ct[0])


@pytest.mark.parametrize("r", [1, 2, 3, 4, 5, 6, 7])
def test_vote_exemplar_copy(r):
    """sb_vote with the strided exemplar copy equals sb_vote without it and the oracle, on a
    coordinate field with chunk seams, frame borders and sources at the exemplar border."""
    rng = np.random.RandomState(r)
    ws, hs, wt, ht = 61, 47, 264, 40
    cs = torch.from_numpy(rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8))
    gs = torch.from_numpy(rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8))
    # chunked field: 8x8 chunks copying random source blocks (some touching the source border)
    yy, xx = np.mgrid[0:ht, 0:wt]
    ox = rng.randint(-10, ws - 2, (ht // 8 + 1, wt // 8 + 1))
    oy = rng.randint(-10, hs - 2, (ht // 8 + 1, wt // 8 + 1))
    sx = np.clip(xx % 8 + ox[yy // 8, xx // 8], 0, ws - 1)
    sy = np.clip(yy % 8 + oy[yy // 8, xx // 8], 0, hs - 1)
    co = (sx | (sy << 16)).astype(np.uint32)
    csd, gsd = cs.to(DEV), gs.to(DEV)
    cod = torch.from_numpy(co.view(np.int32)).to(DEV)
    ex = sb.prepare_exemplar(csd, gsd)
    a = sb.vote(cod, csd, r)
    b = sb.vote(cod, csd, r, exemplar=ex)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert (b.cpu().numpy() == oracle.vote(co, cs.numpy(), r, nthreads=NTH)).all()


@pytest.mark.parametrize("r", [1, 2])
@pytest.mark.parametrize("chunk", [1, 2, 3, 5, 8, 32])
def test_vote_peel_distinct_offsets(r, chunk):
    """The peel vote (r = 1, 2; vote_peel.cu) against the oracle on fields whose 4x4-block
    unions hold from one to (4+2r)^2 distinct offsets: chunk x chunk squares copying random
    source blocks, sources kept >= r from the exemplar border so most tiles take the fast
    path (chunk = 1: every position its own offset, the position-by-position leftovers after
    KMAX peels); a frame border and a ragged width exercise the border tiles."""
    rng = np.random.RandomState(100 * r + chunk)
    ws, hs = 200, 180
    cs = torch.from_numpy(rng.randint(0, 256, (hs, ws, 4)).astype(np.uint8))
    gs = torch.zeros((hs, ws, 4), dtype=torch.uint8)
    csd, gsd = cs.to(DEV), gs.to(DEV)
    ex = sb.prepare_exemplar(csd, gsd)
    for wt, ht in ((384, 48), (261, 37)):
        yy, xx = np.mgrid[0:ht, 0:wt]
        nby, nbx = ht // chunk + 1, wt // chunk + 1
        ox = rng.randint(r, ws - chunk - r, (nby, nbx))
        oy = rng.randint(r, hs - chunk - r, (nby, nbx))
        sx = xx % chunk + ox[yy // chunk, xx // chunk]
        sy = yy % chunk + oy[yy // chunk, xx // chunk]
        co = (sx | (sy << 16)).astype(np.uint32)
        cod = torch.from_numpy(co.view(np.int32)).to(DEV)
        want = oracle.vote(co, cs.numpy(), r, nthreads=NTH)
        for exm in (None, ex):
            got = sb.vote(cod, csd, r, exemplar=exm)
            torch.cuda.synchronize()
            g = got.cpu().numpy()
            if not (g == want).all():
                bad = np.argwhere((g != want).any(-1))
                raise AssertionError(f"{wt}x{ht} exemplar={exm is not None}: {len(bad)} pixels differ, "
                                     f"first {bad[:4].tolist()}")
