#!/usr/bin/env python
"""StyleBlit (arXiv 1807.03249) hot-path benchmark on B200.

One STEP = one pass of the hot path over one batch of synthetic 4K frames per GPU:
  sb_build_lut (the exemplar's guide LUT)
  + sb_stylize_batch (Alg. 2 for every pixel of every frame, per-frame jitter seeds,
    PAPER.md:337-433; coordinates and blit colours C_T[p] = C_S[s] out).
The seam blend is optional in the paper ("When seams become obvious, we can optionally perform
blending"); it is timed in its own run every time (`blend_r2`): LUT + stylize
(coordinates) + sb_vote (r = 2).  `--blend-radius 2` makes it the headline.
Workload (BASELINE.json configs[4] = config 5, per GPU): B frames of 3840x2160 heightfield
normals (seed 5, per-frame phase), 512x512 sphere exemplar, L=5, t=10, C=3.
Frames are sharded by rank (weak scaling: every GPU stylizes its own B frames, no data-path
collective).  Inputs are > L2 (B*33 MB of G_T per step), so no L2 flush is needed.

`value` = whole-job stylized megapixels/s (device-resident inputs, CUDA-event timing, max over
ranks).  `e2e` = the same through sb_stylize_batch_host with pinned host buffers (host->device
copies of G_T and device->host copies of C_T inside the timed region).

`--impl reference` runs the CPU oracle (oracle/, the reference arm of this tier) on the same
config: each step = one 4K frame (stylize + vote) on all host cores, LUT built before timing.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WT, HT = 3840, 2160
CFG_ID = 5


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=64, help="4K frames per GPU per step")
    ap.add_argument("--blend-radius", type=int, default=0,
                    help="0 (default): the stylization proper, blit colours (PAPER.md:387); the optional "
                         "vote blend (PAPER.md:412) is timed separately at r=2 and reported as blend_r2")
    ap.add_argument("--blend-steps", type=int, default=20, help="timed steps of the r=2 blend run (0: skip)")
    ap.add_argument("--mode", default="frame", choices=["frame", "strip"],
                    help="frame: each GPU stylizes its own frames (weak scaling, no collective); "
                         "strip: every frame is split into row strips across GPUs and the C_T strips "
                         "are gathered to rank 0 with NCCL each step")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "p2p"],
                    help="strip mode: nccl = one NCCL gather of the C_T strips after the compute; p2p = rank 0's "
                         "C_T buffer is mapped into every rank (CUDA IPC) and the kernels store their rows into it "
                         "over NVLink/NVSwitch, then a one-element all-reduce orders rank 0 after the writers")
    ap.add_argument("--lut-rgb-steps", type=int, default=10,
                    help="timed steps of the exact 3-channel guide-search run (SB_LUT_RGB, 0: skip)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config sections (BASELINE configs 1, 2, 4, single-frame 4K latency, "
                         "ragged width) and their oracle timings")
    ap.add_argument("--config-steps", type=int, default=10, help="timed steps of each per-config section")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-digest", action="store_true", help="skip the output_sha1 digests of global frames 0, B-1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--json-out", default=None)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons DURING the timed region."""

    def __init__(self, index: int, period_s: float = 0.02):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------- per-config sections
def _levels(torch, sb, prm_kw, cs, gs, lut, gt1, L):
    """Level histogram of one frame (which level accepted each pixel) and the mean
    number of levels a pixel visits; untimed."""
    lv = torch.empty(gt1.shape[0], gt1.shape[1], dtype=torch.uint8, device=gt1.device)
    sb.stylize(sb.Params(**prm_kw), cs, gs, lut, gt1, level=lv)
    hist = torch.bincount(lv.flatten().long(), minlength=L + 1).double()
    frac = (hist / hist.sum()).tolist()
    visited = sum(f * (L - l + 1 if l >= 1 else L) for l, f in enumerate(frac))
    return {"accepted_at_level": {str(l): round(frac[l], 4) for l in range(L, -1, -1)},
            "mean_levels_visited": round(visited, 3)}


def gpu_section(torch, sb, synth, dev, stream, hbm, cid, frames, rad, steps, warmup, wt=None, ht=None):
    """One BASELINE config on the GPU: a batch of `frames` frames per step, the step being
    sb_build_lut + sb_prepare_exemplar + sb_stylize_batch (+ sb_vote for rad > 0) as in the
    headline; CUDA events on the launching stream around every call; value = frames x pixels /
    step time.  wt/ht override the config's target size (the ragged-width row)."""
    cfg = synth.CONFIGS[cid]
    wt, ht = wt or cfg["wt"], ht or cfg["ht"]
    cs, gs = [t.to(dev) for t in synth.exemplar(cfg, device=dev)]
    if (wt, ht) == (cfg["wt"], cfg["ht"]):
        firsts = [synth.target(cid, i, device=dev) for i in range(min(frames, 4 if cid in (1, 3, 5) else 1))]
    else:
        firsts = [synth.heightfield_normals(wt, ht, seed=5, frame=i, device=dev) for i in range(min(frames, 4))]
    gt = torch.empty(frames, ht, wt, 4, dtype=torch.uint8, device=dev)
    for i in range(frames):
        gt[i] = firsts[i % len(firsts)]
    # a host uint32 array built once: the binding passes it to the ABI without per-step conversion
    seeds = ((cfg["seed"] + np.arange(frames, dtype=np.int64)) & 0xFFFFFFFF).astype(np.uint32)
    lut = torch.empty(65536, dtype=torch.int32, device=dev)
    lut_ws = torch.empty(sb.lib().sb_lut_workspace_bytes(), dtype=torch.uint8, device=dev)
    ex = torch.empty(sb.exemplar_bytes(cfg["ws"], cfg["hs"]), dtype=torch.uint8, device=dev)
    coords = torch.empty(frames, ht, wt, dtype=torch.int32, device=dev)
    ct = torch.empty(frames, ht, wt, 4, dtype=torch.uint8, device=dev)
    prm = sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], seed=cfg["seed"],
                    flags=sb.SB_NO_COLOR if rad > 0 else 0, exemplar=ex)
    names = ("lut", "exemplar", "stylize", "vote")
    ev = {k: [] for k in names}
    nl = [0]

    def step(rec):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if rec else None
        if rec:
            e[0].record(stream)
        sb.build_lut(gs, lut, lut_ws)
        n = sb.launch_count()
        if rec:
            e[1].record(stream)
        sb.prepare_exemplar(cs, gs, ex)
        n += sb.launch_count()
        if rec:
            e[2].record(stream)
        sb.stylize_batch(prm, cs, gs, lut, gt, frame_seeds=seeds, ct=None if rad > 0 else ct, coords=coords,
                         want_level=False)
        n += sb.launch_count()
        if rec:
            e[3].record(stream)
        if rad > 0:
            sb.vote(coords, cs, rad, ct=ct, exemplar=ex)
            n += sb.launch_count()
        if rec:
            e[4].record(stream)
            for k, (a, b) in zip(names, ((0, 1), (1, 2), (2, 3), (3, 4))):
                ev[k].append((e[a], e[b]))
            nl[0] += n

    for _ in range(warmup):
        step(False)
    torch.cuda.synchronize(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step(True)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1) / steps
    px = frames * wt * ht
    kt = {k: statistics.mean(a.elapsed_time(b) for a, b in v) for k, v in ev.items()}
    alg = {"stylize": (8 if rad > 0 else 12) * px}
    if rad > 0:
        alg["vote"] = 8 * px
    kernels = {k: {"ms_per_launch": round(kt[k], 4), "share": round(kt[k] / ms, 4)} for k in names if k != "vote" or rad}
    dom = max(alg, key=lambda k: kt[k])
    ach = alg[dom] / (kt[dom] * 1e-3) / 1e9
    prm_l = dict(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], seed=cfg["seed"])
    out = {"value": round(px / (ms * 1e-3) / 1e6, 1), "unit": "MP/s", "ms_per_step": round(ms, 4),
           "frames_per_step": frames, "frame": f"{wt}x{ht}", "exemplar": f"{cfg['ws']}x{cfg['hs']}",
           "L": cfg["L"], "t": cfg["t"], "C": cfg["C"], "blend_radius": rad,
           "kernels": kernels, "gpu_launches": nl[0],
           "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(ach / hbm, 4), "alg_bytes_per_px": alg[dom] // px},
           "levels": _levels(torch, sb, prm_l, cs, gs, lut, gt[0], cfg["L"])}
    del gt, coords, ct, ex
    return out


def single_frame_latency(torch, sb, synth, dev, reps=200):
    """One 4K frame (config 3) at a time, the paper's per-frame regime: the
    per-frame calls captured once in a CUDA graph and replayed back to back (no launch
    overhead); LUT and exemplar copy built once before (per exemplar, not per frame)."""
    cfg = synth.CONFIGS[3]
    cs, gs = [t.to(dev) for t in synth.exemplar(cfg, device=dev)]
    gt = synth.target(3, 0, device=dev)
    lut = sb.build_lut(gs)
    ex = sb.prepare_exemplar(cs, gs)
    coords = torch.empty(gt.shape[0], gt.shape[1], dtype=torch.int32, device=dev)
    ct = torch.empty_like(gt)
    out = {}
    for rad in (0, 2):
        prm = sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], seed=cfg["seed"],
                        blend_radius=rad, exemplar=ex)
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            for _ in range(3):
                sb.stylize(prm, cs, gs, lut, gt, ct=ct, coords=coords, want_level=False)
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            sb.stylize(prm, cs, gs, lut, gt, ct=ct, coords=coords, want_level=False)
        for _ in range(10):
            g.replay()
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b) / reps
        out[f"r{rad}"] = {"ms_per_frame": round(ms, 4), "fps": round(1000.0 / ms, 1),
                          "MPps": round(gt.shape[0] * gt.shape[1] / (ms * 1e-3) / 1e6, 1)}
        del g
    out["note"] = ("one 3840x2160 frame per CUDA-graph replay, replays back to back; r0 = stylize + blit, "
                   "r2 = stylize + vote; LUT and exemplar copy built once per exemplar")
    return out


def oracle_section(cid, rad, frames_1t, frames_nt, nth):
    """The CPU oracle (as it stands) on the same config: LUT built first (timed apart, excluded),
    then stylize (+ vote) per frame at 1 thread and at nth threads."""
    import oracle
    import synth

    cfg = synth.CONFIGS[cid]
    cs, gs = [t.numpy() for t in synth.exemplar(cfg)]
    gts = [synth.target(cid, i).numpy() for i in range(max(frames_1t, frames_nt) if cid in (1, 3, 5) else 1)]
    t0 = time.perf_counter()
    lut = oracle.build_lut(gs, nthreads=nth)
    t_lut = time.perf_counter() - t0

    def run(n, th):
        t = time.perf_counter()
        for i in range(n):
            prm = oracle.Params(t=cfg["t"], L=cfg["L"], C=cfg["C"], seed=(cfg["seed"] + i) & 0xFFFFFFFF)
            _, co, _ = oracle.stylize(prm, cs, gs, lut, gts[i % len(gts)], nthreads=th)
            if rad > 0:
                oracle.vote(co, cs, rad, nthreads=th)
        return time.perf_counter() - t

    px = cfg["wt"] * cfg["ht"]
    d1, dn = run(frames_1t, 1), run(frames_nt, nth)
    return {"value_1thread": round(frames_1t * px / d1 / 1e6, 3), "value_nthreads": round(frames_nt * px / dn / 1e6, 3),
            "unit": "MP/s", "threads": nth, "kind": "oracle", "lut_build_s": round(t_lut, 2),
            "sample": f"{frames_1t} frame(s) at 1 thread ({d1:.2f} s), {frames_nt} frame(s) at {nth} threads "
                      f"({dn:.2f} s); stylize{' + vote r=%d' % rad if rad else ' (blit)'}; LUT build "
                      f"({nth} threads) excluded"}


def animation_section(torch, sb, synth, dev):
    """SURVEY 8(f) #2 as a measured property ("the amount of flickering can be
    controlled by changing the guidance threshold"): config 2 (1 MP rendered objects, static
    guide) over 16 frames with per-frame seeds, per threshold t: flicker = mean |C_T^(i+1) -
    C_T^(i)| over pixels, channels and consecutive frames (8-bit units), for the blit (r = 0)
    and the vote (r = 2); chunk edges = the fraction of 4-neighbour pixel pairs whose offsets
    src - p differ (smaller = larger chunks); the share of pixels at level L.  Untimed."""
    cfg = synth.CONFIGS[2]
    cs, gs = [t.to(dev) for t in synth.exemplar(cfg, device=dev)]
    lut = sb.build_lut(gs)
    gt1 = synth.target(2, device=dev)
    n = 16
    frames = gt1.unsqueeze(0).expand(n, *gt1.shape).contiguous()
    H, W = gt1.shape[:2]
    xs = torch.arange(W, device=dev, dtype=torch.int64).view(1, 1, W)
    ys = torch.arange(H, device=dev, dtype=torch.int64).view(1, H, 1)
    rows = []
    for t in (4.0, 8.0, 12.0, 24.0, 48.0):
        row = {"t": t}
        for r in (0, 2):
            prm = sb.Params(threshold=t, levels=cfg["L"], blend_radius=r, guide_channels=cfg["C"], seed=1)
            ct, co, lv = sb.stylize_batch(prm, cs, gs, lut, frames)  # seeds 1 .. 16
            d = (ct[1:].to(torch.int16) - ct[:-1].to(torch.int16)).abs().float().mean().item()
            row[f"flicker_r{r}"] = round(d, 3)
            if r == 0:
                c = co.to(torch.int64) & 0xFFFFFFFF
                off = ((c & 0xFFFF) - xs) * 65536 + ((c >> 16) - ys)
                e = ((off[:, :, 1:] != off[:, :, :-1]).sum() + (off[:, 1:] != off[:, :-1]).sum()).item()
                row["chunk_edge_fraction"] = round(e / (n * (H * (W - 1) + (H - 1) * W)), 4)
                row["share_level_L"] = round((lv == cfg["L"]).float().mean().item(), 4)
        rows.append(row)
    prm = sb.Params(threshold=12.0, levels=cfg["L"], guide_channels=cfg["C"], seed=1)
    same = sb.stylize_batch(prm, cs, gs, lut, frames, frame_seeds=[5] * n)[0]
    still = (same[1:].to(torch.int16) - same[:-1].to(torch.int16)).abs().float().mean().item()
    return {"workload": "cfg2 1 MP static guide, 16 frames, seeds 1..16, L=5, C=3", "rows": rows,
            "flicker_fixed_seed_t12": round(still, 3),
            "note": "flicker grows with t and chunks grow (fewer edges); a fixed seed gives identical frames"}


def config_sections(args, torch, sb, synth, dev, stream, hbm, with_oracle):
    """BASELINE.json configs other than the headline, each with its own value, roofline, level
    histogram and the oracle timed beside it; plus the single-frame 4K latency and a ragged
    width row.  Not part of the headline value."""
    nth = os.cpu_count() or 1
    st, wu = args.config_steps, 3
    secs = {}
    plan = [("cfg1_64px_normal_L3", 1, 4096, 0, (64, 4)),
            ("cfg2_1MP_objects_L5_blend_r2", 2, 64, 2, (1, 1)),
            ("cfg4_1MP_uvwarp_displacement_L5_blend_r2", 4, 64, 2, (1, 1))]
    for name, cid, frames, rad, (f1, fn) in plan:
        sec = gpu_section(torch, sb, synth, dev, stream, hbm, cid, frames, rad, st, wu)
        if with_oracle:
            sec["oracle"] = oracle_section(cid, rad, f1, fn, nth)
        secs[name] = sec
    secs["single_frame_4k"] = single_frame_latency(torch, sb, synth, dev)
    rag = gpu_section(torch, sb, synth, dev, stream, hbm, 5, args.frames, 0, st, wu, wt=3838, ht=2160)
    rag["note"] = "cfg5 workload at a width not divisible by 4 (3838): the tiled kernel's per-pixel row I/O"
    secs["ragged_3838x2160"] = rag
    secs["animation_flicker_vs_t"] = animation_section(torch, sb, synth, dev)
    return secs


# ----------------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1807_03249_b200 as sb
    import synth
    from paper_1807_03249_b200 import sharding

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS[CFG_ID]
    B, r = args.frames, args.blend_radius
    # exemplar replicated on every GPU; frames of this rank: global indices rank*B .. rank*B+B-1
    cs, gs = [t.to(dev) for t in synth.exemplar(cfg, device=dev)]
    base = synth.heightfield_normals(WT, HT, seed=5, frame=0, device=dev)
    gt = torch.empty(B, HT, WT, 4, dtype=torch.uint8, device=dev)
    n_distinct = min(B, 8)  # G_T content barely matters for speed; 8 distinct phases, cycled
    for i in range(n_distinct):
        gt[i] = synth.heightfield_normals(WT, HT, seed=5, frame=rank * B + i, device=dev)
    for i in range(n_distinct, B):
        gt[i] = gt[i % n_distinct]
    del base
    strip = args.mode == "strip"
    if strip:  # all ranks work on the same frames, each on its own row strip
        for i in range(n_distinct):
            gt[i] = synth.heightfield_normals(WT, HT, seed=5, frame=i, device=dev)
        for i in range(n_distinct, B):
            gt[i] = gt[i % n_distinct]
    rb, re_ = sharding.strip_rows(HT, world, rank) if strip else (0, HT)
    frame0 = 0 if strip else rank * B
    seeds = ((cfg["seed"] + frame0 + np.arange(B, dtype=np.int64)) & 0xFFFFFFFF).astype(np.uint32)
    coords = torch.empty(B, HT, WT, dtype=torch.int32, device=dev)
    ct = torch.empty(B, HT, WT, 4, dtype=torch.uint8, device=dev)
    lut = torch.empty(65536, dtype=torch.int32, device=dev)
    lut_ws = torch.empty(sb.lib().sb_lut_workspace_bytes(), dtype=torch.uint8, device=dev)
    ex = torch.empty(sb.exemplar_bytes(cs.shape[1], cs.shape[0]), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    p2p = strip and world > 1 and args.gather == "p2p"
    # the C_T buffer the kernels write: local, or (p2p) rank 0's buffer mapped into this rank
    ct_out = sharding.peer_output(ct if rank == 0 else None, tuple(ct.shape), torch.uint8, rank) if p2p else ct
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    px_step = B * WT * HT if not strip else B * WT * (re_ - rb)  # pixels this rank outputs
    px_job = world * B * WT * HT if not strip else B * WT * HT

    def time_path(rad: int, steps: int, warmup: int):
        """Time `steps` steps of the path with blend radius rad (0: blit colours straight from
        the stylize kernel; > 0: stylize -> coords, then the vote kernel)."""
        r_halo = rad if strip else 0
        flags = sb.SB_NO_COLOR if rad > 0 else 0
        prm = sb.Params(threshold=cfg["t"], levels=cfg["L"], blend_radius=0, guide_channels=cfg["C"],
                        seed=cfg["seed"], flags=flags, row_begin=max(0, rb - r_halo), row_end=min(HT, re_ + r_halo),
                        exemplar=ex)
        ev = {k: [] for k in ("lut", "exemplar", "stylize", "vote", "gather")}
        launches = [0]

        def step(record: bool):
            es = [torch.cuda.Event(enable_timing=True) for _ in range(6)] if record else None
            if record:
                es[0].record(stream)
            sb.build_lut(gs, lut, lut_ws)
            n = sb.launch_count()
            if record:
                es[5].record(stream)
            # the strided exemplar copy (per exemplar, like the LUT): part of every step
            sb.prepare_exemplar(cs, gs, ex)
            n += sb.launch_count()
            if record:
                es[1].record(stream)
            sb.stylize_batch(prm, cs, gs, lut, gt, frame_seeds=seeds, ct=None if rad > 0 else ct_out, coords=coords,
                             want_level=False)
            n += sb.launch_count()
            if record:
                es[2].record(stream)
            if rad > 0:
                sb.vote(coords, cs, rad, ct=ct_out, row_begin=rb, row_end=re_, exemplar=ex)
                n += sb.launch_count()
            if record:
                es[3].record(stream)
            if p2p:  # the strips are already in rank 0's buffer: order rank 0 after every writer
                dist.all_reduce(flag)
            elif strip and world > 1:  # the one exchange step: C_T strips -> rank 0 over NCCL
                sharding.gather_strips(ct[:, rb:re_], HT, world, rank, dst=0, row_axis=1,
                                       out=ct if rank == 0 else None)
            if record:
                es[4].record(stream)
                ev["lut"].append((es[0], es[5]))
                ev["exemplar"].append((es[5], es[1]))
                ev["stylize"].append((es[1], es[2]))
                ev["vote"].append((es[2], es[3]))
                ev["gather"].append((es[3], es[4]))
                launches[0] += n

        for _ in range(warmup):
            step(False)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            t0.record(stream)
            for _ in range(steps):
                step(True)
            t1.record(stream)
            torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ms = t0.elapsed_time(t1)
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        ms_step = ms / steps
        kt = {k: statistics.mean(a.elapsed_time(b) for a, b in v) for k, v in ev.items()}
        # algorithmic bytes per launch: stylize reads G_T and writes coords (+ C_T
        # when it blits); the vote reads coords and writes C_T
        alg = {"stylize": (8 if rad > 0 else 12) * px_step, "lut": gs.numel() + 65536 * 4,
               "exemplar": 4 * gs.numel()}
        if rad > 0:
            alg["vote"] = 8 * px_step
        kernels = {k: {"ms_per_launch": round(kt[k], 4), "share": round(kt[k] / ms_step, 4),
                       "GBps_alg": round(alg[k] / (kt[k] * 1e-3) / 1e9, 1)} for k in alg}
        if strip and world > 1:
            gbytes = (world - 1) * B * WT * (HT // world) * 4  # strips arriving at rank 0
            kernels["gather"] = {"ms_per_step": round(kt["gather"], 4), "share": round(kt["gather"] / ms_step, 4),
                                 "GBps_into_rank0": round(gbytes / (kt["gather"] * 1e-3) / 1e9, 1)}
        dom = max([k for k in ("stylize", "vote") if k in alg], key=lambda k: kt[k])
        return dict(ms_step=ms_step, value=px_job / (ms_step * 1e-3) / 1e6, kernels=kernels, kt=kt, alg=alg,
                    dom=dom, launches=launches[0], clocks=clk.summary())

    r = args.blend_radius
    main = time_path(r, args.steps, args.warmup)
    # determinism across GPU counts: SHA-1 of the C_T of global frames 0 and B-1,
    # which rank 0 holds at every N (frame mode: its own first frames; strip mode: the gathered
    # frames) with the same inputs and seeds -- the digests must not change with N
    digests = None
    if rank == 0 and not args.no_digest:
        import hashlib
        torch.cuda.synchronize(dev)
        digests = {f"frame_{i}": hashlib.sha1(ct[i].cpu().numpy().tobytes()).hexdigest()[:16] for i in (0, B - 1)}
    ms_step, value, dom, kt, alg = main["ms_step"], main["value"], main["dom"], main["kt"], main["alg"]
    hbm, hbm_src = peaks()
    ach = alg[dom] / (kt[dom] * 1e-3) / 1e9
    # measured DRAM traffic of the same kernel: one `ncu --set full` capture (profiles/traffic.json,
    # written by tools/ncu_traffic.py), per pixel, scaled to this launch
    traffic = None
    roof_issue = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        key = dom if not (dom == "stylize" and r > 0) else "stylize_coords"
        traffic = round(tj[key]["bytes_per_px"] * px_step)
        # the bound the kernel actually meets: instruction issue.  Peak = SMs x 4
        # schedulers x 1 warp-instruction/clock at the max SM clock; achieved = the warp
        # instructions per pixel of the ncu capture x the pixels per second measured here.
        ipp = tj[key].get("warp_inst_per_px")
        if ipp:
            props = torch.cuda.get_device_properties(dev)
            mhz = main["clocks"].get("sm_max_mhz") or 1965
            peak_i = props.multi_processor_count * 4 * mhz * 1e6
            ach_i = ipp * px_step / (kt[dom] * 1e-3)
            roof_issue = {"bound": "alu", "kernel": dom, "achieved": round(ach_i / 1e9, 1),
                          "peak": round(peak_i / 1e9, 1), "unit": "G warp-instructions/s",
                          "frac": round(ach_i / peak_i, 4), "warp_inst_per_px": round(ipp, 3),
                          "simt_efficiency": round(tj[key].get("simt_efficiency", 0.0), 4),
                          "peak_source": "SMs x 4 issue slots x max SM clock (B200_PROFILING.md unit counts)"}
    except Exception:
        pass
    kernels = main["kernels"]
    blend = None
    if r == 0 and args.blend_steps > 0:
        # the optional seam blend at the config's r = 2: its own timed run
        bl = time_path(2, args.blend_steps, max(3, min(args.warmup, 5)))
        blend = {"value": round(bl["value"], 1), "unit": "MP/s", "ms_per_step": round(bl["ms_step"], 4),
                 "blend_radius": 2, "kernels": bl["kernels"], "gpu_launches": bl["launches"], "clocks": bl["clocks"],
                 "step": "LUT build + stylize (coords) + vote r=2"}

    # ---- NEXT #3: the exact 3-channel guide search (SB_LUT_RGB, R26).  The 2^24-entry
    #      table is built once per exemplar (timed on its own); a step = stylize with it.
    lut_rgb = None
    if args.lut_rgb_steps > 0 and not strip:
        lut3 = torch.empty(1 << 24, dtype=torch.int32, device=dev)
        ws3 = torch.empty(sb.lib().sb_lut3_workspace_bytes(), dtype=torch.uint8, device=dev)
        sb.build_lut3(gs, lut3, ws3)
        torch.cuda.synchronize(dev)
        a3, b3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a3.record(stream)
        for _ in range(3):
            sb.build_lut3(gs, lut3, ws3)
        b3.record(stream)
        torch.cuda.synchronize(dev)
        build_ms = a3.elapsed_time(b3) / 3
        prm3 = sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], seed=cfg["seed"], lut_rgb=True,
                         exemplar=ex)
        for _ in range(3):
            sb.stylize_batch(prm3, cs, gs, lut3, gt, frame_seeds=seeds, ct=ct, coords=coords, want_level=False)
        torch.cuda.synchronize(dev)
        a3.record(stream)
        for _ in range(args.lut_rgb_steps):
            sb.stylize_batch(prm3, cs, gs, lut3, gt, frame_seeds=seeds, ct=ct, coords=coords, want_level=False)
        b3.record(stream)
        torch.cuda.synchronize(dev)
        ms3 = a3.elapsed_time(b3) / args.lut_rgb_steps
        lut_rgb = {"value": round(px_job / (ms3 * 1e-3) / 1e6, 1), "unit": "MP/s", "ms_per_step": round(ms3, 4),
                   "lut3_build_ms": round(build_ms, 3),
                   "step": "stylize (coords + blit colours) with the exact 3-channel table; table built once "
                           "per exemplar (lut3_build_ms, 2^24 entries)"}
        del lut3, ws3

    # ---- level histogram of the headline workload: which level accepted each
    #      pixel and the mean number of levels a pixel visits (outside any timed region)
    levels = None
    if not strip:
        nf = min(B, 4)
        prm_l = sb.Params(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], seed=cfg["seed"])
        lv = torch.empty(nf, HT, WT, dtype=torch.uint8, device=dev)
        sb.stylize_batch(prm_l, cs, gs, lut, gt[:nf], frame_seeds=seeds[:nf], ct=ct[:nf], coords=coords[:nf],
                         level=lv)
        hist = torch.bincount(lv.flatten().long(), minlength=cfg["L"] + 1).double()
        frac = (hist / hist.sum()).tolist()
        Lc = cfg["L"]
        visited = sum(f * (Lc - l + 1 if l >= 1 else Lc) for l, f in enumerate(frac))
        levels = {"accepted_at_level": {str(l): round(frac[l], 4) for l in range(Lc, -1, -1)},
                  "mean_levels_visited": round(visited, 3), "frames": nf,
                  "note": "level 0 = no level accepted, LUT look-up (reading R12)"}
        del lv

    # ---- e2e through the host-buffer ABI call (pinned host memory, copies inside timing)
    def run_e2e(rgb: bool):
        # the step's whole batch through host memory (fill/drain of the copy pipeline amortised
        # over the batch); SB_E2E_FRAMES caps it (pinned host memory: 2 x 33 MB per frame).
        # rgb: the packed-RGB host frames of SB_HOST_RGB (3 bytes per pixel each way; C = 3).
        Be = min(B, int(os.environ.get("SB_E2E_FRAMES", "64")))
        ch = 3 if rgb else 4
        gt_h = gt[:Be, ..., :ch].contiguous().cpu().pin_memory()
        ct_h = torch.empty_like(gt_h).pin_memory()
        prm_e = sb.Params(threshold=cfg["t"], levels=cfg["L"], blend_radius=r, guide_channels=cfg["C"],
                          seed=cfg["seed"], exemplar=ex, flags=sb.SB_HOST_RGB if rgb else 0)
        depth = int(os.environ.get("SB_E2E_DEPTH", "2"))
        ws_e = sb.host_workspace(WT, HT, r, depth, device=dev)

        def e2e_step():
            sb.build_lut(gs, lut, lut_ws)
            sb.prepare_exemplar(cs, gs, ex)
            sb.stylize_batch_host(prm_e, cs, gs, lut, gt_h, ct_h, frame_seeds=seeds[:Be], workspace=ws_e, depth=depth)

        e2e_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize(dev)
        ems = a.elapsed_time(b) / args.e2e_steps
        if world > 1:
            tt = torch.tensor([ems], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        res = {"value": round(world * Be * WT * HT / (ems * 1e-3) / 1e6, 1), "unit": "MP/s",
               "h2d_bytes_per_step": Be * WT * HT * ch, "d2h_bytes_per_step": Be * WT * HT * ch,
               "frames_per_step": Be, "ms_per_step": round(ems, 3),
               "api": (f"sb_stylize_batch_host (pinned host G_T in, pinned host C_T out, {depth}-deep copy/compute "
                       "pipeline" + ("; SB_HOST_RGB: packed RGB frames, C_T channels 0..2)" if rgb else ")"))}
        del gt_h, ct_h, ws_e
        return res

    e2e = e2e_rgb = None
    if not args.no_e2e and args.e2e_steps > 0 and not strip:
        e2e = run_e2e(False)
        if cfg["C"] <= 3:
            e2e_rgb = run_e2e(True)

    configs = None
    if not args.no_configs and not strip:
        del gt, coords, ct  # the sections allocate their own batches
        configs = config_sections(args, torch, sb, synth, dev, stream, hbm,
                                  with_oracle=(rank == 0 and world == 1 and not args.no_cpu_baseline))
        if "ragged_3838x2160" in configs:
            configs["ragged_3838x2160"]["vs_3840"] = round(configs["ragged_3838x2160"]["value"] / value, 4)

    # ---- parity spot check of this run's outputs (sampled pixels of frame 0 vs oracle) is in tests/.
    out = {
        "metric": "stylized megapixels/s (4K UHD frames/s) per B200 and 8-GPU; % HBM roofline",
        "value": round(value, 1),
        "unit": "MP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak" if not strip else "strong",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (seeded heightfield-normal 4K frames, sphere-normal exemplar, painted style)",
        "config": {"workload": f"cfg5: {B} x 4K UHD (3840x2160) frames per GPU, 512x512 exemplar, L={cfg['L']}, "
                               f"t={cfg['t']}, C={cfg['C']}, blend r={r}; step = LUT build + strided exemplar copy + stylize"
                               + (" + vote" if r > 0 else " (blit colours)"),
                   "frames_per_gpu": B, "global_frames": B * world, "levels": cfg["L"], "threshold": cfg["t"],
                   "blend_radius": r,
                   "parallelism": (f"frame-sharded x{world} (no data-path collective)" if not strip else
                                   f"row-strip-sharded x{world}, C_T strips gathered to rank 0 "
                                   + ("(kernels store into rank 0's buffer over NVLink peer memory)" if p2p
                                      else "(NCCL gather)")),
                   "l2": "inputs larger than L2 (G_T %.2f GB per GPU per step); no flush" % (4 * px_step / 1e9)},
        "fps_4k": round(value * 1e6 / (WT * HT), 1),
        "kernels": kernels,
        "roofline_issue": roof_issue,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(ach / hbm, 4), "frac_nominal_8tbs": round(ach / 8000.0, 4),
                     "traffic": traffic, "peak_source": hbm_src,
                     "alg_bytes_per_launch": alg[dom], "alg_bytes_per_px": alg[dom] // px_step},
        "gpu_launches": main["launches"],
        "clocks": main["clocks"],
        "output_sha1": digests,
        "e2e": e2e,
        "e2e_rgb": e2e_rgb,
        "blend_r2": blend,
        "lut_rgb": lut_rgb,
        "levels": levels,
        "configs": configs,
    }
    return out, rank, world


# ----------------------------------------------------------------------------------- oracle
def cpu_baseline(args):
    """The oracle on the headline workload: LUT built first (excluded, reported apart), then
    stylize (+ vote) on 4 frames at all host threads and on 1 frame at 1 thread."""
    nth = os.cpu_count() or 1
    sec = oracle_section(CFG_ID, args.blend_radius, 1, 4, nth)
    return {"value": sec["value_nthreads"], "unit": "MP/s", "cores": nth, "kind": "oracle",
            "value_1thread": sec["value_1thread"], "lut_build_s": sec["lut_build_s"],
            "sample": "cfg5 4K frames: " + sec["sample"]}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return None, rank, world
    import oracle
    import synth

    cfg = synth.CONFIGS[CFG_ID]
    nth = os.cpu_count() or 1
    cs, gs = [t.numpy() for t in synth.exemplar(cfg)]
    lut = oracle.build_lut(gs, nthreads=nth)
    frames = [synth.heightfield_normals(WT, HT, seed=5, frame=i).numpy() for i in range(2)]
    r = args.blend_radius

    def step(i):
        prm = oracle.Params(t=cfg["t"], L=cfg["L"], C=cfg["C"], seed=(cfg["seed"] + i) & 0xFFFFFFFF)
        _, coords, _ = oracle.stylize(prm, cs, gs, lut, frames[i % 2], nthreads=nth)
        if r > 0:
            oracle.vote(coords, cs, r, nthreads=nth)

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i)
    dt = (time.perf_counter() - t0) / args.steps
    v = round(WT * HT / dt / 1e6, 3)
    out = {
        "impl": "reference",
        "metric": "stylized megapixels/s (4K UHD frames/s) per B200 and 8-GPU; % HBM roofline",
        "value": v, "unit": "MP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 2), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"cfg5: 4K UHD frames, 512x512 exemplar, L={cfg['L']}, t={cfg['t']}, C={cfg['C']}, "
                               f"blend r={r}; reference step = 1 frame on the CPU oracle (LUT built before timing)"},
        "cpu_baseline": {"value": v, "unit": "MP/s", "cores": nth, "kind": "oracle",
                         "sample": f"1 4K frame per step (stylize{" + vote r=" + str(r) if r else ", blit colours"}), {nth} host threads"},
        "e2e": {"value": v, "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return out, rank, world


def main():
    args = parse()
    if args.impl == "reference":
        out, rank, world = run_reference(args)
    else:
        out, rank, world = run_ours(args)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args)
    if rank == 0 and out is not None:
        line = json.dumps(out)
        print(line, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(line + "\n")
    if args.impl == "ours" and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
