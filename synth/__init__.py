"""Seeded synthetic inputs for StyleBlit.

This module holds NONE of the method's arithmetic: it only makes guide and style
rasters (uint8 x4, row-major [H, W, 4]).  Both the CUDA path (bench, tests) and the
CPU oracle (tests) are fed the same bytes produced here.

Fields are evaluated with torch so large batches (4K frames) can be generated on the
GPU outside any timed region; random parameters come from numpy's seeded RNG, so the
parameters are identical on every device.  Everything is computed in float64: torch's
float32 transcendental kernels round differently in vectorised and scalar tail paths
(which depend on memory alignment), which made a few bytes differ between processes; in
float64 a value would have to land within ~1e-16 of a rounding boundary to flip.  (The
bytes may still differ between CPU and GPU, which never matters: parity always feeds one
set of bytes to both sides.)

Generators:
  G1 sphere_normal       -- the "lit sphere" exemplar guide
  G2 painted_style       -- a painted-looking RGBA exemplar C_S
  G3 heightfield_normals -- full-frame normal map of a smooth height field (per-frame phase)
  G4 render_objects      -- normal pass of analytic spheres/tori ("rendered 3D model")
  G5 uv_identity         -- UV / texture-coordinate guide
  G6 warp_uv             -- G5 seen through a smooth displacement field
"""
from __future__ import annotations

import math

import numpy as np
import torch

__all__ = [
    "sphere_normal", "painted_style", "heightfield_normals", "render_objects",
    "uv_identity", "warp_uv", "config", "CONFIGS",
]


def _enc(n: torch.Tensor) -> torch.Tensor:
    """Normal in [-1,1] -> byte, clamp(floor((n+1)*127.5 + 0.5), 0, 255)."""
    return torch.clamp(torch.floor((n + 1.0) * 127.5 + 0.5), 0, 255).to(torch.uint8)


def _grid(W: int, H: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    y = torch.arange(H, device=device, dtype=torch.float64).view(H, 1).expand(H, W)
    x = torch.arange(W, device=device, dtype=torch.float64).view(1, W).expand(H, W)
    return x, y


def sphere_normal(W: int, H: int, device="cpu") -> torch.Tensor:
    """G1: camera-space normals of a sphere filling 96% of the shorter side; A = 0;
    (0,0,0,0) outside the disk (far in guide space from every front-facing normal)."""
    x, y = _grid(W, H, device)
    cx, cy, R = (W - 1) / 2.0, (H - 1) / 2.0, 0.48 * min(W, H)
    nx, ny = (x - cx) / R, (cy - y) / R
    r2 = nx * nx + ny * ny
    inside = r2 <= 1.0
    nz = torch.sqrt(torch.clamp(1.0 - r2, min=0.0))
    out = torch.zeros(H, W, 4, dtype=torch.uint8, device=device)
    out[..., 0] = torch.where(inside, _enc(nx), 0)
    out[..., 1] = torch.where(inside, _enc(ny), 0)
    out[..., 2] = torch.where(inside, _enc(nz), 0)
    return out


def _value_noise(W: int, H: int, rng: np.random.RandomState, cells: int, device) -> torch.Tensor:
    g = torch.from_numpy(rng.rand(cells + 1, cells + 1)).to(device)
    x, y = _grid(W, H, device)
    fx, fy = x / max(W - 1, 1) * cells, y / max(H - 1, 1) * cells
    ix, iy = torch.clamp(fx.floor().long(), 0, cells - 1), torch.clamp(fy.floor().long(), 0, cells - 1)
    tx, ty = fx - ix, fy - iy
    tx, ty = tx * tx * (3 - 2 * tx), ty * ty * (3 - 2 * ty)
    a, b = g[iy, ix], g[iy, ix + 1]
    c, d = g[iy + 1, ix], g[iy + 1, ix + 1]
    return (a * (1 - tx) + b * tx) * (1 - ty) + (c * (1 - tx) + d * tx) * ty


def painted_style(W: int, H: int, seed: int = 11, device="cpu") -> torch.Tensor:
    """G2: a painted-looking exemplar C_S: multi-octave value noise (pigment), oriented
    strokes, shaded by the sphere's n_z (a lit sphere); RGBA8 with A = 255."""
    rng = np.random.RandomState(seed)
    x, y = _grid(W, H, device)
    noise = sum(_value_noise(W, H, rng, c, device) * w for c, w in ((4, 0.5), (16, 0.3), (64, 0.2)))
    strokes = torch.zeros(H, W, device=device, dtype=torch.float64)
    for _ in range(24):
        ang = rng.uniform(0, math.pi)
        freq = rng.uniform(0.05, 0.25)
        ph = rng.uniform(0, 2 * math.pi)
        amp = rng.uniform(0.02, 0.08)
        strokes = strokes + amp * torch.sin(freq * (x * math.cos(ang) + y * math.sin(ang)) + ph)
    cx, cy, R = (W - 1) / 2.0, (H - 1) / 2.0, 0.48 * min(W, H)
    r2 = ((x - cx) / R) ** 2 + ((y - cy) / R) ** 2
    nz = torch.sqrt(torch.clamp(1.0 - r2, min=0.0))
    base = np.array([rng.uniform(0.1, 0.3), rng.uniform(0.2, 0.4), rng.uniform(0.5, 0.8)], np.float64)
    hi = np.array([rng.uniform(0.8, 1.0), rng.uniform(0.7, 0.9), rng.uniform(0.3, 0.6)], np.float64)
    shade = torch.clamp(0.15 + 0.85 * nz + 0.35 * (noise - 0.5) + strokes, 0, 1)
    out = torch.empty(H, W, 4, dtype=torch.uint8, device=device)
    for c in range(3):
        v = base[c] * (1 - shade) + hi[c] * shade + 0.15 * (noise - 0.5)
        out[..., c] = torch.clamp(v * 255.0 + 0.5, 0, 255).to(torch.uint8)
    out[..., 3] = 255
    return out


def _normals_from_height(zx: torch.Tensor, zy: torch.Tensor) -> torch.Tensor:
    """n = normalize(-dz/dx, -dz/dy, 1), y axis pointing up as in G1."""
    nx, ny, nz = -zx, zy, torch.ones_like(zx)
    inv = torch.rsqrt(nx * nx + ny * ny + nz * nz)
    out = torch.zeros(*zx.shape, 4, dtype=torch.uint8, device=zx.device)
    out[..., 0] = _enc(nx * inv)
    out[..., 1] = _enc(ny * inv)
    out[..., 2] = _enc(nz * inv)
    return out


def heightfield_normals(W: int, H: int, seed: int = 3, frame: int = 0, device="cpu") -> torch.Tensor:
    """G3: normals of z = sum_k a_k exp(-|p-c_k|^2 / 2 s_k^2) + sum_m b_m sin(w_m . p + phi_m
    + frame * d_m).  Every pixel is a valid front-facing normal.  Slopes are scaled to
    the image size so the normal gamut is similar at every resolution."""
    rng = np.random.RandomState(seed)
    x, y = _grid(W, H, device)
    S = float(min(W, H))
    zx = torch.zeros(H, W, device=device, dtype=torch.float64)
    zy = torch.zeros(H, W, device=device, dtype=torch.float64)
    for _ in range(12):
        cx, cy = rng.uniform(0, W), rng.uniform(0, H)
        s = rng.uniform(0.05, 0.2) * S
        a = rng.uniform(-1.0, 1.0) * s * 1.2
        g = a * torch.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2 * s * s))
        zx = zx + g * (-(x - cx) / (s * s))
        zy = zy + g * (-(y - cy) / (s * s))
    for _ in range(6):
        ang = rng.uniform(0, 2 * math.pi)
        k = rng.uniform(2.0, 12.0) * 2 * math.pi / S
        wx, wy = k * math.cos(ang), k * math.sin(ang)
        ph, dph = rng.uniform(0, 2 * math.pi), rng.uniform(0.05, 0.3)
        b = rng.uniform(0.05, 0.25) / k
        arg = wx * x + wy * y + ph + frame * dph
        c = b * torch.cos(arg)
        zx = zx + c * wx
        zy = zy + c * wy
    return _normals_from_height(zx, zy)


def heightfield_batch(N: int, W: int, H: int, seed: int = 5, device="cpu") -> torch.Tensor:
    """N frames of G3 with a per-frame phase shift (config 5), shape [N, H, W, 4]."""
    out = torch.empty(N, H, W, 4, dtype=torch.uint8, device=device)
    for i in range(N):
        out[i] = heightfield_normals(W, H, seed=seed, frame=i, device=device)
    return out


def render_objects(W: int, H: int, seed: int = 2, device="cpu") -> torch.Tensor:
    """G4: normal pass of analytic spheres and tori (orthographic camera along -z) over a
    camera-facing background (128,128,255,0)."""
    rng = np.random.RandomState(seed)
    x, y = _grid(W, H, device)
    S = float(min(W, H))
    depth = torch.full((H, W), -1e9, device=device, dtype=torch.float64)
    nx = torch.zeros(H, W, device=device, dtype=torch.float64)
    ny = torch.zeros(H, W, device=device, dtype=torch.float64)
    nz = torch.ones(H, W, device=device, dtype=torch.float64)
    for _ in range(5):  # spheres
        cx, cy, R, cz = rng.uniform(0.15, 0.85) * W, rng.uniform(0.15, 0.85) * H, rng.uniform(0.08, 0.25) * S, rng.uniform(0, 1)
        dx, dy = (x - cx) / R, (cy - y) / R
        r2 = dx * dx + dy * dy
        hit = r2 < 1.0
        z = torch.sqrt(torch.clamp(1 - r2, min=0))
        zz = cz + z * R / S
        m = hit & (zz > depth)
        depth = torch.where(m, zz, depth)
        nx, ny, nz = torch.where(m, dx, nx), torch.where(m, dy, ny), torch.where(m, z, nz)
    for _ in range(3):  # tori in the image plane, tube seen from the front
        cx, cy = rng.uniform(0.2, 0.8) * W, rng.uniform(0.2, 0.8) * H
        Rm, rt, cz = rng.uniform(0.12, 0.25) * S, rng.uniform(0.03, 0.07) * S, rng.uniform(0, 1)
        px_, py_ = x - cx, cy - y
        rho = torch.sqrt(px_ * px_ + py_ * py_) + 1e-6
        dr = (rho - Rm) / rt
        hit = dr.abs() < 1.0
        z = torch.sqrt(torch.clamp(1 - dr * dr, min=0))
        zz = cz + z * rt / S + 0.5
        m = hit & (zz > depth)
        depth = torch.where(m, zz, depth)
        tnx, tny = dr * px_ / rho, dr * py_ / rho
        nx, ny, nz = torch.where(m, tnx, nx), torch.where(m, tny, ny), torch.where(m, z, nz)
    inv = torch.rsqrt(nx * nx + ny * ny + nz * nz)
    out = torch.zeros(H, W, 4, dtype=torch.uint8, device=device)
    out[..., 0] = _enc(nx * inv)
    out[..., 1] = _enc(ny * inv)
    out[..., 2] = _enc(nz * inv)
    return out


def _region_label(u: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
    """A segmentation guide: 5 'semantic regions' of the UV square (a
    central disc and four quadrants), labels 0, 64, 128, 192, 255 -- spaced far apart."""
    lab = (64 * ((u >= 0.5).to(torch.int32) + 2 * (v >= 0.5).to(torch.int32))).to(torch.int32)
    disc = (u - 0.5) ** 2 + (v - 0.45) ** 2 < 0.04
    return torch.where(disc, torch.full_like(lab, 255), lab).to(torch.uint8)


def uv_identity(W: int, H: int, device="cpu", labels: bool = False) -> torch.Tensor:
    """G5: (round(255x/(W-1)), round(255y/(H-1)), 0, label); injective when W, H <= 256.
    With labels=True channel 3 holds the region label of the UV position."""
    x, y = _grid(W, H, device)
    out = torch.zeros(H, W, 4, dtype=torch.uint8, device=device)
    u, v = x / max(W - 1, 1), y / max(H - 1, 1)
    out[..., 0] = torch.floor(255.0 * u + 0.5).to(torch.uint8)
    out[..., 1] = torch.floor(255.0 * v + 0.5).to(torch.uint8)
    if labels:
        out[..., 3] = _region_label(u, v)
    return out


def warp_uv(W: int, H: int, seed: int = 4, n_rbf: int = 8, amp: float = 40.0,
            sigma: float = 170.0, device="cpu", labels: bool = False) -> torch.Tensor:
    """G6: G5 evaluated at clamp(p + sum_k A_k exp(-|p-c_k|^2 / 2 sigma^2)) (a smooth
    displacement field, the synthetic stand-in for FaceStyle's landmark warp)."""
    rng = np.random.RandomState(seed)
    x, y = _grid(W, H, device)
    scale = min(W, H) / 1024.0
    dx = torch.zeros(H, W, device=device, dtype=torch.float64)
    dy = torch.zeros(H, W, device=device, dtype=torch.float64)
    s = sigma * scale
    for _ in range(n_rbf):
        cx, cy = rng.uniform(0, W), rng.uniform(0, H)
        ax, ay = rng.uniform(-amp, amp) * scale, rng.uniform(-amp, amp) * scale
        g = torch.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2 * s * s))
        dx, dy = dx + ax * g, dy + ay * g
    wx = torch.clamp(x + dx, 0, W - 1)
    wy = torch.clamp(y + dy, 0, H - 1)
    out = torch.zeros(H, W, 4, dtype=torch.uint8, device=device)
    u, v = wx / max(W - 1, 1), wy / max(H - 1, 1)
    out[..., 0] = torch.floor(255.0 * u + 0.5).to(torch.uint8)
    out[..., 1] = torch.floor(255.0 * v + 0.5).to(torch.uint8)
    if labels:
        out[..., 3] = _region_label(u, v)
    return out


# ---------------------------------------------------------------------------------------
# BASELINE.json configs.  t was calibrated once with the oracle so that
# 40-80 % of pixels accept at level L and < 5 % fall back to level 0, then frozen
# (DESIGN.md "Input recipe").
# ---------------------------------------------------------------------------------------
CONFIGS = {
    1: dict(name="cfg1_64px_normal_L3", wt=64, ht=64, ws=64, hs=64, L=3, t=32.0, r=0, C=3, seed=0x5EED),
    2: dict(name="cfg2_1MP_objects_L5_blend", wt=1024, ht=1024, ws=512, hs=512, L=5, t=12.0, r=2, C=3, seed=0x5EED),
    3: dict(name="cfg3_4K_heightfield_L5", wt=3840, ht=2160, ws=512, hs=512, L=5, t=10.0, r=2, C=3, seed=0x5EED),
    4: dict(name="cfg4_1MP_uvwarp_L5_blend", wt=1024, ht=1024, ws=1024, hs=1024, L=5, t=1.25, r=2, C=2, seed=0x5EED),
    5: dict(name="cfg5_4K_batch_heightfield_L5", wt=3840, ht=2160, ws=512, hs=512, L=5, t=10.0, r=2, C=3, seed=0x5EED),
}


def exemplar(cfg: dict, device="cpu") -> tuple[torch.Tensor, torch.Tensor]:
    """(C_S, G_S) of a config."""
    ws, hs = cfg["ws"], cfg["hs"]
    if cfg.get("guide", "normal") == "uv" or cfg["C"] == 2:
        return painted_style(ws, hs, seed=11, device=device), uv_identity(ws, hs, device=device)
    return painted_style(ws, hs, seed=11, device=device), sphere_normal(ws, hs, device=device)


def target(cfg_id: int, frame: int = 0, device="cpu") -> torch.Tensor:
    """G_T of a config (one frame)."""
    cfg = CONFIGS[cfg_id]
    wt, ht = cfg["wt"], cfg["ht"]
    if cfg_id == 1:
        return heightfield_normals(wt, ht, seed=1, frame=frame, device=device)
    if cfg_id == 2:
        return render_objects(wt, ht, seed=2, device=device)
    if cfg_id == 3:
        return heightfield_normals(wt, ht, seed=3, frame=frame, device=device)
    if cfg_id == 4:
        return warp_uv(wt, ht, seed=4, device=device)
    if cfg_id == 5:
        return heightfield_normals(wt, ht, seed=5, frame=frame, device=device)
    raise KeyError(cfg_id)


def config(cfg_id: int, device="cpu"):
    """(cfg, C_S, G_S, G_T) for config 1..5 (frame 0)."""
    cfg = CONFIGS[cfg_id]
    cs, gs = exemplar(cfg, device)
    return cfg, cs, gs, target(cfg_id, 0, device)
