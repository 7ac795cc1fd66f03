"""StyleBlit (arXiv 1807.03249) hot path on B200: a thin Python binding of include/styleblit.h.

The names match the C ABI (``sb_build_lut`` -> :func:`build_lut`, ``sb_stylize`` ->
:func:`stylize`, ``sb_stylize_batch`` -> :func:`stylize_batch`,
``sb_stylize_batch_host`` -> :func:`stylize_batch_host`).  This module only marshals
arguments: every step of the method runs in the sm_100a kernels of ``libstyleblit.so``.
PyTorch provides device memory and the current CUDA stream.  There is no CPU fallback: the
functions raise if the library is missing or a tensor is not on a CUDA device.

Tensors: images are ``uint8 [H, W, 4]`` (batches ``[N, H, W, 4]``), the LUT is ``int32
[65536]`` (reinterpreted as uint32), coordinates are ``int32 [H, W]`` holding ``x | y << 16``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import SB_HOST_RGB, SB_JITTER_ZERO, SB_LABEL, SB_LUT_RGB, SB_NO_COLOR, StyleBlitError, check, lib

__all__ = [
    "Params", "build_lut", "build_lut3", "exemplar_bytes", "prepare_exemplar", "stylize", "stylize_batch", "vote", "stylize_batch_host", "launch_count",
    "version", "SB_JITTER_ZERO", "SB_NO_COLOR", "SB_LABEL", "SB_LUT_RGB", "SB_HOST_RGB", "StyleBlitError",
]


@dataclass
class Params:
    """sb_params: the paper's t and L plus blend radius, channels, jitter seed."""

    threshold: float
    levels: int
    blend_radius: int = 0
    guide_channels: int = 3
    seed: int = 0x5EED
    flags: int = 0
    row_begin: int = 0
    row_end: int = 0
    weights: tuple = (0, 0, 0, 0)  # per-channel integer weights; all zero = unit weights
    label_channel: int | None = None  # segmentation label byte (sets SB_LABEL)
    lut_rgb: bool = False             # `lut` is the 2^24-entry table of build_lut3 (sets SB_LUT_RGB)
    exemplar: torch.Tensor | None = None  # strided exemplar copy of prepare_exemplar(cs, gs) (speed only)

    def c(self) -> _lib.SbParams:
        flags = int(self.flags) | (SB_LABEL if self.label_channel is not None else 0)
        flags |= SB_LUT_RGB if self.lut_rgb else 0
        w = (C.c_uint8 * 4)(*[int(v) for v in self.weights])
        return _lib.SbParams(float(self.threshold), int(self.levels), int(self.blend_radius),
                             int(self.guide_channels), int(self.seed) & 0xFFFFFFFF, flags,
                             int(self.row_begin), int(self.row_end), w,
                             -1 if self.label_channel is None else int(self.label_channel),
                             None if self.exemplar is None else _dev(self.exemplar, "exemplar", torch.uint8, (1,)))


def _dev(t: torch.Tensor, name: str, dtype: torch.dtype, ndim: tuple[int, ...]) -> int:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() not in ndim:
        raise ValueError(f"{name} must have {ndim} dims, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _img_wh(t: torch.Tensor, name: str) -> tuple[int, int]:
    if t.shape[-1] != 4:
        raise ValueError(f"{name} must have 4 bytes per pixel, got shape {tuple(t.shape)}")
    return int(t.shape[-2]), int(t.shape[-3])


def _stream(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def build_lut(gs: torch.Tensor, lut: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
              stream=None) -> torch.Tensor:
    """sb_build_lut: the exact 256x256 guide look-up table of G_S."""
    _dev(gs, "gs", torch.uint8, (3,))
    ws, hs = _img_wh(gs, "gs")
    if lut is None:
        lut = torch.empty(65536, dtype=torch.int32, device=gs.device)
    _dev(lut, "lut", torch.int32, (1,))
    if workspace is None:
        workspace = torch.empty(lib().sb_lut_workspace_bytes(), dtype=torch.uint8, device=gs.device)
    check(lib().sb_build_lut(gs.data_ptr(), ws, hs, lut.data_ptr(), workspace.data_ptr(), _stream(stream)))
    return lut


def build_lut3(gs: torch.Tensor, lut3: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
               stream=None) -> torch.Tensor:
    """sb_build_lut3: the exact 3-channel guide search tabulated for all 2^24 keys
    ("or a tree search"; R26).  64 MiB table, 128 MiB workspace."""
    _dev(gs, "gs", torch.uint8, (3,))
    ws, hs = _img_wh(gs, "gs")
    if lut3 is None:
        lut3 = torch.empty(1 << 24, dtype=torch.int32, device=gs.device)
    _dev(lut3, "lut3", torch.int32, (1,))
    if workspace is None:
        workspace = torch.empty(lib().sb_lut3_workspace_bytes(), dtype=torch.uint8, device=gs.device)
    check(lib().sb_build_lut3(gs.data_ptr(), ws, hs, lut3.data_ptr(), workspace.data_ptr(), _stream(stream)))
    return lut3


def exemplar_bytes(ws: int, hs: int) -> int:
    """sb_exemplar_bytes: size of the strided exemplar copy (2 * hs * 2^18 bytes)."""
    return int(lib().sb_exemplar_bytes(int(ws), int(hs)))


def prepare_exemplar(cs: torch.Tensor, gs: torch.Tensor, out: torch.Tensor | None = None,
                     stream=None) -> torch.Tensor:
    """sb_prepare_exemplar: G_S and C_S copied to rows of 2^16 pixels, so the stylize kernel's
    exemplar gathers index them with the packed coordinate itself.  Pass
    the result as Params(exemplar=...); results are identical with and without it."""
    _dev(cs, "cs", torch.uint8, (3,))
    _dev(gs, "gs", torch.uint8, (3,))
    ws, hs = _img_wh(gs, "gs")
    if _img_wh(cs, "cs") != (ws, hs):
        raise ValueError("cs and gs must have the same size")
    if exemplar_bytes(ws, hs) == 0:
        raise ValueError(f"no strided exemplar copy for a {ws}x{hs} exemplar (hs > SB_EXEMPLAR_MAX_HS); "
                         "use Params(exemplar=None)")
    if out is None:
        out = torch.empty(exemplar_bytes(ws, hs), dtype=torch.uint8, device=gs.device)
    _dev(out, "out", torch.uint8, (1,))
    if out.numel() < exemplar_bytes(ws, hs):
        raise ValueError(f"out has {out.numel()} bytes; needs {exemplar_bytes(ws, hs)}")
    check(lib().sb_prepare_exemplar(cs.data_ptr(), gs.data_ptr(), ws, hs, out.data_ptr(), _stream(stream)))
    return out


def _check_lut(prm: Params, lut: torch.Tensor) -> None:
    want = (1 << 24) if prm.lut_rgb else 65536
    if lut.numel() != want:
        raise ValueError(f"lut has {lut.numel()} entries; {'lut_rgb' if prm.lut_rgb else '2-channel'} needs {want}")


def _check_out(t: torch.Tensor, name: str, shape: tuple[int, ...], dtype: torch.dtype, device) -> None:
    """A caller-supplied output must match exactly: the ABI takes raw pointers, so a short
    buffer would be overrun by the kernels."""
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.device != torch.device(device):
        raise ValueError(f"{name} is on {t.device}, the inputs on {device}")
    if t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor of shape {tuple(shape)}, "
                         f"got {t.dtype} {tuple(t.shape)}")


def _outputs(prm: Params, shape_px: tuple[int, ...], device, ct, coords, level, want_level: bool):
    no_color = bool(prm.flags & SB_NO_COLOR)
    if ct is None and not no_color:
        ct = torch.empty(*shape_px, 4, dtype=torch.uint8, device=device)
    elif ct is not None:
        _check_out(ct, "ct", (*shape_px, 4), torch.uint8, device)
    if coords is None:
        coords = torch.empty(*shape_px, dtype=torch.int32, device=device)
    else:
        _check_out(coords, "coords", shape_px, torch.int32, device)
    if level is None and want_level:
        level = torch.empty(*shape_px, dtype=torch.uint8, device=device)
    elif level is not None:
        _check_out(level, "level", shape_px, torch.uint8, device)
    return ct, coords, level


def _check_exemplar(ex: torch.Tensor | None, ws: int, hs: int, device) -> None:
    if ex is None:
        return
    need = exemplar_bytes(ws, hs)
    if need == 0:
        raise ValueError(f"no strided exemplar copy for a {ws}x{hs} exemplar (hs > SB_EXEMPLAR_MAX_HS); pass None")
    if ex.device != torch.device(device) or ex.dtype != torch.uint8 or ex.numel() < need:
        raise ValueError(f"exemplar must be a uint8 tensor of >= {need} bytes on {device} "
                         f"(prepare_exemplar(cs, gs)), got {ex.dtype} {ex.numel()} bytes on {ex.device}")


def _seeds(frame_seeds, n: int):
    """frame_seeds -> a HOST uint32 array the ABI reads during the call.  A contiguous 1-D numpy
    uint32 array (or CPU uint32-compatible tensor) is passed without copying; other sequences
    are reduced mod 2^32 (a 4096-entry Python list costs ~0.1 ms; precompute arrays in loops)."""
    if frame_seeds is None:
        return None
    if isinstance(frame_seeds, torch.Tensor):
        if frame_seeds.is_cuda:
            raise ValueError("frame_seeds must be a HOST array")
        frame_seeds = frame_seeds.numpy()
    if isinstance(frame_seeds, np.ndarray) and frame_seeds.dtype == np.uint32 and frame_seeds.ndim == 1:
        arr = np.ascontiguousarray(frame_seeds)
    else:
        arr = (np.asarray(frame_seeds, dtype=np.int64).reshape(-1) & 0xFFFFFFFF).astype(np.uint32)
    if arr.shape[0] != n:
        raise ValueError(f"frame_seeds has {arr.shape[0]} entries for {n} frames")
    return arr


def _u32ptr(arr):
    return None if arr is None else arr.ctypes.data_as(C.POINTER(C.c_uint32))


def stylize(prm: Params, cs: torch.Tensor, gs: torch.Tensor, lut: torch.Tensor, gt: torch.Tensor,
            ct: torch.Tensor | None = None, coords: torch.Tensor | None = None, level: torch.Tensor | None = None,
            want_level: bool = True, stream=None):
    """sb_stylize: Alg. 2 for every pixel of G_T (+ voting when prm.blend_radius > 0).
    Returns (ct, coords, level)."""
    return stylize_batch(prm, cs, gs, lut, gt.unsqueeze(0), None,
                         None if ct is None else ct.unsqueeze(0),
                         None if coords is None else coords.unsqueeze(0),
                         None if level is None else level.unsqueeze(0), want_level, stream, _squeeze=True)


def stylize_batch(prm: Params, cs: torch.Tensor, gs: torch.Tensor, lut: torch.Tensor, gt: torch.Tensor,
                  frame_seeds=None, ct: torch.Tensor | None = None, coords: torch.Tensor | None = None,
                  level: torch.Tensor | None = None, want_level: bool = True, stream=None, _squeeze: bool = False):
    """sb_stylize_batch over gt [N, H, W, 4]; frame i jittered with frame_seeds[i]
    (default prm.seed + i).  Returns (ct, coords, level)."""
    _dev(cs, "cs", torch.uint8, (3,))
    _dev(gs, "gs", torch.uint8, (3,))
    _dev(lut, "lut", torch.int32, (1,))
    _check_lut(prm, lut)
    _dev(gt, "gt", torch.uint8, (4,))
    ws, hs = _img_wh(gs, "gs")
    if _img_wh(cs, "cs") != (ws, hs):
        raise ValueError("cs and gs must have the same size")
    n = int(gt.shape[0])
    wt, ht = _img_wh(gt, "gt")
    ct, coords, level = _outputs(prm, (n, ht, wt), gt.device, ct, coords, level, want_level)
    _check_exemplar(prm.exemplar, ws, hs, gt.device)
    for t, name in ((cs, "cs"), (gs, "gs"), (lut, "lut")):
        if t.device != gt.device:
            raise ValueError(f"{name} is on {t.device}, gt on {gt.device}")
    ptr = lambda t, name, dt, nd: 0 if t is None else _dev(t, name, dt, nd)  # noqa: E731
    seeds = _seeds(frame_seeds, n)
    p = prm.c()
    check(lib().sb_stylize_batch(C.byref(p), n, _u32ptr(seeds), cs.data_ptr(), gs.data_ptr(), ws, hs, lut.data_ptr(),
                                 gt.data_ptr(), wt, ht, ptr(ct, "ct", torch.uint8, (4,)),
                                 ptr(coords, "coords", torch.int32, (3,)), ptr(level, "level", torch.uint8, (3,)),
                                 _stream(stream)))
    if _squeeze:
        sq = lambda t: None if t is None else t[0]  # noqa: E731
        return sq(ct), sq(coords), sq(level)
    return ct, coords, level


def vote(coords: torch.Tensor, cs: torch.Tensor, r: int, ct: torch.Tensor | None = None,
         row_begin: int = 0, row_end: int = 0, exemplar: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """sb_vote: C_T from a coordinate field.  coords [H,W] or [N,H,W] int32.
    exemplar: optional strided copy from prepare_exemplar(cs, gs) (speed only)."""
    squeeze = coords.dim() == 2
    co = coords.unsqueeze(0) if squeeze else coords
    _dev(co, "coords", torch.int32, (3,))
    _dev(cs, "cs", torch.uint8, (3,))
    n, ht, wt = (int(v) for v in co.shape)
    ws, hs = _img_wh(cs, "cs")
    if ct is None:
        ct = torch.empty(n, ht, wt, 4, dtype=torch.uint8, device=co.device)
    elif squeeze:
        ct = ct.unsqueeze(0)
    _check_out(ct, "ct", (n, ht, wt, 4), torch.uint8, co.device)
    if cs.device != co.device:
        raise ValueError(f"cs is on {cs.device}, coords on {co.device}")
    _check_exemplar(exemplar, ws, hs, co.device)
    ex = None if exemplar is None else _dev(exemplar, "exemplar", torch.uint8, (1,))
    check(lib().sb_vote(co.data_ptr(), n, wt, ht, cs.data_ptr(), ws, hs, int(r), ct.data_ptr(), int(row_begin),
                        int(row_end), ex, _stream(stream)))
    return ct[0] if squeeze else ct


def host_workspace(wt: int, ht: int, blend_radius: int = 0, depth: int = 2, device="cuda") -> torch.Tensor:
    return torch.empty(lib().sb_host_workspace_bytes(wt, ht, blend_radius, depth), dtype=torch.uint8, device=device)


def stylize_batch_host(prm: Params, cs: torch.Tensor, gs: torch.Tensor, lut: torch.Tensor, gt_host: torch.Tensor,
                       ct_host: torch.Tensor, coords_host: torch.Tensor | None = None, frame_seeds=None,
                       workspace: torch.Tensor | None = None, depth: int = 2, stream=None):
    """sb_stylize_batch_host: HOST gt [N,H,W,4] in, HOST ct [N,H,W,4] out (pinned memory for
    full copy bandwidth); copies and compute overlap inside the library.  Blocks until done.
    With prm.flags & SB_HOST_RGB the host frames are packed RGB: gt [N,H,W,3], ct [N,H,W,3]."""
    ch = 3 if prm.flags & SB_HOST_RGB else 4
    for t, name in ((gt_host, "gt_host"), (ct_host, "ct_host")):
        if t.is_cuda or t.dtype != torch.uint8 or not t.is_contiguous() or t.dim() != 4 or t.shape[-1] != ch:
            raise ValueError(f"{name} must be a contiguous host uint8 [N,H,W,{ch}] tensor")
    if tuple(ct_host.shape) != tuple(gt_host.shape):
        raise ValueError(f"ct_host shape {tuple(ct_host.shape)} != gt_host shape {tuple(gt_host.shape)}")
    n = int(gt_host.shape[0])
    wt, ht = int(gt_host.shape[2]), int(gt_host.shape[1])
    if coords_host is not None:
        if (coords_host.is_cuda or coords_host.dtype != torch.int32 or not coords_host.is_contiguous()
                or tuple(coords_host.shape) != (n, ht, wt)):
            raise ValueError(f"coords_host must be a contiguous host int32 tensor of shape {(n, ht, wt)}")
    ws, hs = _img_wh(gs, "gs")
    if workspace is None:
        workspace = host_workspace(wt, ht, prm.blend_radius, depth, device=cs.device)
    need = int(lib().sb_host_workspace_bytes(wt, ht, prm.blend_radius, depth))
    if workspace.device != cs.device or workspace.numel() * workspace.element_size() < need:
        raise ValueError(f"workspace must hold >= {need} bytes on {cs.device}")
    _check_exemplar(prm.exemplar, ws, hs, cs.device)
    seeds = _seeds(frame_seeds, n)
    _check_lut(prm, lut)
    p = prm.c()
    check(lib().sb_stylize_batch_host(C.byref(p), n, _u32ptr(seeds), _dev(cs, "cs", torch.uint8, (3,)),
                                      _dev(gs, "gs", torch.uint8, (3,)), ws, hs, _dev(lut, "lut", torch.int32, (1,)),
                                      gt_host.data_ptr(), wt, ht, ct_host.data_ptr(),
                                      0 if coords_host is None else coords_host.data_ptr(),
                                      workspace.data_ptr(), workspace.numel(), depth, _stream(stream)))
    return ct_host


def launch_count() -> int:
    """Kernels launched by the last ABI call on this thread."""
    return int(lib().sb_last_launch_count())


def version() -> str:
    return lib().sb_version().decode()
