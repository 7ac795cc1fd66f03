"""CPU oracle for StyleBlit (arXiv 1807.03249) -- TEST INFRASTRUCTURE ONLY.

A ctypes front end over ``oracle/styleblit_oracle.c`` (plain C99, fp64 where the paper
writes real-valued formulas).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this module.
The product package ``paper_1807_03249_b200`` never imports it and shares no code with it.

Every function follows PAPER.md Alg. 2 (lines 337-393) and the voting paragraph
(lines 412-421); the readings of ambiguous passages (R1..R27) are listed in DESIGN.md.
Parity of every function is pinned by tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "styleblit_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

# Built with -O2 and NO -ffast-math: the fp64 comparisons must be IEEE exact.
CFLAGS = ["-std=c99", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", "-pthread"]


def build(force: bool = False) -> str:
    """Compile the oracle into oracle/liboracle.so (gcc)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "styleblit_oracle.h"))
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class _Params(C.Structure):
    _fields_ = [
        ("t", C.c_double),
        ("L", C.c_int32),
        ("C", C.c_int32),
        ("seed", C.c_uint32),
        ("zero_jitter", C.c_int32),
        ("w", C.c_int32 * 4),
        ("label_channel", C.c_int32),
        ("lut_rgb", C.c_int32),
    ]


@dataclass
class Params:
    """The paper's inputs t and L plus readings R5/R11/R18."""

    t: float
    L: int
    C: int = 3
    seed: int = 0x5EED
    zero_jitter: bool = False
    weights: tuple = (1, 1, 1, 1)   # per-channel weights of e^2
    label_channel: int | None = None  # segmentation label byte
    lut_rgb: bool = False             # u* by exact search over channels 0..2 (R26)

    def c(self) -> _Params:
        # The GPU ABI takes t as float32; the oracle sees the same real number.
        return _Params(float(np.float32(self.t)), self.L, self.C, self.seed & 0xFFFFFFFF,
                       1 if self.zero_jitter else 0, (C.c_int32 * 4)(*[int(v) for v in self.weights]),
                       -1 if self.label_channel is None else int(self.label_channel),
                       1 if self.lut_rgb else 0)


_lib = None


def lib():
    global _lib
    if _lib is None:
        l = C.CDLL(build())
        u8p, u32p, i32 = C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.c_int32
        l.or_lowbias32.restype = C.c_uint32
        l.or_lowbias32.argtypes = [C.c_uint32]
        l.or_cell_hash.restype = C.c_uint32
        l.or_cell_hash.argtypes = [i32, i32, i32, C.c_uint32]
        l.or_jitter.argtypes = [i32, i32, i32, C.c_uint32, i32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        l.or_seed_point_j.argtypes = [i32, i32, i32, C.c_double, C.c_double, C.POINTER(i32), C.POINTER(i32)]
        l.or_seed_point.argtypes = [i32, i32, i32, C.c_uint32, i32, C.POINTER(i32), C.POINTER(i32)]
        l.or_nearest_seed.argtypes = [i32, i32, i32, C.c_uint32, i32, C.POINTER(i32), C.POINTER(i32)]
        l.or_lut_entry.restype = C.c_uint32
        l.or_lut_entry.argtypes = [u8p, i32, i32, i32, i32]
        l.or_build_lut.argtypes = [u8p, i32, i32, u32p, i32]
        l.or_stylize_pixel.argtypes = [C.POINTER(_Params), u8p, i32, i32, u32p, u8p, i32, i32, i32, i32,
                                       C.POINTER(C.c_uint32), C.POINTER(C.c_uint8)]
        l.or_stylize.argtypes = [C.POINTER(_Params), u8p, u8p, i32, i32, u32p, u8p, i32, i32, u8p, u32p, u8p, i32]
        l.or_vote.argtypes = [u32p, i32, i32, u8p, i32, i32, i32, u8p, i32]
        l.or_lut3_entry.restype = C.c_uint32
        l.or_lut3_entry.argtypes = [u8p, i32, i32, i32, i32, i32]
        l.or_lut3_entries.argtypes = [u8p, i32, i32, u32p, C.c_int64, u32p, i32]
        l.or_blit_bruteforce.argtypes = [C.POINTER(_Params), u8p, u8p, i32, i32, u32p, u8p, i32, i32, u8p, u32p, u8p]
        l.or_version.restype = C.c_char_p
        _lib = l
    return _lib


def _u8(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _u32(a: np.ndarray | None):
    if a is None:
        return C.POINTER(C.c_uint32)()
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _img(a: np.ndarray) -> tuple[int, int]:
    assert a.ndim == 3 and a.shape[2] == 4 and a.dtype == np.uint8, a.shape
    return a.shape[1], a.shape[0]


# ---------------------------------------------------------------------------------------
def lowbias32(x: int) -> int:
    return lib().or_lowbias32(x & 0xFFFFFFFF)


def cell_hash(bx: int, by: int, l: int, seed: int) -> int:
    return lib().or_cell_hash(bx, by, l, seed & 0xFFFFFFFF)


def jitter(bx: int, by: int, l: int, seed: int, zero_jitter: bool = False) -> tuple[float, float]:
    jx, jy = C.c_double(), C.c_double()
    lib().or_jitter(bx, by, l, seed & 0xFFFFFFFF, int(zero_jitter), C.byref(jx), C.byref(jy))
    return jx.value, jy.value


def seed_point_j(px: int, py: int, h: int, jx: float, jy: float) -> tuple[int, int]:
    sx, sy = C.c_int32(), C.c_int32()
    lib().or_seed_point_j(px, py, h, jx, jy, C.byref(sx), C.byref(sy))
    return sx.value, sy.value


def seed_point(px: int, py: int, l: int, seed: int, zero_jitter: bool = False) -> tuple[int, int]:
    sx, sy = C.c_int32(), C.c_int32()
    lib().or_seed_point(px, py, l, seed & 0xFFFFFFFF, int(zero_jitter), C.byref(sx), C.byref(sy))
    return sx.value, sy.value


def nearest_seed(px: int, py: int, l: int, seed: int, zero_jitter: bool = False) -> tuple[int, int]:
    qx, qy = C.c_int32(), C.c_int32()
    lib().or_nearest_seed(px, py, l, seed & 0xFFFFFFFF, int(zero_jitter), C.byref(qx), C.byref(qy))
    return qx.value, qy.value


def lut_entry(gs: np.ndarray, g0: int, g1: int) -> int:
    ws, hs = _img(gs)
    return lib().or_lut_entry(_u8(gs), ws, hs, g0, g1)


def lut3_entry(gs: np.ndarray, g0: int, g1: int, g2: int) -> int:
    ws, hs = _img(gs)
    return lib().or_lut3_entry(_u8(gs), ws, hs, g0, g1, g2)


def lut3_entries(gs: np.ndarray, keys: np.ndarray, nthreads: int = 1) -> np.ndarray:
    """Exact 3-channel search for keys g0 | g1<<8 | g2<<16 (R26)."""
    ws, hs = _img(gs)
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    out = np.zeros(keys.shape, np.uint32)
    lib().or_lut3_entries(_u8(gs), ws, hs, _u32(keys), keys.size, _u32(out), nthreads)
    return out


def build_lut(gs: np.ndarray, nthreads: int = 1) -> np.ndarray:
    ws, hs = _img(gs)
    lut = np.zeros(65536, np.uint32)
    lib().or_build_lut(_u8(gs), ws, hs, _u32(lut), nthreads)
    return lut


def stylize_pixel(prm: Params, gs, lut, gt, px: int, py: int) -> tuple[int, int]:
    ws, hs = _img(gs)
    wt, ht = _img(gt)
    c, lv = C.c_uint32(), C.c_uint8()
    p = prm.c()
    lib().or_stylize_pixel(C.byref(p), _u8(gs), ws, hs, _u32(lut), _u8(gt), wt, ht, px, py,
                           C.byref(c), C.byref(lv))
    return c.value, lv.value


def stylize(prm: Params, cs, gs, lut, gt, nthreads: int = 1):
    """Returns (ct, coords, level) for one frame (blit colours)."""
    ws, hs = _img(gs)
    assert _img(cs) == (ws, hs)
    wt, ht = _img(gt)
    ct = np.zeros((ht, wt, 4), np.uint8)
    coords = np.zeros((ht, wt), np.uint32)
    level = np.zeros((ht, wt), np.uint8)
    p = prm.c()
    lib().or_stylize(C.byref(p), _u8(cs), _u8(gs), ws, hs, _u32(lut), _u8(gt), wt, ht,
                     _u8(ct), _u32(coords), _u8(level), nthreads)
    return ct, coords, level


def blit_bruteforce(prm: Params, cs, gs, lut, gt):
    """Alg. 1: (ct, coords, level), level 1 = copied, 0 = fallback."""
    ws, hs = _img(gs)
    wt, ht = _img(gt)
    ct = np.zeros((ht, wt, 4), np.uint8)
    coords = np.zeros((ht, wt), np.uint32)
    level = np.zeros((ht, wt), np.uint8)
    p = prm.c()
    lib().or_blit_bruteforce(C.byref(p), _u8(cs), _u8(gs), ws, hs, _u32(lut), _u8(gt), wt, ht,
                             _u8(ct), _u32(coords), _u8(level))
    return ct, coords, level


def vote(coords: np.ndarray, cs: np.ndarray, r: int, nthreads: int = 1) -> np.ndarray:
    ht, wt = coords.shape
    ws, hs = _img(cs)
    ct = np.zeros((ht, wt, 4), np.uint8)
    coords = np.ascontiguousarray(coords, dtype=np.uint32)
    lib().or_vote(_u32(coords), wt, ht, _u8(cs), ws, hs, r, _u8(ct), nthreads)
    return ct


def version() -> str:
    return lib().or_version().decode()
