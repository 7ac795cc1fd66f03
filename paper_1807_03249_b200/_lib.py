"""ctypes loader for libstyleblit.so (the C ABI of include/styleblit.h).

Argument marshalling only.  There is no fallback: if the shared library is missing or fails
to load, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libstyleblit.so")
# development hook for A/B timing of kernel variants: another build of the same library
SO_PATH = os.environ.get("SB_LIBRARY", SO_PATH)

SB_OK, SB_EINVAL, SB_EUNSUPPORTED, SB_ECUDA = 0, 1, 2, 3
SB_JITTER_ZERO = 0x1
SB_NO_COLOR = 0x2
SB_LABEL = 0x4
SB_LUT_RGB = 0x8
SB_HOST_RGB = 0x10
SB_MAX_LEVELS = 15
SB_MAX_RADIUS = 8

# every symbol include/styleblit.h declares
EXPORTS = (
    "sb_lut_workspace_bytes", "sb_build_lut", "sb_lut3_workspace_bytes", "sb_build_lut3", "sb_exemplar_bytes",
    "sb_prepare_exemplar", "sb_stylize", "sb_stylize_batch", "sb_vote",
    "sb_host_workspace_bytes", "sb_stylize_batch_host", "sb_last_launch_count",
    "sb_last_error", "sb_version",
)


class SbParams(C.Structure):
    _fields_ = [
        ("threshold", C.c_float),
        ("levels", C.c_int32),
        ("blend_radius", C.c_int32),
        ("guide_channels", C.c_int32),
        ("seed", C.c_uint32),
        ("flags", C.c_uint32),
        ("row_begin", C.c_int32),
        ("row_end", C.c_int32),
        ("weights", C.c_uint8 * 4),
        ("label_channel", C.c_int32),
        ("exemplar", C.c_void_p),
    ]


class StyleBlitError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"status {status}: {msg}")
        self.status = status


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(
            f"{SO_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    l = C.CDLL(SO_PATH)
    vp, i32, u32p, u8p = C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p
    l.sb_lut_workspace_bytes.restype = C.c_size_t
    l.sb_lut_workspace_bytes.argtypes = []
    l.sb_build_lut.restype = C.c_int
    l.sb_build_lut.argtypes = [u8p, i32, i32, u32p, vp, vp]
    l.sb_lut3_workspace_bytes.restype = C.c_size_t
    l.sb_lut3_workspace_bytes.argtypes = []
    l.sb_build_lut3.restype = C.c_int
    l.sb_build_lut3.argtypes = [u8p, i32, i32, u32p, vp, vp]
    l.sb_exemplar_bytes.restype = C.c_size_t
    l.sb_exemplar_bytes.argtypes = [i32, i32]
    l.sb_prepare_exemplar.restype = C.c_int
    l.sb_prepare_exemplar.argtypes = [u8p, u8p, i32, i32, u8p, vp]
    l.sb_stylize.restype = C.c_int
    l.sb_stylize.argtypes = [C.POINTER(SbParams), u8p, u8p, i32, i32, u32p, u8p, i32, i32, u8p, u32p, u8p, vp]
    l.sb_stylize_batch.restype = C.c_int
    l.sb_stylize_batch.argtypes = [C.POINTER(SbParams), i32, C.POINTER(C.c_uint32), u8p, u8p, i32, i32, u32p, u8p,
                                   i32, i32, u8p, u32p, u8p, vp]
    l.sb_vote.restype = C.c_int
    l.sb_vote.argtypes = [u32p, i32, i32, i32, u8p, i32, i32, i32, u8p, i32, i32, u8p, vp]
    l.sb_host_workspace_bytes.restype = C.c_size_t
    l.sb_host_workspace_bytes.argtypes = [i32, i32, i32, i32]
    l.sb_stylize_batch_host.restype = C.c_int
    l.sb_stylize_batch_host.argtypes = [C.POINTER(SbParams), i32, C.POINTER(C.c_uint32), u8p, u8p, i32, i32, u32p,
                                        u8p, i32, i32, u8p, u32p, vp, C.c_size_t, i32, vp]
    l.sb_last_launch_count.restype = C.c_int32
    l.sb_last_error.restype = C.c_char_p
    l.sb_version.restype = C.c_char_p
    _lib = l
    return l


def check(status: int) -> None:
    if status != SB_OK:
        raise StyleBlitError(status, lib().sb_last_error().decode())
