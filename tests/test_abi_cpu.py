"""Host-side checks of the C ABI that need no GPU: the library builds for sm_100a, loads, exports
every symbol include/styleblit.h declares, and rejects invalid arguments with the documented
status codes before touching the device."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_1807_03249_b200 as sb
from paper_1807_03249_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _lib.lib()


def header_symbols():
    syms = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", fn)).read()
            txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
            syms |= set(re.findall(r"\b(sb_[a-z_0-9]+)\s*\(", txt))
    return syms


def test_exports_every_declared_symbol(lib):
    declared = header_symbols()
    assert declared == set(_lib.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.SO_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sb_[a-z_0-9]+)", out))
    assert declared <= exported, declared - exported
    for s in declared:
        assert hasattr(lib, s)


def test_sm100a_cubin_present(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.SO_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_workspace(lib):
    assert b"sm_100a" in lib.sb_version()
    assert lib.sb_lut_workspace_bytes() == 65536 * 12
    assert lib.sb_lut3_workspace_bytes() == (1 << 24) * 8
    assert lib.sb_host_workspace_bytes(3840, 2160, 0, 2) >= 2 * 3 * 3840 * 2160 * 4
    assert lib.sb_host_workspace_bytes(0, 10, 0, 2) == 0


def _prm(**kw):
    d = dict(threshold=10.0, levels=5, blend_radius=0, guide_channels=3, seed=1, flags=0, row_begin=0, row_end=0)
    d.update(kw)
    return _lib.SbParams(**d)


FAKE = 0x10000  # never dereferenced: validation fails first


@pytest.mark.parametrize("kw,needle", [
    (dict(threshold=-1.0), "threshold"),
    (dict(threshold=float("nan")), "threshold"),
    (dict(threshold=float("inf")), "threshold"),
    (dict(levels=0), "levels"),
    (dict(levels=16), "levels"),
    (dict(blend_radius=-1), "blend_radius"),
    (dict(blend_radius=9), "blend_radius"),
    (dict(guide_channels=1), "guide_channels"),
    (dict(guide_channels=5), "guide_channels"),
    (dict(flags=0x80), "flags"),
    (dict(row_begin=5, row_end=5), "row"),
    (dict(row_begin=-1, row_end=5), "row"),
    (dict(row_begin=0, row_end=65), "row"),
])
def test_invalid_params(lib, kw, needle):
    p = _prm(**kw)
    st = lib.sb_stylize(C.byref(p), FAKE, FAKE, 64, 64, FAKE, FAKE, 64, 64, FAKE, FAKE, 0, None)
    assert st == _lib.SB_EINVAL
    assert needle in lib.sb_last_error().decode()


@pytest.mark.parametrize("args,needle", [
    (dict(cs=0), "cs"), (dict(gs=0), "gs"), (dict(lut=0), "lut"), (dict(gt=0), "gt"), (dict(ct=0), "ct"),
    (dict(ws=0), "source"), (dict(hs=65536), "source"), (dict(wt=65536), "target"),
    (dict(gt=FAKE + 4), "aligned"),
])
def test_invalid_pointers_and_sizes(lib, args, needle):
    a = dict(cs=FAKE, gs=FAKE, ws=64, hs=64, lut=FAKE, gt=FAKE, wt=64, ht=64, ct=FAKE, coords=FAKE)
    a.update(args)
    p = _prm()
    st = lib.sb_stylize(C.byref(p), a["cs"], a["gs"], a["ws"], a["hs"], a["lut"], a["gt"], a["wt"], a["ht"],
                        a["ct"], a["coords"], 0, None)
    assert st == _lib.SB_EINVAL
    assert needle in lib.sb_last_error().decode()


def test_limits_match_survey_8b(lib):
    """sides in [1, 65535], L in [1, 15], r in [0, 8] are accepted (validation only:
    n_frames = 0 launches nothing)."""
    for kw, dims in ((dict(levels=15), (64, 64, 64, 64)), (dict(blend_radius=8), (64, 64, 64, 64)),
                     (dict(), (65535, 1, 65535, 1)), (dict(), (1, 65535, 1, 65535))):
        p = _prm(**kw)
        ws, hs, wt, ht = dims
        st = lib.sb_stylize_batch(C.byref(p), 0, None, FAKE, FAKE, ws, hs, FAKE, FAKE, wt, ht, FAKE, FAKE, 0, None)
        assert st == _lib.SB_OK, (kw, dims, lib.sb_last_error().decode())
    assert _lib.SB_MAX_LEVELS == 15 and _lib.SB_MAX_RADIUS == 8


def test_vote_needs_coords(lib):
    p = _prm(blend_radius=2)
    st = lib.sb_stylize(C.byref(p), FAKE, FAKE, 64, 64, FAKE, FAKE, 64, 64, FAKE, 0, 0, None)
    assert st == _lib.SB_EINVAL and "coords" in lib.sb_last_error().decode()


def test_no_color_allows_null_ct(lib):
    # ct may be NULL with SB_NO_COLOR: validation passes (on this GPU-less host the launch then
    # fails with SB_ECUDA); without the flag the same call is SB_EINVAL naming ct
    p = _prm(flags=_lib.SB_NO_COLOR)
    st = lib.sb_stylize(C.byref(p), FAKE, FAKE, 64, 64, FAKE, FAKE, 64, 64, 0, FAKE, 0, None)
    assert st != _lib.SB_EINVAL, lib.sb_last_error().decode()
    st = lib.sb_stylize(C.byref(_prm()), FAKE, FAKE, 64, 64, FAKE, FAKE, 64, 64, 0, FAKE, 0, None)
    assert st == _lib.SB_EINVAL and "ct" in lib.sb_last_error().decode()


def test_empty_batch_allows_null_frame_buffers(lib):
    """n_frames = 0: the per-frame buffers hold zero bytes and may be NULL (styleblit.h); the
    exemplar-level inputs are still required; nothing is launched."""
    p = _prm(blend_radius=2)
    assert lib.sb_stylize_batch(C.byref(p), 0, None, FAKE, FAKE, 64, 64, FAKE, 0, 64, 64, 0, 0, 0, None) == _lib.SB_OK
    assert lib.sb_last_launch_count() == 0
    assert lib.sb_stylize_batch(C.byref(p), 0, None, 0, FAKE, 64, 64, FAKE, 0, 64, 64, 0, 0, 0, None) == _lib.SB_EINVAL
    assert lib.sb_vote(0, 0, 64, 64, FAKE, 64, 64, 2, 0, 0, 0, None, None) == _lib.SB_OK
    assert lib.sb_vote(0, 1, 64, 64, FAKE, 64, 64, 2, 0, 0, 0, None, None) == _lib.SB_EINVAL


def test_build_lut_invalid(lib):
    assert lib.sb_build_lut(0, 4, 4, FAKE, FAKE, None) == _lib.SB_EINVAL
    assert lib.sb_build_lut(FAKE, 4, 4, FAKE, 0, None) == _lib.SB_EINVAL
    assert "workspace" in lib.sb_last_error().decode()
    assert lib.sb_build_lut(FAKE, 0, 4, FAKE, FAKE, None) == _lib.SB_EINVAL


def test_build_lut3_invalid(lib):
    assert lib.sb_build_lut3(0, 4, 4, FAKE, FAKE, None) == _lib.SB_EINVAL
    assert "gs" in lib.sb_last_error().decode()
    assert lib.sb_build_lut3(FAKE, 4, 4, 0, FAKE, None) == _lib.SB_EINVAL
    assert lib.sb_build_lut3(FAKE, 4, 4, FAKE, 0, None) == _lib.SB_EINVAL
    assert "sb_lut3_workspace_bytes" in lib.sb_last_error().decode()
    assert lib.sb_build_lut3(FAKE, 4, 65536, FAKE, FAKE, None) == _lib.SB_EINVAL


def test_exemplar_copy_abi(lib):
    assert lib.sb_exemplar_bytes(512, 512) == 2 * 512 * (1 << 18)
    assert lib.sb_exemplar_bytes(37, 29) == 2 * 29 * (1 << 18)
    assert lib.sb_exemplar_bytes(0, 5) == 0 and lib.sb_exemplar_bytes(40000, 5) == 0
    assert lib.sb_prepare_exemplar(FAKE, FAKE, 4, 4, 0, None) == _lib.SB_EINVAL
    assert "sb_exemplar_bytes" in lib.sb_last_error().decode()
    assert lib.sb_prepare_exemplar(0, FAKE, 4, 4, FAKE, None) == _lib.SB_EINVAL
    assert lib.sb_prepare_exemplar(FAKE, FAKE, 4, 4, FAKE + 4, None) == _lib.SB_EINVAL
    assert "aligned" in lib.sb_last_error().decode()
    p = _prm()
    p.exemplar = FAKE + 8   # misaligned strided copy is refused before any launch
    st = lib.sb_stylize(C.byref(p), FAKE, FAKE, 64, 64, FAKE, FAKE, 64, 64, FAKE, 0, 0, None)
    assert st == _lib.SB_EINVAL and "exemplar" in lib.sb_last_error().decode()


def test_host_rgb_flag(lib):
    p = _prm(flags=_lib.SB_HOST_RGB)
    # device entry points refuse it
    st = lib.sb_stylize(C.byref(p), FAKE, FAKE, 64, 64, FAKE, FAKE, 64, 64, FAKE, 0, 0, None)
    assert st == _lib.SB_EINVAL and "SB_HOST_RGB" in lib.sb_last_error().decode()
    ws = lib.sb_host_workspace_bytes(64, 64, 0, 2)
    p4 = _prm(flags=_lib.SB_HOST_RGB, guide_channels=4)
    st = lib.sb_stylize_batch_host(C.byref(p4), 1, None, FAKE, FAKE, 64, 64, FAKE, FAKE, 64, 64, FAKE, 0, FAKE, ws, 2,
                                   None)
    assert st == _lib.SB_EINVAL and "guide_channels" in lib.sb_last_error().decode()
    st = lib.sb_stylize_batch_host(C.byref(p), 1, None, FAKE, FAKE, 64, 64, FAKE, FAKE, 62, 64, FAKE, 0, FAKE,
                                   lib.sb_host_workspace_bytes(62, 64, 0, 2), 2, None)
    assert st == _lib.SB_EUNSUPPORTED and "wt" in lib.sb_last_error().decode()


def test_host_batch_invalid(lib):
    p = _prm()
    st = lib.sb_stylize_batch_host(C.byref(p), 1, None, FAKE, FAKE, 64, 64, FAKE, FAKE, 64, 64, FAKE, 0, FAKE, 16, 2,
                                   None)
    assert st == _lib.SB_EINVAL and "workspace_bytes" in lib.sb_last_error().decode()
    st = lib.sb_stylize_batch_host(C.byref(p), 1, None, FAKE, FAKE, 64, 64, FAKE, FAKE, 64, 64, FAKE, 0, FAKE, 16, 0,
                                   None)
    assert st == _lib.SB_EINVAL and "depth" in lib.sb_last_error().decode()


def test_binding_refuses_cpu_tensors():
    import torch

    g = torch.zeros(8, 8, 4, dtype=torch.uint8)
    with pytest.raises(ValueError, match="CUDA"):
        sb.build_lut(g)
    with pytest.raises(ValueError, match="CUDA"):
        sb.stylize(sb.Params(10, 3), g, g, torch.zeros(65536, dtype=torch.int32), g)


def test_product_does_not_import_oracle():
    """The product package never imports or links the oracle (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_1807_03249_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                for bad in ("import oracle", "from oracle", "liboracle", "styleblit_oracle", "or_stylize"):
                    assert bad not in txt, (fn, bad)
    for fn in os.listdir(os.path.join(ROOT, "oracle")):
        if fn.endswith((".c", ".h", ".py")):
            txt = open(os.path.join(ROOT, "oracle", fn)).read()
            assert "import paper_1807_03249_b200" not in txt and "styleblit.h\"" not in txt


def test_host_batch_negative_frames_and_exemplar_cap(lib):
    p = _prm()
    st = lib.sb_stylize_batch_host(C.byref(p), -1, None, FAKE, FAKE, 64, 64, FAKE, FAKE, 64, 64, FAKE, 0, FAKE,
                                   lib.sb_host_workspace_bytes(64, 64, 0, 2), 2, None)
    assert st == _lib.SB_EINVAL and "n_frames" in lib.sb_last_error().decode()
    assert lib.sb_exemplar_bytes(512, 512) == 2 * 512 * (1 << 18)
    assert lib.sb_exemplar_bytes(512, 4096) == 2 * 4096 * (1 << 18)
    assert lib.sb_exemplar_bytes(512, 4097) == 0
    st = lib.sb_prepare_exemplar(FAKE, FAKE, 64, 5000, FAKE, None)
    assert st == _lib.SB_EUNSUPPORTED and "SB_EXEMPLAR_MAX_HS" in lib.sb_last_error().decode()


def test_binding_output_and_seed_validation():
    """The binding checks caller-supplied outputs (shape, dtype, device) and frame_seeds
    before any raw pointer reaches the ABI (host-side logic, no GPU needed)."""
    import torch

    t = torch.zeros(2, 8, 8, dtype=torch.int32)
    sb._check_out(t, "coords", (2, 8, 8), torch.int32, "cpu")
    with pytest.raises(ValueError, match="shape"):
        sb._check_out(t, "coords", (2, 8, 9), torch.int32, "cpu")
    with pytest.raises(ValueError, match="shape"):
        sb._check_out(t, "coords", (2, 8, 8), torch.uint8, "cpu")
    with pytest.raises(ValueError, match="on"):
        sb._check_out(t, "coords", (2, 8, 8), torch.int32, "meta")
    assert sb._seeds(None, 3) is None
    assert list(sb._seeds([1, 2, 3], 3)) == [1, 2, 3]
    with pytest.raises(ValueError, match="frame_seeds"):
        sb._seeds([1, 2], 3)
    with pytest.raises(ValueError, match="frame_seeds"):
        sb._seeds([1, 2, 3, 4], 3)
