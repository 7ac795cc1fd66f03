"""The checked build (libstyleblit_checked.so: the product sources compiled with -DSB_CHECKED,
device bounds checks on every shared-memory slot and global gather/store index) -- the stand-in
for compute-sanitizer memcheck, which this GPU pool does not allow
(profiles/r02_sanitizer_unavailable.txt).

* The parity cases of the product (configs 1-4, voting radii 1..8, ragged widths, strips, deep
  hierarchies, wide images) run against the checked build in a subprocess: no check fires and
  every result still equals the oracle.
* A deliberately corrupted LUT (entries outside the exemplar) makes the checked build trap with
  an SB_CHECK message -- the checks are live.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1807_03249_b200", "libstyleblit_checked.so")


def _env():
    if not os.path.exists(CHECKED):
        from paper_1807_03249_b200 import _build

        _build.build(checked=True)
    return dict(os.environ, SB_LIBRARY=CHECKED)


def test_parity_suite_under_checked_build():
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_parity_gpu.py",
                        "tests/test_limits_gpu.py", "tests/test_lut3_gpu.py", "tests/test_sharding_gpu.py"],
                       cwd=ROOT, env=_env(), capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "SB_CHECK" not in r.stdout + r.stderr


BAD_LUT = r'''
import sys
import torch
sys.path.insert(0, ".")
import paper_1807_03249_b200 as sb
import synth
cfg, cs, gs, gt = synth.config(1)
cs, gs, gt = cs.cuda(), gs.cuda(), gt.cuda()
lut = torch.full((65536,), (30000 << 16) | 30000, dtype=torch.int32, device="cuda")  # outside the 64x64 exemplar
prm = sb.Params(threshold=0.0, levels=3, guide_channels=3)  # t = 0: every pixel takes the look-up
sb.stylize(prm, cs, gs, lut, gt)
torch.cuda.synchronize()
print("no trap")
'''


def test_checked_build_traps_on_a_bad_lut():
    r = subprocess.run([sys.executable, "-c", BAD_LUT], cwd=ROOT, env=_env(), capture_output=True, text=True,
                       timeout=300)
    out = r.stdout + r.stderr
    assert r.returncode != 0 and "SB_CHECK(final coordinate) failed" in out, out[-3000:]
