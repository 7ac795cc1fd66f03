"""Build libstyleblit.so in-tree with nvcc for sm_100a (called by __graft_entry__.build())."""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libstyleblit.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps() -> list[str]:
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "styleblit.h")]


SO_CHECKED = os.path.join(HERE, "libstyleblit_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """nvcc -> libstyleblit.so.  checked=True: libstyleblit_checked.so with -DSB_CHECKED (device
    bounds checks on every shared-memory slot and global gather/store index, sb_device.cuh),
    the stand-in for compute-sanitizer memcheck, which this GPU pool does not allow; select it
    with SB_LIBRARY=.../libstyleblit_checked.so."""
    so = SO_CHECKED if checked else SO
    if not force and os.path.exists(so) and os.path.getmtime(so) >= max(os.path.getmtime(d) for d in deps()):
        return so
    # one nvcc per source file in parallel (the translation units are independent), then one link
    extra = ["-DSB_CHECKED"] if checked else []
    work = tempfile.mkdtemp(prefix="sb_build_")
    srcs = sources()
    objs = [os.path.join(work, os.path.basename(c) + ".o") for c in srcs]

    def compile_one(i):
        cmd = [NVCC, *NVCC_FLAGS, *extra, "-c", "-o", objs[i], srcs[i]]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    try:
        with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 1)) as ex:
            results = list(ex.map(compile_one, range(len(srcs))))
        tmp = so + f".tmp{os.getpid()}"
        link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
        rl = subprocess.run(link, capture_output=True, text=True) if all(r.returncode == 0 for _, r in results) else None
        log = os.path.join(HERE, "build_checked.log" if checked else "build.log")
        with open(log, "w") as f:
            for cmd, r in results:
                f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if rl is not None:
                f.write(" ".join(link) + "\n" + rl.stdout + rl.stderr)
        for cmd, r in results:
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed ({r.returncode}) on {cmd[-1]}:\n{r.stderr[-4000:]}")
        if rl.returncode != 0:
            raise RuntimeError(f"nvcc link failed ({rl.returncode}):\n{rl.stderr[-4000:]}")
        if verbose:
            print("".join(r.stderr for _, r in results))
        os.replace(tmp, so)
    finally:
        shutil.rmtree(work, ignore_errors=True)
    return so


if __name__ == "__main__":
    import sys

    print(build(force=True, verbose=True, checked="--checked" in sys.argv))
