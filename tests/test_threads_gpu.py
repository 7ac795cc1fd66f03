"""Concurrent use of the ABI from several host threads (the library holds no
state beyond per-device caches and per-thread host-pipeline streams).  ctypes releases the GIL
during each call, so the C entry points really run concurrently: 4 threads, each on its own
CUDA stream, run different workloads (L, r, strided copy or not, ragged width) several times
over, and 2 threads drive the host pipeline at once; every result must equal the serial one
bit for bit."""
import threading

import numpy as np
import pytest
import torch

import paper_1807_03249_b200 as sb
import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")

CASES = [dict(L=5, r=0, ex=True, w=384), dict(L=4, r=2, ex=False, w=256), dict(L=3, r=3, ex=True, w=131),
         dict(L=5, r=8, ex=False, w=200)]


def _inputs():
    cfg = synth.CONFIGS[1]
    cs, gs = [t.to(DEV) for t in synth.exemplar(cfg)]
    lut = sb.build_lut(gs)
    ex = sb.prepare_exemplar(cs, gs)
    torch.cuda.synchronize()
    return cfg, cs, gs, lut, ex


def _run(case, cfg, cs, gs, lut, ex):
    gt = torch.stack([synth.heightfield_normals(case["w"], 72, seed=2, frame=i) for i in range(3)]).to(DEV)
    prm = sb.Params(threshold=cfg["t"], levels=case["L"], blend_radius=case["r"], guide_channels=3, seed=9,
                    exemplar=ex if case["ex"] else None)
    ct, co, lv = sb.stylize_batch(prm, cs, gs, lut, gt)
    torch.cuda.current_stream().synchronize()
    return ct.cpu(), co.cpu(), lv.cpu()


def test_threads_device_calls():
    cfg, cs, gs, lut, ex = _inputs()
    serial = [_run(c, cfg, cs, gs, lut, ex) for c in CASES]
    errors, results = [], {}

    def worker(k):
        try:
            s = torch.cuda.Stream(device=DEV)
            with torch.cuda.stream(s):
                for it in range(4):
                    results[(k, it)] = _run(CASES[k], cfg, cs, gs, lut, ex)
        except Exception as e:  # surfaced below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(k,)) for k in range(len(CASES))]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
    assert not errors, errors
    for (k, it), got in results.items():
        for a, b in zip(got, serial[k]):
            assert torch.equal(a, b), (k, it)
    assert len(results) == 4 * len(CASES)


def test_threads_host_pipeline():
    cfg, cs, gs, lut, ex = _inputs()
    gts = [torch.stack([synth.heightfield_normals(256, 64, seed=3 + k, frame=i) for i in range(5)]).pin_memory()
           for k in range(2)]
    prm = sb.Params(threshold=cfg["t"], levels=5, guide_channels=3, seed=4, exemplar=ex)

    def host(k):
        ct = torch.empty_like(gts[k]).pin_memory()
        sb.stylize_batch_host(prm, cs, gs, lut, gts[k], ct)
        return ct

    serial = [host(k).clone() for k in range(2)]
    out, errors = {}, []

    def worker(k):
        try:
            for it in range(3):
                out[(k, it)] = host(k).clone()
        except Exception as e:
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
    assert not errors, errors
    assert len(out) == 6
    for (k, it), ct in out.items():
        assert torch.equal(ct, serial[k]), (k, it)
    # and the device batch agrees with the host pipeline
    d = sb.stylize_batch(prm, cs, gs, lut, gts[0].to(DEV))[0].cpu()
    assert torch.equal(d, serial[0])
