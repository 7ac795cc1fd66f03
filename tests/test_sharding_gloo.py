"""Multi-process (world_size 2, gloo, CPU) tests of the sharding host logic.

The per-strip compute here is the CPU oracle evaluated on the strip's rows only (plus the
vote's coordinate halo), standing in for sb_stylize with row_begin/row_end on a GPU; the
partition and the gather are the product's own code (paper_1807_03249_b200/sharding.py).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1807_03249_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_strip_rows_partition():
    for ht in (1, 2, 7, 64, 2160):
        for world in (1, 2, 3, 4, 8):
            rows = [sharding.strip_rows(ht, world, r) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == ht
            for (b0, e0), (b1, e1) in zip(rows, rows[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in rows]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        sharding.strip_rows(10, 2, 2)


def _strip_compute(prm, cs, gs, lut, gt, r, b, e):
    """Oracle on rows [b, e) only: coords for [b-r, e+r) then the vote for [b, e)."""
    ht, wt = gt.shape[:2]
    cb, ce = max(0, b - r), min(ht, e + r)
    coords = np.zeros((ht, wt), np.uint32)
    for py in range(cb, ce):
        for px in range(wt):
            coords[py, px] = oracle.stylize_pixel(prm, gs, lut, gt, px, py)[0]
    ct = oracle.vote(coords, cs, r) if r > 0 else cs[coords >> 16, coords & 0xFFFF]
    return torch.from_numpy(np.ascontiguousarray(ct[b:e]))


def _worker(rank, world, port, r, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.CONFIGS[1]
        cs, gs = [t.numpy() for t in synth.exemplar(cfg)]
        gt = synth.heightfield_normals(40, 37, seed=1).numpy()
        lut = oracle.build_lut(gs)
        prm = oracle.Params(t=cfg["t"], L=3, C=3, seed=cfg["seed"])
        full = sharding.stylize_strip_mode(lambda b, e: _strip_compute(prm, cs, gs, lut, gt, r, b, e),
                                           gt.shape[0], world, rank, dst=0)
        if rank == 0:
            _, coords, _ = oracle.stylize(prm, cs, gs, lut, gt)
            want = oracle.vote(coords, cs, r) if r > 0 else cs[coords >> 16, coords & 0xFFFF]
            q.put(bool((full.numpy() == want).all()))
        else:
            q.put(full is None)
        # frame mode: every frame owned by exactly one rank
        owned = torch.zeros(11, dtype=torch.int64)
        b, e = sharding.frame_range(11, world, rank)
        owned[b:e] = 1
        dist.all_reduce(owned)
        q.put(bool((owned == 1).all()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("r", [0, 2])
def test_strip_mode_gather_world2(r):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, r, q)) for k in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    results = [q.get(timeout=10) for _ in range(2 * world)]
    assert all(results), results


def _peer_worker(rank, world, port, path, q):
    """Strip mode with the consumer's buffer mapped into every rank (sharding.peer_output):
    each rank writes only its own rows straight into rank 0's buffer, a barrier orders rank 0
    after the writers.  CUDA IPC is replaced by a file mapping (the same host logic)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.CONFIGS[1]
        cs, gs = [t.numpy() for t in synth.exemplar(cfg)]
        gt = synth.heightfield_normals(40, 37, seed=2).numpy()
        lut = oracle.build_lut(gs)
        prm = oracle.Params(t=cfg["t"], L=3, C=3, seed=cfg["seed"])
        shape = (37, 40, 4)
        local = None
        if rank == 0:
            local = torch.from_numpy(np.memmap(path, dtype=np.uint8, mode="w+", shape=shape))
            local.fill_(0)
        share = lambda t: path  # noqa: E731
        open_ = lambda h, shp, dt: torch.from_numpy(np.memmap(h, dtype=np.uint8, mode="r+", shape=shp))  # noqa: E731
        out = sharding.peer_output(local, shape, torch.uint8, rank, share=share, open_=open_)
        b, e = sharding.strip_rows(shape[0], world, rank)
        out[b:e] = _strip_compute(prm, cs, gs, lut, gt, 0, b, e)  # the "kernel" stores its rows
        dist.barrier()  # stands in for the stream-ordered all-reduce after the writers' kernels
        if rank == 0:
            _, coords, _ = oracle.stylize(prm, cs, gs, lut, gt)
            q.put(bool((out.numpy() == cs[coords >> 16, coords & 0xFFFF]).all()))
        else:
            q.put(True)
    finally:
        dist.destroy_process_group()


def test_strip_mode_peer_output_world2(tmp_path):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    path = str(tmp_path / "ct.bin")
    procs = [ctx.Process(target=_peer_worker, args=(k, world, port, path, q)) for k in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    results = [q.get(timeout=10) for _ in range(world)]
    assert all(results), results


def _gather_worker(rank, world, port, q):
    """gather_strips on a batch [B, H, W, 4] (row_axis=1) with uneven strips and an empty
    strip (H < world): rank 0 receives straight into its output rows; its own strip is
    computed in place (a view of the output, so no copy)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ok = True
        for B, H, W in ((3, 37, 5), (2, 2, 4)):
            full = torch.arange(B * H * W * 4, dtype=torch.int32).reshape(B, H, W, 4) % 251
            full = full.to(torch.uint8)
            b, e = sharding.strip_rows(H, world, rank)
            if rank == 0:
                out = torch.zeros_like(full)
                out[:, b:e] = full[:, b:e]  # "computed in place"
                got = sharding.gather_strips(out[:, b:e], H, world, rank, dst=0, row_axis=1, out=out)
                ok &= got is out and torch.equal(out, full)
            else:
                ok &= sharding.gather_strips(full[:, b:e].clone(), H, world, rank, dst=0, row_axis=1) is None
        q.put(bool(ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_strips_into_output_rows(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    results = [q.get(timeout=10) for _ in range(world)]
    assert all(results), results
