"""Device-side tests of the multi-GPU paths of paper_1807_03249_b200/sharding.py on ONE GPU.

The pool gives one GPU per call, so the two paths are exercised the only ways one device allows
(no ranks on one GPU wait on each other's kernels):

* NCCL: a 1-rank NCCL process group on cuda:0 runs the strip-mode step as bench.py does
  (stylize over row_begin/row_end with the vote's coordinate halo, the vote, gather_strips into
  the output rows, the one-element all-reduce that orders the consumer) -- parity against the
  oracle for the full frame.
* CUDA IPC (the fused compute + gather of DESIGN.md section 9): 2 processes share cuda:0.
  Rank 0 owns C_T; rank 1 maps it with peer_output (CUDA IPC handle through a gloo object
  broadcast) and its stylize / vote kernels store their strip rows straight into rank 0's
  buffer; a gloo all-reduce after a device synchronize orders rank 0 after the writer.  Rank 0
  then checks the assembled frame against the oracle, bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_frame(r, frames):
    import oracle
    import synth

    cfg = synth.CONFIGS[1]
    cs, gs = [t.numpy() for t in synth.exemplar(cfg)]
    lut = oracle.build_lut(gs, nthreads=8)
    out = []
    for f, gt in enumerate(frames):
        prm = oracle.Params(t=cfg["t"], L=cfg["L"], C=cfg["C"], seed=(cfg["seed"] + f) & 0xFFFFFFFF)
        ct, coords, _ = oracle.stylize(prm, cs, gs, lut, gt, nthreads=8)
        out.append(oracle.vote(coords, cs, r, nthreads=8) if r > 0 else ct)
    return np.stack(out)


def _frames(H, W, n):
    import synth

    return [synth.heightfield_normals(W, H, seed=1, frame=i).numpy() for i in range(n)]


def _strip_step(sb, prm_kw, cs, gs, lut, gt, ex, ct_out, coords, rb, re_, r, H):
    """One strip-mode step of this rank (bench.py run_ours): coords for the strip plus the
    r-row halo (recomputed, no halo exchange), then the blit or the vote into ct_out rows."""
    prm = sb.Params(**prm_kw, flags=sb.SB_NO_COLOR if r > 0 else 0, row_begin=max(0, rb - r),
                    row_end=min(H, re_ + r), exemplar=ex)
    n = gt.shape[0]
    seeds = [(prm_kw["seed"] + i) & 0xFFFFFFFF for i in range(n)]
    sb.stylize_batch(prm, cs, gs, lut, gt, frame_seeds=seeds, ct=None if r > 0 else ct_out, coords=coords,
                     want_level=False)
    if r > 0:
        sb.vote(coords, cs, r, ct=ct_out, row_begin=rb, row_end=re_, exemplar=ex)


def _setup(dev, H, W, n):
    import paper_1807_03249_b200 as sb
    import synth

    cfg = synth.CONFIGS[1]
    cs, gs = [t.to(dev) for t in synth.exemplar(cfg)]
    gt = torch.from_numpy(np.stack(_frames(H, W, n))).to(dev)
    lut = sb.build_lut(gs)
    ex = sb.prepare_exemplar(cs, gs)
    prm_kw = dict(threshold=cfg["t"], levels=cfg["L"], guide_channels=cfg["C"], seed=cfg["seed"])
    return sb, cfg, cs, gs, gt, lut, ex, prm_kw


def _nccl_worker(port, q):
    import torch.distributed as dist

    from paper_1807_03249_b200 import sharding

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dev = torch.device("cuda:0")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        H, W, n = 70, 100, 3
        sb, cfg, cs, gs, gt, lut, ex, prm_kw = _setup(dev, H, W, n)
        ok = True
        for r in (0, 2):
            ct = torch.zeros(n, H, W, 4, dtype=torch.uint8, device=dev)
            coords = torch.empty(n, H, W, dtype=torch.int32, device=dev)
            rb, re_ = sharding.strip_rows(H, 1, 0)
            _strip_step(sb, prm_kw, cs, gs, lut, gt, ex, ct, coords, rb, re_, r, H)
            got = sharding.gather_strips(ct[:, rb:re_], H, 1, 0, dst=0, row_axis=1, out=ct)
            flag = torch.zeros(1, dtype=torch.int32, device=dev)
            dist.all_reduce(flag)
            torch.cuda.synchronize()
            ok &= got is ct and bool(np.array_equal(ct.cpu().numpy(), _oracle_frame(r, gt.cpu().numpy())))
        dist.destroy_process_group()
        q.put(("ok", bool(ok)))
    except Exception as e:  # report, do not hang the parent
        q.put(("err", repr(e)))


def _ipc_worker(rank, world, port, r, q):
    import torch.distributed as dist

    from paper_1807_03249_b200 import sharding

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        dev = torch.device("cuda:0")
        H, W, n = 75, 132, 2  # ragged strips (75 rows over 2 ranks), a width not divisible by 128
        sb, cfg, cs, gs, gt, lut, ex, prm_kw = _setup(dev, H, W, n)
        ct = torch.zeros(n, H, W, 4, dtype=torch.uint8, device=dev) if rank == 0 else None
        ct_out = sharding.peer_output(ct, (n, H, W, 4), torch.uint8, rank)
        if rank != 0:
            assert ct_out.data_ptr() != 0 and tuple(ct_out.shape) == (n, H, W, 4)
        coords = torch.empty(n, H, W, dtype=torch.int32, device=dev)
        rb, re_ = sharding.strip_rows(H, world, rank)
        _strip_step(sb, prm_kw, cs, gs, lut, gt, ex, ct_out, coords, rb, re_, r, H)
        torch.cuda.synchronize()  # this rank's stores into rank 0's buffer are complete ...
        dist.all_reduce(torch.zeros(1))  # ... before rank 0 reads it
        ok = True
        if rank == 0:
            ok = bool(np.array_equal(ct.cpu().numpy(), _oracle_frame(r, gt.cpu().numpy())))
        dist.barrier()  # rank 1 keeps its mapping open until rank 0 has read the frame
        del ct_out
        dist.destroy_process_group()
        q.put(("ok", ok))
    except Exception as e:
        q.put(("err", repr(e)))


def _run(target, args_of, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=args_of(k, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    res = [q.get(timeout=30) for _ in range(world)]
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert all(kind == "ok" and v for kind, v in res), res


def test_nccl_one_rank_strip_step():
    _run(_nccl_worker, lambda k, port, q: (port, q), 1)


@pytest.mark.parametrize("r", [0, 2])
def test_ipc_two_processes_store_into_rank0(r):
    _run(_ipc_worker, lambda k, port, q: (k, 2, port, r, q), 2)
