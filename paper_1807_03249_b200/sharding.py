"""Multi-GPU partitioning of the StyleBlit hot path.

Every pixel of Alg. 2 is independent ("fully parallel ... every target
pixel will be visited only once") and the jitter is a function of global cell coordinates,
level and frame seed, so any partition reproduces the single-GPU result bit for bit.

* Frame mode (the headline, weak scaling): rank k stylizes its own frames; the exemplar and
  LUT are replicated; no data-path collective.
* Strip mode (single-frame latency): each frame is cut into row strips, one per rank.  A rank
  computes its strip through sb_params.row_begin/row_end (the vote's r-row coordinate halo is
  recomputed inside the library, so no halo exchange is needed) and the strips are gathered
  to the consumer rank -- the one real exchange step.  Two ways: `gather_strips` (grouped
  NCCL send/recv after the compute, received straight into the consumer's output rows), or
  `peer_output` (the consumer's output buffer is mapped into every rank through CUDA IPC and
  each rank's stylize kernel stores its rows straight into it over NVLink / NVSwitch, so the
  transfer overlaps the compute tile by tile; a one-element all-reduce then orders the
  consumer after every writer).

The functions take a torch.distributed process group and work with any backend (NCCL for
CUDA tensors, gloo for the CPU tests in tests/test_sharding_gloo.py).  Compute is passed in
as a callable so this module holds no part of the method's arithmetic.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def strip_rows(ht: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [begin, end) of rank's strip: contiguous, balanced to within one row."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(ht, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def frame_range(n_frames: int, world: int, rank: int) -> tuple[int, int]:
    """Frames [begin, end) of rank in frame mode (contiguous, balanced)."""
    return strip_rows(n_frames, world, rank)


def gather_strips(strip: torch.Tensor, ht: int, world: int, rank: int, dst: int = 0, group=None,
                  row_axis: int = 0, out: torch.Tensor | None = None):
    """Gather each rank's row strip to rank `dst` with grouped point-to-point transfers.

    `strip` holds this rank's rows along `row_axis` (e.g. [h_k, W, 4], or a batch
    [B, h_k, W, 4] with row_axis=1), each leading-index slice contiguous.  On dst, `out` (the
    full frame(s); allocated when None) receives every other rank's strip straight into its own
    rows -- one recv per rank and leading index, all in one group (one NCCL group call), no
    padding, no receive buffers, no reassembly copy; dst's own strip is copied only when it is
    not already a view of `out` (the bench computes it in place).  Returns `out` on dst, None
    elsewhere.
    """
    lead = tuple(strip.shape[:row_axis])
    n_lead = 1
    for v in lead:
        n_lead *= v
    rest = tuple(strip.shape[row_axis + 1:])

    def rows(t: torch.Tensor, i: int) -> torch.Tensor:
        """Leading index i (flattened) of t, rows along dimension 0 of the result."""
        return t.reshape(n_lead, *t.shape[row_axis:])[i]

    b_me, e_me = strip_rows(ht, world, rank)
    if strip.shape[row_axis] != e_me - b_me:
        raise ValueError(f"rank {rank} strip has {strip.shape[row_axis]} rows, expected {e_me - b_me}")
    ops = []
    if rank == dst:
        if out is None:
            out = torch.empty(*lead, ht, *rest, dtype=strip.dtype, device=strip.device)
        mine = out.narrow(row_axis, b_me, e_me - b_me)
        if mine.data_ptr() != strip.data_ptr():
            mine.copy_(strip)
        for r in range(world):
            if r == dst:
                continue
            b, e = strip_rows(ht, world, r)
            if e == b:
                continue
            for i in range(n_lead):
                ops.append(dist.P2POp(dist.irecv, rows(out, i).narrow(0, b, e - b), r, group))
    elif e_me > b_me:
        for i in range(n_lead):
            t = rows(strip, i)
            if not t.is_contiguous():
                t = t.contiguous()
            ops.append(dist.P2POp(dist.isend, t, dst, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return out if rank == dst else None


def _share_cuda_ipc(t: torch.Tensor):
    return t.untyped_storage()._share_cuda_()


def _open_cuda_ipc(handle, shape, dtype):
    # handle[0] is the owner's device index.  Same device: no peer access needed.  Another
    # device: torch opens the handle with cudaIpcMemLazyEnablePeerAccess, which enables peer
    # access from the current device; refuse up front where the hardware cannot do it.
    here = torch.cuda.current_device()
    owner = int(handle[0])
    if owner != here and not torch.cuda.can_device_access_peer(here, owner):
        raise RuntimeError(f"cuda:{here} cannot access cuda:{owner} as a peer: use the NCCL gather")
    storage = torch.UntypedStorage._new_shared_cuda(*handle)
    out = torch.empty(0, dtype=dtype, device=storage.device)
    strides, acc = [], 1
    for n in reversed(shape):
        strides.insert(0, acc)
        acc *= n
    out.set_(storage, 0, tuple(shape), tuple(strides))
    return out


def peer_output(local: torch.Tensor | None, shape, dtype, rank: int, src: int = 0, group=None,
                share: Callable | None = None, open_: Callable | None = None):
    """Rank src's output tensor, mapped into every rank: on src `local` itself, elsewhere a
    tensor over the same device memory (CUDA IPC), whose pointer a kernel on this rank's GPU
    stores to over NVLink / NVSwitch peer access.  The handle travels with one object
    broadcast.  `share` / `open_` default to CUDA IPC; tests pass stand-ins."""
    share = share or _share_cuda_ipc
    open_ = open_ or _open_cuda_ipc
    obj = [share(local) if rank == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    if rank == src:
        return local
    return open_(obj[0], shape, dtype)


def stylize_strip_mode(compute: Callable[[int, int], torch.Tensor], ht: int, world: int, rank: int, dst: int = 0,
                       group=None):
    """Strip-mode frame: `compute(row_begin, row_end)` returns this rank's C_T strip
    [row_end - row_begin, W, 4] (on GPUs: sb_stylize with row_begin/row_end); the strips are
    gathered to dst.  Returns the full frame on dst, None elsewhere."""
    b, e = strip_rows(ht, world, rank)
    return gather_strips(compute(b, e), ht, world, rank, dst=dst, group=group)
