"""Multi-GPU partitioning of the StyleBlit hot path.

Every pixel of Alg. 2 is independent ("fully parallel ... every target
pixel will be visited only once") and the jitter is a function of global cell coordinates,
level and frame seed, so any partition reproduces the single-GPU result bit for bit.

* Frame mode (the headline, weak scaling): rank k stylizes its own frames; the exemplar and
  LUT are replicated; no data-path collective.
* Strip mode (single-frame latency): each frame is cut into row strips, one per rank.  A rank
  computes its strip through sb_params.row_begin/row_end (the vote's r-row coordinate halo is
  recomputed inside the library, so no halo exchange is needed) and the strips are gathered
  to the consumer rank -- the one real exchange step.  Two ways: `gather_strips` (one NCCL
  gather after the compute), or `peer_output` (the consumer's output buffer is mapped into
  every rank through CUDA IPC and each rank's stylize kernel stores its rows straight into it
  over NVLink / NVSwitch, so the transfer overlaps the compute tile by tile; a one-element
  all-reduce then orders the consumer after every writer).

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
                  row_axis: int = 0):
    """Gather each rank's row strip (rows along `row_axis`, e.g. [h_k, W, 4] or a batch
    [B, h_k, W, 4] with row_axis=1) to rank `dst` in ONE collective.

    Strips are padded to the largest strip height so the collective sees equal shapes, then
    trimmed.  Returns the full frame(s) on dst and None elsewhere.
    """
    hmax = max(e - b for b, e in (strip_rows(ht, world, r) for r in range(world)))
    shape = list(strip.shape)
    shape[row_axis] = hmax
    pad = torch.zeros(shape, dtype=strip.dtype, device=strip.device)
    pad.narrow(row_axis, 0, strip.shape[row_axis]).copy_(strip)
    if rank == dst:
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.gather(pad, gather_list=bufs, dst=dst, group=group)
        shape[row_axis] = ht
        out = torch.empty(shape, dtype=strip.dtype, device=strip.device)
        for r in range(world):
            b, e = strip_rows(ht, world, r)
            out.narrow(row_axis, b, e - b).copy_(bufs[r].narrow(row_axis, 0, e - b))
        return out
    dist.gather(pad, gather_list=None, dst=dst, group=group)
    return None


def _share_cuda_ipc(t: torch.Tensor):
    return t.untyped_storage()._share_cuda_()


def _open_cuda_ipc(handle, shape, dtype):
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
