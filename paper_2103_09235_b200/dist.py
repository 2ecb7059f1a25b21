"""torch.distributed plumbing for the slab-decomposed run (one process per GPU).

Only bootstrap and host-side bookkeeping live here: the NCCL unique id is
broadcast through the default process group (gloo or nccl), and the slab
arithmetic mirrors stencil_plan_layout_dist.  The halo exchange itself runs
inside the library (ncclSend/ncclRecv on its comm stream, or the fused
peer stores of the sweep kernel with make_peer_comm).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .api import Comm


def make_comm(device=None) -> Comm:
    """Create the library's NCCL communicator over the current process group."""
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = Comm.unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    if dist.get_backend() == "nccl":
        t = t.to(device or torch.device("cuda", torch.cuda.current_device()))
    dist.broadcast(t, src=0)
    return Comm(bytes(t.cpu().tolist()), rank, world)


def all_gather_bytes(blob: bytes, device=None):
    """Every rank's `blob` (equal lengths) in rank order, over the default group."""
    t = torch.tensor(list(blob), dtype=torch.uint8)
    if dist.get_backend() == "nccl":
        t = t.to(device or torch.device("cuda", torch.cuda.current_device()))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [bytes(o.cpu().tolist()) for o in out]


def make_peer_comm(buf0, buf1, device=None) -> Comm:
    """The fused peer-store exchange (NEXT-2) over the current process group:
    CUDA IPC handles of every rank's two ping-pong buffers and flag words are
    all-gathered, and each rank maps its neighbours' (rank +- 1)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    comm = Comm.peer(rank, world, buf0, buf1)
    comm.attach(all_gather_bytes(comm.handles(), device))
    return comm


def slab(n0: int, rank: int, world: int):
    """Interior planes [lo, hi) of axis 0 owned by `rank` (balanced split)."""
    if n0 % world:
        raise ValueError("axis-0 extent %d not divisible by %d ranks" % (n0, world))
    per = n0 // world
    return rank * per, (rank + 1) * per


def exchange_plan(n0_local: int, rank: int, world: int, hx: int):
    """The per-sweep halo exchange of rank `rank` as (peer, send [lo,hi), recv [lo,hi))
    in local plane coordinates — the same schedule stencil_run_dist issues."""
    ops = []
    if rank > 0:
        ops.append((rank - 1, (0, hx), (-hx, 0)))
    if rank < world - 1:
        ops.append((rank + 1, (n0_local - hx, n0_local), (n0_local, n0_local + hx)))
    return ops
