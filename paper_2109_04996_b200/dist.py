"""Multi-GPU plumbing for the partitioned box.

One process per GPU under torchrun.  torch.distributed is only the
bootstrap: rank 0 makes the hxf (NCCL) communicator id and broadcasts it;
from then on the solver's interface sum-exchange and dot all-reduces run
inside the hxf library on the solve stream (dist.cu), captured into the same
CUDA graph as the operator and vector kernels.
"""
from __future__ import annotations

import os

from . import _core

COMM_ID_BYTES = 128


def env_rank_world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def broadcast_unique_id(make_id=None) -> bytes:
    """Rank 0 makes a communicator id (default: hxf/NCCL), every rank gets it
    over the already-initialised torch.distributed process group."""
    import torch.distributed as dist

    make_id = make_id or _core.Communicator.unique_id
    obj = [make_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != COMM_ID_BYTES:
        raise RuntimeError("hxf: malformed communicator id from rank 0")
    return bytes(uid)


def nccl_communicator(device: int) -> "_core.Communicator":
    """The hxf communicator of this rank (torch.distributed must be initialised)."""
    import torch.distributed as dist

    uid = broadcast_unique_id()
    return _core.Communicator.nccl(device, dist.get_world_size(), dist.get_rank(), uid)


def p2p_capacity(dims_local, p: int, m: int) -> int:
    """Doubles per mailbox slot: the largest interface plane of a sub-box of
    dims_local elements, times the components."""
    nx, ny, nz = (int(d) * p + 1 for d in dims_local)
    return m * max(ny * nz, nx * nz, nx * ny)


def p2p_communicator(device: int, cap: int) -> "_core.Communicator":
    """Peer-to-peer hxf communicator of this rank (one process per GPU,
    torch.distributed initialised): allocate the mailbox, all-gather the CUDA
    IPC handles, open the peers'.  The solver then exchanges planes by direct
    peer stores (NVLink) and reduces dots in peer memory, graph-captured."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    mailbox, handle = _core.Communicator.p2p_alloc(device, world, cap)
    handles = [None] * world
    dist.all_gather_object(handles, bytes(handle))
    return _core.Communicator.p2p(mailbox, world, rank, cap, handles)


def partition_summary(dims, nranks: int, p: int) -> dict:
    """Process grid, per-rank sub-box sizes and the largest interface plane."""
    subs = [_core.subdomain(tuple(dims), nranks, r) for r in range(nranks)]
    n_local = [int((s.dims[0] * p + 1) * (s.dims[1] * p + 1) * (s.dims[2] * p + 1)) for s in subs]
    return {"grid": list(subs[0].grid), "sub_dims": [list(s.dims) for s in subs],
            "max_local_nodes": max(n_local)}
