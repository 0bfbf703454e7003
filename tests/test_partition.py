"""Partitioned box, host side; CPU only.

The sub-box lattices must reproduce the global mesh numbering and
coordinates bit-exactly (the "assembly map" parity: the oracle's restriction
indices, oracle/hexfem_oracle.c after mesh.cpp:80-104), and every global node
must be owned by exactly one rank.  A world_size-2 gloo job checks the same
across processes plus the communicator-id bootstrap the bench uses.
"""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2109_04996_b200 import _core, dist as hdist

CASES = [((4, 3, 2), 2), ((4, 4, 4), 8), ((5, 4, 3), 4), ((6, 2, 3), 6), ((3, 3, 3), 1)]


def _lattice_ids(dims, p):
    NX, NY, NZ = (d * p + 1 for d in dims)
    return NX, NY, NZ


def test_proc_grid():
    assert list(_core.proc_grid(1, (25, 25, 25))) == [1, 1, 1]
    assert list(_core.proc_grid(2, (25, 25, 25))) == [2, 1, 1]
    assert list(_core.proc_grid(4, (25, 25, 25))) == [2, 2, 1]
    assert list(_core.proc_grid(8, (25, 25, 25))) == [2, 2, 2]
    assert list(_core.proc_grid(2, (4, 8, 4))) == [1, 2, 1]  # longest axis first
    with pytest.raises(ValueError):
        _core.subdomain((1, 1, 1), 2, 0)  # fewer elements than ranks on the axis


@pytest.mark.parametrize("dims,nranks", CASES)
@pytest.mark.parametrize("p", [1, 3])
def test_cover_and_ownership(dims, nranks, p):
    NX, NY, NZ = _lattice_ids(dims, p)
    owners = np.zeros(NX * NY * NZ, dtype=np.int64)
    copies = np.zeros(NX * NY * NZ, dtype=np.int64)
    elems = 0
    for r in range(nranks):
        s = _core.subdomain(dims, nranks, r)
        ids = _core.global_node_ids(s, p)
        own = _core.owned_nodes(s, p)
        np.add.at(copies, ids, 1)
        np.add.at(owners, ids[own], 1)
        elems += int(np.prod(s.dims))
        # neighbours are symmetric
        for a in range(3):
            lo, hi = s.neighbor[a]
            if lo >= 0:
                assert _core.subdomain(dims, nranks, lo).neighbor[a][1] == r
            if hi >= 0:
                assert _core.subdomain(dims, nranks, hi).neighbor[a][0] == r
    assert elems == int(np.prod(dims))
    assert copies.min() >= 1
    assert np.all(owners == 1)


@pytest.mark.parametrize("dims,nranks", CASES[:3])
@pytest.mark.parametrize("deform", ["none", "sine"])
def test_assembly_map_bit_exact(dims, nranks, deform):
    """Local restriction -> global ids == the oracle's global indices, and
    sub-box coordinates == global coordinates, bit for bit."""
    p = 3
    g = oracle.setup("bp3", p, dims, deform)
    gidx = g.indices.reshape(g.num_elements, -1)
    gcoords = g.coords.reshape(3, -1)
    n1 = p + 1
    k = np.arange(n1)
    kx, ky, kz = (k[None, None, :], k[None, :, None], k[:, None, None])
    for r in range(nranks):
        s = _core.subdomain(dims, nranks, r)
        ids = _core.global_node_ids(s, p)
        NX, NY, _ = _lattice_ids(s.dims, p)
        lc = np.asarray(_core.submesh_coords(s, p, deform)).reshape(3, -1)
        assert np.array_equal(lc, gcoords[:, ids])
        for ez in range(s.dims[2]):
            for ey in range(s.dims[1]):
                for ex in range(s.dims[0]):
                    local = ((ex * p + kx) + NX * ((ey * p + ky) + NY * (ez * p + kz))).ravel()
                    ge = ((s.offset[0] + ex) + dims[0] * ((s.offset[1] + ey)
                                                         + dims[1] * (s.offset[2] + ez)))
                    assert np.array_equal(ids[local], gidx[ge])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, dims, p, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        uid = hdist.broadcast_unique_id(make_id=lambda: bytes(range(128)))
        s = _core.subdomain(dims, world, rank)
        ids = torch.from_numpy(_core.global_node_ids(s, p))
        own = torch.from_numpy(_core.owned_nodes(s, p).astype(np.int64))
        n = torch.tensor([ids.numel()])
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, n)
        mx = int(max(t.item() for t in sizes))
        pad = lambda t: torch.cat([t, torch.full((mx - t.numel(),), -1, dtype=torch.int64)])
        all_ids = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
        all_own = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(all_ids, pad(ids))
        dist.all_gather(all_own, pad(own))
        if rank == 0:
            NX, NY, NZ = _lattice_ids(dims, p)
            count = np.zeros(NX * NY * NZ, dtype=np.int64)
            for i, o in zip(all_ids, all_own):
                i, o = i.numpy(), o.numpy()
                keep = (i >= 0) & (o == 1)
                np.add.at(count, i[keep], 1)
            q.put((uid == bytes(range(128)), bool(np.all(count == 1))))
        else:
            q.put((uid == bytes(range(128)), True))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partition():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, (4, 3, 2), 3, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(a and b for a, b in res)
