"""Multi-rank host logic on CPU (gloo, world_size 2 and 4).

The GPU data path of a partitioned solve is covered on one device by
tests/test_gpu_slabs.py (same kernels, ghost layers and reductions; device
copies instead of NCCL). Here real processes check what the NCCL transport
relies on: the partition every rank computes independently is one consistent
cover of the grid, the library's own halo plan (tmg_halo_plan: the operations
exchange() issues as ncclSend / ncclRecv) pairs every send with the matching receive
and delivers exactly the neighbour's boundary layer, the NCCL id reaches all
ranks, and the slabs of a global array reassemble it.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_06850_b200 import GridSpec
from paper_2410_06850_b200 import dist as D

GRID = GridSpec(64, 64, 64)
NCC, SD = 4, 2  # 4 cc layers of 16 cells; coarse cells of 8^3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out, shape=(64, 64, 64), ncc=(NCC,) * 3, sd=SD):
    GRID = GridSpec(*shape)
    NCC3 = tuple(ncc)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        part = D.partition(GRID, NCC3, sd, world, rank)
        parts = [None] * world
        dist.all_gather_object(parts, part)
        # one consistent cover of z, bricks, cc elements and cells
        assert parts[0]["z0"] == 0 and parts[-1]["z1"] == GRID.nz
        for a, b in zip(parts, parts[1:]):
            assert a["z1"] == b["z0"]
            assert a["brick0"] + a["bricks"] == b["brick0"]
            assert a["elem0"] + a["elems"] == b["elem0"]
            assert a["cell0"] + a["cells"] == b["cell0"]
        assert sum(p["cells"] for p in parts) == GRID.num_cells()
        assert [p["lo"] for p in parts] == [0] + [1] * (world - 1)
        assert [p["hi"] for p in parts] == [1] * (world - 1) + [0]
        # halo exchange following the library's plan: bricks hold their
        # global index; ghosts start at -1 and must end as the neighbour's ids
        L = (NCC3[0] * sd) * (NCC3[1] * sd)  # bricks per z-layer
        Le = NCC3[0] * NCC3[1]  # cc elements per z-layer
        # the library's own plan (tmg_halo_plan = the ops exchange() issues
        # over NCCL), carried out with gloo point-to-point
        for elem, base, count, layer in ((False, part["brick0"], part["bricks"], L),
                                         (True, part["elem0"], part["elems"], Le)):
            lo_u = base - part["lo"] * layer
            n_u = count + (part["lo"] + part["hi"]) * layer
            win = -np.ones(n_u, dtype=np.int64)
            win[base - lo_u:base - lo_u + count] = np.arange(base, base + count)
            plan = D.halo_plan(GRID, NCC3, sd, world, rank, elem=elem)
            assert len(plan) == 2 * (part["lo"] + part["hi"])
            reqs, recv = [], []
            for op, peer, u0, nu in plan:
                assert nu == layer and abs(peer - rank) == 1
                if op == "send":  # own layers only
                    assert base <= u0 and u0 + nu <= base + count
                    reqs.append(dist.isend(torch.from_numpy(win[u0 - lo_u:u0 - lo_u + nu].copy()),
                                           peer))
                else:  # ghost layers only
                    assert u0 + nu <= base or u0 >= base + count
                    buf = torch.empty(nu, dtype=torch.int64)
                    reqs.append(dist.irecv(buf, peer))
                    recv.append((u0, buf))
            for q in reqs:
                q.wait()
            for u0, buf in recv:
                win[u0 - lo_u:u0 - lo_u + len(buf)] = buf.numpy()
            np.testing.assert_array_equal(win, np.arange(lo_u, lo_u + n_u))
        # NCCL unique id hand-off (host-only call)
        nid = D.broadcast_nccl_id(dist)
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        assert len(nid) == 128 and all(i == ids[0] for i in ids)
        # slabs of a global array reassemble it
        g = np.arange(GRID.num_cells(), dtype=np.float64)
        pieces = [None] * world
        dist.all_gather_object(pieces, D.slab(g, part))
        np.testing.assert_array_equal(np.concatenate(pieces), g)
        out[rank] = 1
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_partition_and_halo_plan_gloo(world):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    assert sorted(out.keys()) == list(range(world))


def test_partition_and_halo_plan_gloo_generic_shape():
    """a non-cubic hierarchy (coarse cells of 12 x 8 x 8, generic kernels):
    the slab partition and the halo plan are per brick / cc-element layer,
    whatever the brick shape"""
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(2, _free_port(), out, (48, 32, 64), (2, 2, 4), 2),
                       nprocs=2, join=True, start_method="spawn")
    assert sorted(out.keys()) == [0, 1]


def test_partition_errors():
    from paper_2410_06850_b200 import ConfigError
    with pytest.raises(ConfigError):
        D.partition(GRID, NCC, SD, 3, 0)  # 3 does not divide 4 cc layers
    with pytest.raises(ValueError):
        D.partition(GRID, NCC, SD, 2, 2)  # rank out of range
