"""Host side of the partitioned (multi-GPU) solve.

One process per GPU. The grid is split along z into slabs of whole
cc-element layers (tmg_partition); rank r owns bricks [brick0, brick0 +
bricks) and keeps one ghost brick layer per neighbouring rank. The CUDA
library moves the data (NCCL send/recv of whole brick layers, all-reduce of
the CG dot products, all-gather of the coarse-coarse right-hand side); this
module holds what the host needs around it: the slab of a global array, the
NCCL id hand-off over torch.distributed, and the library's own halo plan
(tmg_halo_plan, the operations exchange() issues) so the multi-process logic
can be checked on CPU with gloo (tests/test_dist_cpu.py).
"""
from __future__ import annotations

import numpy as np

from .solver import Context, GridSpec, nccl_unique_id, partition


def slab(values: np.ndarray, part: dict) -> np.ndarray:
    """The rank's cells of a global x-fastest array (z-slowest, contiguous)."""
    return np.ascontiguousarray(values[part["cell0"]:part["cell0"] + part["cells"]])


def halo_plan(grid: GridSpec, ncc, sd: int, nranks: int, rank: int,
              elem: bool = False) -> list[tuple[str, int, int, int]]:
    """The library's own halo exchange of slab `rank` (tmg_halo_plan: the
    operations exchange() in csrc/abi.cu issues as ncclSend / ncclRecv):
    [("send" | "recv", peer, first global unit, units)], units = bricks or
    cc elements (elem)."""
    import ctypes as C
    from .solver import _Grid, _raise, native
    L = native()
    ncc3 = (ncc,) * 3 if np.isscalar(ncc) else tuple(ncc)
    g = _Grid(grid.nx, grid.ny, grid.nz, grid.lx, grid.ly, grid.lz, (C.c_int64 * 3)(*ncc3), sd)
    ops = (C.c_int64 * 16)()
    n = L.tmg_halo_plan(C.byref(g), C.c_int(nranks), C.c_int(rank), C.c_int(int(elem)), ops,
                        C.c_int(4))
    if n < 0:
        _raise(-n, L.tmg_last_error(None).decode())
    return [("send" if ops[4 * i] else "recv", int(ops[4 * i + 1]), int(ops[4 * i + 2]),
             int(ops[4 * i + 3])) for i in range(n)]


def broadcast_nccl_id(torch_dist) -> bytes:
    """Rank 0 makes the NCCL unique id; every rank returns the same bytes."""
    obj = [nccl_unique_id() if torch_dist.get_rank() == 0 else None]
    torch_dist.broadcast_object_list(obj, src=0)
    return obj[0]


def dist_context(grid: GridSpec, ncc, sd: int, torch_dist, device: int) -> Context:
    """This rank's slab context (collective: every rank must call it)."""
    rank, world = torch_dist.get_rank(), torch_dist.get_world_size()
    nid = broadcast_nccl_id(torch_dist)
    return Context(grid, ncc, sd, device=device, rank=rank, nranks=world, nccl_id=nid)


__all__ = ["slab", "halo_plan", "broadcast_nccl_id", "dist_context", "partition"]
