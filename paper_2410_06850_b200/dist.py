"""Host side of the partitioned (multi-GPU) solve.

One process per GPU. The grid is split along z into slabs of whole
cc-element layers (tmg_partition); rank r owns bricks [brick0, brick0 +
bricks) and keeps one ghost brick layer per neighbouring rank. The CUDA
library moves the data (NCCL send/recv of whole brick layers, all-reduce of
the CG dot products, all-gather of the coarse-coarse right-hand side); this
module holds what the host needs around it: the slab of a global array, the
NCCL id hand-off over torch.distributed, and the halo plan the library
follows, written out as data so it can be checked on CPU with gloo
(tests/test_dist_cpu.py).
"""
from __future__ import annotations

import numpy as np

from .solver import Context, GridSpec, nccl_unique_id, partition


def slab(values: np.ndarray, part: dict) -> np.ndarray:
    """The rank's cells of a global x-fastest array (z-slowest, contiguous)."""
    return np.ascontiguousarray(values[part["cell0"]:part["cell0"] + part["cells"]])


def halo_plan(part: dict, rank: int, layer: int) -> list[tuple[int, tuple, tuple]]:
    """(peer, (send start, stop), (recv start, stop)) in global brick (or cc
    element) units for one ghost exchange; `layer` units per z-layer. Mirrors
    exchange() in csrc/abi.cu: the own bottom layer goes to rank - 1 and its
    top layer comes back as the lower ghost; symmetrically above."""
    u0, nu = part["brick0"], part["bricks"]
    plan = []
    if part["lo"]:
        plan.append((rank - 1, (u0, u0 + layer), (u0 - layer, u0)))
    if part["hi"]:
        plan.append((rank + 1, (u0 + nu - layer, u0 + nu), (u0 + nu, u0 + nu + layer)))
    return plan


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
