"""Artifact writers (io.cpp:8-78, io.hpp): legacy-VTK cell scalars and the
trajectory / timings / bench CSVs, byte-identical to the reference's output.
write_vtk_cell_scalars(binary=True) writes the same dataset as big-endian
binary legacy VTK (ASCII at 9 digits is ~1.6 GB per
field at 512^3)."""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

import numpy as np

from .solver import GridSpec


def write_vtk_cell_scalars(grid: GridSpec, field, field_name: str, path: str,
                           binary: bool = False) -> None:
    """write_vtk_cell_scalars (io.cpp:8-34): STRUCTURED_POINTS with point
    dimensions (nx+1, ny+1, nz+1), spacing (hx, hy, hz), CELL_DATA."""
    f = np.ascontiguousarray(field, dtype=np.float64).ravel()
    if f.size != grid.num_cells():
        raise ValueError("write_vtk_cell_scalars: size mismatch")
    head = ("# vtk DataFile Version 3.0\n"
            f"{field_name}\n"
            f"{'BINARY' if binary else 'ASCII'}\n"
            "DATASET STRUCTURED_POINTS\n"
            f"DIMENSIONS {grid.nx + 1} {grid.ny + 1} {grid.nz + 1}\n"
            "ORIGIN 0 0 0\n"
            "SPACING %.9g %.9g %.9g\n" % (grid.lx / grid.nx, grid.ly / grid.ny, grid.lz / grid.nz)
            + f"CELL_DATA {grid.num_cells()}\n"
            f"SCALARS {field_name} double 1\n"
            "LOOKUP_TABLE default\n")
    with open(path, "wb") as out:
        out.write(head.encode())
        if binary:
            out.write(f.astype(">f8").tobytes())
            out.write(b"\n")
        else:
            step = 1 << 20
            for a in range(0, f.size, step):
                out.write("".join("%.9g\n" % v for v in f[a:a + step].tolist()).encode())


def write_trajectory_csv(trajectory: Iterable, path: str) -> None:
    """write_trajectory_csv (io.cpp:36-48)."""
    with open(path, "w") as out:
        out.write("level,iter,cost,volume,ls1_iters,ls2_iters\n")
        for r in trajectory:
            out.write("%d,%d,%.12g,%.12g,%d,%d\n" % (r.level, r.iter, r.cost, r.volume,
                                                      r.ls1_iters, r.ls2_iters))


def write_timings_csv(trajectory: Iterable, path: str) -> None:
    """write_timings_csv (io.cpp:50-62)."""
    with open(path, "w") as out:
        out.write("level,iter,setup_s,ls1_s,ls2_s\n")
        for r in trajectory:
            out.write("%d,%d,%.6g,%.6g,%.6g\n" % (r.level, r.iter, r.setup_seconds,
                                                  r.ls1_seconds, r.ls2_seconds))


@dataclass
class BenchRow:
    """BenchRow (io.hpp:30-37); iterations = -1 marks a did-not-finish entry."""
    phase: str
    preconditioner: str
    cr: int
    dof: int
    iterations: int
    seconds: float


def write_bench_csv(rows: Iterable[BenchRow], path: str) -> None:
    """write_bench_csv (io.cpp:64-76)."""
    with open(path, "w") as out:
        out.write("phase,preconditioner,cr,dof,iterations,seconds\n")
        for r in rows:
            out.write("%s,%s,%d,%d,%d,%.6g\n" % (r.phase, r.preconditioner, r.cr, r.dof,
                                                 r.iterations, r.seconds))
