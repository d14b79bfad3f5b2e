"""Artifact writers (paper_2410_06850_b200/io.py) byte-identical to the
reference's io.cpp (compiled in oracle/_ref)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
from paper_2410_06850_b200 import GridSpec, IterationLog
from paper_2410_06850_b200.io import (BenchRow, write_bench_csv, write_timings_csv,
                                      write_trajectory_csv, write_vtk_cell_scalars)

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int)


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(DP)


@needs_ref
def test_vtk_ascii_matches_reference(tmp_path):
    g = GridSpec(5, 3, 4, 1.0, 0.75, 2.0)
    rng = np.random.default_rng(0)
    f = np.concatenate([rng.standard_normal(56) * 10.0 ** rng.integers(-12, 12, 56),
                        [0.0, -0.0, 1.0, 1e300]])[:60]
    a, b = tmp_path / "a.vtk", tmp_path / "b.vtk"
    write_vtk_cell_scalars(g, f, "rho", str(a))
    R = O.ref()
    R.ref_write_vtk.argtypes = [C.c_int64] * 3 + [C.c_double] * 3 + [DP, C.c_char_p, C.c_char_p]
    assert R.ref_write_vtk(5, 3, 4, 1.0, 0.75, 2.0, _d(f), b"rho", str(b).encode()) == 0
    assert a.read_bytes() == b.read_bytes()


def test_vtk_binary_roundtrip(tmp_path):
    g = GridSpec(4, 4, 2)
    f = np.arange(32, dtype=float) / 7.0
    p = tmp_path / "c.vtk"
    write_vtk_cell_scalars(g, f, "t", str(p), binary=True)
    raw = p.read_bytes()
    head_end = raw.index(b"LOOKUP_TABLE default\n") + len(b"LOOKUP_TABLE default\n")
    assert b"BINARY" in raw[:head_end]
    np.testing.assert_array_equal(np.frombuffer(raw[head_end:head_end + 256], dtype=">f8"), f)


@needs_ref
def test_csvs_match_reference(tmp_path):
    rows = [IterationLog(level=l, iter=i, cost=1.0 / (i + 3) * 10 ** l, volume=0.3 - 1e-3 * i,
                         ls1_iters=10 + i, ls2_iters=11 + i, setup_seconds=0.0123 * i,
                         ls1_seconds=1.5e-3 * i, ls2_seconds=2.25e-3)
            for l in range(2) for i in range(1, 4)]
    write_trajectory_csv(rows, str(tmp_path / "t.csv"))
    write_timings_csv(rows, str(tmp_path / "s.csv"))
    n = len(rows)
    col = lambda k, t: (t * n)(*[getattr(r, k) for r in rows])
    R = O.ref()
    R.ref_write_trajectory.argtypes = [C.c_int, IP, IP, DP, DP, IP, IP, DP, DP, DP, C.c_char_p,
                                       C.c_char_p]
    assert R.ref_write_trajectory(
        n, col("level", C.c_int), col("iter", C.c_int), col("cost", C.c_double),
        col("volume", C.c_double), col("ls1_iters", C.c_int), col("ls2_iters", C.c_int),
        col("setup_seconds", C.c_double), col("ls1_seconds", C.c_double),
        col("ls2_seconds", C.c_double), str(tmp_path / "rt.csv").encode(),
        str(tmp_path / "rs.csv").encode()) == 0
    assert (tmp_path / "t.csv").read_bytes() == (tmp_path / "rt.csv").read_bytes()
    assert (tmp_path / "s.csv").read_bytes() == (tmp_path / "rs.csv").read_bytes()
    bench = [BenchRow("setup", "mmg", 6, 2097152, 0, 0.0293), BenchRow("ls1", "mmg", 6, 2097152,
                                                                       33, 0.0176),
             BenchRow("ls1", "jacobi", 6, 2097152, -1, 1.7366)]
    write_bench_csv(bench, str(tmp_path / "b.csv"))
    m = len(bench)
    strs = lambda k: (C.c_char_p * m)(*[getattr(r, k).encode() for r in bench])
    R.ref_write_bench.argtypes = [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p), IP,
                                  C.POINTER(C.c_int64), IP, DP, C.c_char_p]
    assert R.ref_write_bench(m, strs("phase"), strs("preconditioner"),
                             (C.c_int * m)(*[r.cr for r in bench]),
                             (C.c_int64 * m)(*[r.dof for r in bench]),
                             (C.c_int * m)(*[r.iterations for r in bench]),
                             (C.c_double * m)(*[r.seconds for r in bench]),
                             str(tmp_path / "rb.csv").encode()) == 0
    assert (tmp_path / "b.csv").read_bytes() == (tmp_path / "rb.csv").read_bytes()
