"""Python front-end over the C ABI (include/topmg_b200.h).

Mirrors the reference's solver interface (proj/core/include/topmg/solver.hpp)
so the tests read like the reference's: ``GridSpec``, ``BoundarySpec``,
``MmgOptions``, ``PrecondKind``, ``make_preconditioner`` and ``pcg`` with the
same argument meaning and the same error classes (``ConfigError``,
``SolverError``, ``ValueError`` for std::invalid_argument). All compute runs in
``libtopmg_b200.so``; there is no CPU fallback — importing the native library
fails loudly when it has not been built.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TMG_LIB", os.path.join(_HERE, "libtopmg_b200.so"))

TMG_OK, TMG_ECONFIG, TMG_ESOLVER, TMG_EARG, TMG_ECUDA, TMG_ENOTSUP = range(6)


class ConfigError(RuntimeError):
    """topmg::ConfigError (grid.hpp:16-19)."""


class SolverError(RuntimeError):
    """topmg::SolverError (grid.hpp:21-24)."""


class CudaError(RuntimeError):
    pass


class NotSupportedError(RuntimeError):
    pass


class _Grid(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("lx", C.c_double), ("ly", C.c_double), ("lz", C.c_double),
                ("ncc", C.c_int64 * 3), ("sd", C.c_int64)]


class _Patch(C.Structure):
    _fields_ = [("face", C.c_int), ("u0", C.c_double), ("v0", C.c_double),
                ("u1", C.c_double), ("v1", C.c_double), ("value", C.c_double)]


class _Opts(C.Structure):
    _fields_ = [("kind", C.c_int), ("num_local_basis", C.c_int64),
                ("num_cc_basis", C.c_int64), ("smoother_sweeps", C.c_int),
                ("eig_tol", C.c_double), ("eig_degree", C.c_int), ("eig_max_outer", C.c_int),
                ("warm_start", C.c_int), ("fine_blocks", C.c_int)]


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("status", C.c_int),
                ("setup_seconds", C.c_double), ("solve_seconds", C.c_double),
                ("final_relative_residual", C.c_double), ("restarts", C.c_int)]


class _SimpOpts(C.Structure):
    _fields_ = [("volfrac", C.c_double), ("rmin", C.c_double), ("move", C.c_double),
                ("kappa_lo", C.c_double), ("kappa_hi", C.c_double), ("p", C.c_int),
                ("source", C.c_double), ("rtol", C.c_double), ("maxit", C.c_int)]


class _SimpReport(C.Structure):
    _fields_ = [("iteration", C.c_int), ("cost", C.c_double), ("volume", C.c_double),
                ("change", C.c_double), ("ls1_iterations", C.c_int), ("ls2_iterations", C.c_int),
                ("setup_seconds", C.c_double), ("ls1_seconds", C.c_double),
                ("ls2_seconds", C.c_double), ("step_seconds", C.c_double)]


class _DesignGen(C.Structure):
    _fields_ = [("vf", C.c_double), ("seed", C.c_uint64), ("passes", C.c_int),
                ("radius", C.c_int)]


class _TreeGen(C.Structure):
    _fields_ = [("vf", C.c_double), ("seed", C.c_uint64), ("passes", C.c_int),
                ("radius", C.c_int), ("depth", C.c_int), ("length0", C.c_double),
                ("lshrink", C.c_double), ("width0", C.c_double), ("wshrink", C.c_double),
                ("spread", C.c_double), ("amp", C.c_double), ("dom", C.c_double * 3),
                ("global_n", C.c_int64 * 3), ("z0", C.c_int64)]


class _OptimOpts(C.Structure):
    _fields_ = [("vstar", C.c_double), ("move_limit", C.c_double), ("asy_init", C.c_double),
                ("asy_incr", C.c_double), ("asy_decr", C.c_double), ("kappa_lo", C.c_double),
                ("kappa_hi", C.c_double), ("f0", C.c_double), ("p", C.c_int),
                ("rtol", C.c_double), ("maxit", C.c_int), ("warm_start", C.c_int)]


class _IterLog(C.Structure):
    _fields_ = [("iter", C.c_int), ("cost", C.c_double), ("volume", C.c_double),
                ("ls1_iters", C.c_int), ("ls2_iters", C.c_int), ("setup_seconds", C.c_double),
                ("ls1_seconds", C.c_double), ("ls2_seconds", C.c_double),
                ("dx_inf", C.c_double), ("lambda", C.c_double), ("step_seconds", C.c_double)]


_lib = None
_DP = C.POINTER(C.c_double)


def native():
    """Load libtopmg_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {_HERE}` or "
                "`python -c 'import __graft_entry__; __graft_entry__.build()'`")
        L = C.CDLL(LIB_PATH)
        L.tmg_last_error.restype = C.c_char_p
        L.tmg_last_error.argtypes = [C.c_void_p]
        L.tmg_device_bytes.restype = C.c_int64
        L.tmg_kernel_launches.restype = C.c_int64
        L.tmg_stream.restype = C.c_void_p
        L.tmg_destroy.argtypes = [C.c_void_p]
        _lib = L
    return _lib


EXPORTED_SYMBOLS = (
    "tmg_create", "tmg_destroy", "tmg_last_error", "tmg_set_conductivity", "tmg_set_design",
    "tmg_assemble_rhs", "tmg_setup", "tmg_pcg", "tmg_apply_operator",
    "tmg_apply_preconditioner", "tmg_upload_rhs", "tmg_upload_x0", "tmg_solve_resident",
    "tmg_download_solution", "tmg_get_local_bases", "tmg_get_coarse_operator",
    "tmg_get_fine_factor_slots",
    "tmg_get_cc_restriction", "tmg_get_sizes", "tmg_profile_solve", "tmg_device_bytes",
    "tmg_stream", "tmg_kernel_launches", "tmg_create_slabs", "tmg_nccl_unique_id",
    "tmg_create_dist", "tmg_partition", "tmg_set_x0_interpolated", "tmg_set_design_interpolated",
    "tmg_sensitivity", "tmg_simp_init", "tmg_simp_step", "tmg_simp_download",
    "tmg_optim_init", "tmg_optim_step", "tmg_optim_evaluate", "tmg_optim_download",
    "tmg_set_design_generated", "tmg_solve_resident_ex", "tmg_apply_operator_abs",
    "tmg_set_design_tree", "tmg_halo_plan", "tmg_set_design_frozen",
)


def _raise(code: int, msg: str):
    if code == TMG_OK:
        return
    cls = {TMG_ECONFIG: ConfigError, TMG_ESOLVER: SolverError, TMG_EARG: ValueError,
           TMG_ECUDA: CudaError, TMG_ENOTSUP: NotSupportedError}.get(code, RuntimeError)
    raise cls(msg)


def _ptr(a):
    return a.ctypes.data_as(_DP)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ inputs

@dataclass
class GridSpec:
    """GridSpec (grid.hpp:30-55)."""
    nx: int
    ny: int
    nz: int
    lx: float = 1.0
    ly: float = 1.0
    lz: float = 1.0

    def num_cells(self):
        return self.nx * self.ny * self.nz


@dataclass
class DirichletPatch:
    face: int
    u0: float
    v0: float
    u1: float
    v1: float
    value: float = 0.0


@dataclass
class BoundarySpec:
    """BoundarySpec (grid.hpp:70-91)."""
    patches: List[DirichletPatch] = field(default_factory=list)

    @staticmethod
    def bottom_center_patch(lx: float, ly: float, side: float, value: float) -> "BoundarySpec":
        # grid.cpp:107-119
        return BoundarySpec([DirichletPatch(4, 0.5 * (lx - side), 0.5 * (ly - side),
                                            0.5 * (lx + side), 0.5 * (ly + side), value)])

    def _c(self):
        arr = (_Patch * max(1, len(self.patches)))()
        for i, p in enumerate(self.patches):
            arr[i] = _Patch(p.face, p.u0, p.v0, p.u1, p.v1, p.value)
        return arr, len(self.patches)


class PrecondKind:
    """PrecondKind (solver.hpp:160)."""
    NONE, JACOBI, BLOCK_JACOBI, TWO_GRID, MMG = range(5)
    _names = {"none": 0, "jacobi": 1, "block_jacobi": 2, "two_grid": 3, "mmg": 4}

    @classmethod
    def parse(cls, name: str) -> int:
        # parse_precond_kind (solver.cpp:422-429)
        if name not in cls._names:
            raise ConfigError("unknown preconditioner kind: " + name)
        return cls._names[name]


@dataclass
class MmgOptions:
    """MmgOptions (solver.hpp:141-146)."""
    num_local_basis: int = 4
    num_cc_basis: int = 8
    smoother_sweeps: int = 1
    eig_tol: float = 0.0
    eig_degree: int = 0
    eig_max_outer: int = 0
    warm_start: bool = False  # start the local eigensolver from the previous set-up's bases
    # fine smoother partition (mmg, two_grid): "cc", the default, is the
    # reference build_mmg's fine_blocks_by_cc (solver.cpp:353-361; cc elements
    # of 8^3, 16^3 or 32^3 cells on the GPU); "coarse_cell" opts into one
    # exact block per coarse cell, the fast GPU partition
    fine_blocks: str = "cc"

    def _c(self, kind):
        fb = {"cc": 0, "coarse_cell": 1}
        if self.fine_blocks not in fb:
            raise ValueError(f"fine_blocks must be one of {list(fb)}")
        return _Opts(kind, self.num_local_basis, self.num_cc_basis, self.smoother_sweeps,
                     self.eig_tol, self.eig_degree, self.eig_max_outer, int(self.warm_start),
                     fb[self.fine_blocks])


@dataclass
class SolveReport:
    """SolveReport (solver.hpp:15-22)."""
    preconditioner: str = ""
    iterations: int = 0
    converged: bool = False
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0
    status: int = 0
    final_relative_residual: float = 0.0
    restarts: int = 0  # residual replacements (solve_resident(true_residual=True))


@dataclass
class PcgResult:
    x: np.ndarray
    report: SolveReport


def partition(grid: GridSpec, ncc, sd: int, nranks: int, rank: int) -> dict:
    """Slab `rank` of `nranks` (tmg_partition; host-only, no GPU needed)."""
    L = native()
    ncc3 = (ncc,) * 3 if np.isscalar(ncc) else tuple(ncc)
    g = _Grid(grid.nx, grid.ny, grid.nz, grid.lx, grid.ly, grid.lz, (C.c_int64 * 3)(*ncc3), sd)
    out = (C.c_int64 * 10)()
    rc = L.tmg_partition(C.byref(g), C.c_int(nranks), C.c_int(rank), out)
    if rc:
        _raise(rc, L.tmg_last_error(None).decode())
    keys = ("z0", "z1", "brick0", "bricks", "elem0", "elems", "cell0", "cells", "lo", "hi")
    return dict(zip(keys, (int(v) for v in out)))


def nccl_unique_id() -> bytes:
    """NCCL unique id for tmg_create_dist (make on rank 0, broadcast)."""
    buf = C.create_string_buffer(128)
    rc = native().tmg_nccl_unique_id(buf, C.c_int(128))
    if rc:
        _raise(rc, native().tmg_last_error(None).decode())
    return buf.raw


class Context:
    """One GPU solve context: grid hierarchy + problem + preconditioner."""

    def __init__(self, grid: GridSpec, ncc: Sequence[int] | int, sd: int, device: int = 0,
                 slabs: int = 1, rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None):
        """slabs > 1: the grid split into z-slabs inside this process (one GPU);
        nranks > 1: this process holds slab `rank` and talks NCCL to the others
        (host arrays are then the rank's own slab, see partition())."""
        L = native()
        ncc3 = (ncc,) * 3 if np.isscalar(ncc) else tuple(ncc)
        self._g = _Grid(grid.nx, grid.ny, grid.nz, grid.lx, grid.ly, grid.lz,
                        (C.c_int64 * 3)(*ncc3), sd)
        self.grid = grid
        self.ncc = ncc3
        self.sd = sd
        self.slabs = slabs
        self.rank, self.nranks = rank, nranks
        ptr = C.c_void_p()
        if nranks > 1:
            if slabs != 1:
                raise ValueError("a distributed context holds one slab per rank")
            idb = C.create_string_buffer(bytes(nccl_id), 128)
            rc = L.tmg_create_dist(C.byref(self._g), C.c_int(device), C.c_int(rank),
                                   C.c_int(nranks), idb, C.byref(ptr))
        elif slabs > 1:
            rc = L.tmg_create_slabs(C.byref(self._g), C.c_int(device), C.c_int(slabs),
                                    C.byref(ptr))
        else:
            rc = L.tmg_create(C.byref(self._g), C.c_int(device), C.byref(ptr))
        if rc:
            _raise(rc, L.tmg_last_error(None).decode())
        self._p = ptr
        self.kind_name = None
        # cells of every host array this context takes or returns
        self.cells = (partition(grid, ncc3, sd, nranks, rank)["cells"] if nranks > 1
                      else grid.num_cells())

    def close(self):
        if getattr(self, "_p", None):
            native().tmg_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc:
            _raise(rc, native().tmg_last_error(self._p).decode())

    # problem
    def set_conductivity(self, kappa, boundary: BoundarySpec):
        k = _f64(kappa)
        parr, n = boundary._c()
        self._check(native().tmg_set_conductivity(self._p, _ptr(k), parr, C.c_int(n)))

    def set_design(self, rho, kappa_lo, kappa_hi=1.0, p=3, boundary: BoundarySpec = None):
        r = _f64(rho)
        parr, n = boundary._c()
        self._check(native().tmg_set_design(self._p, _ptr(r), C.c_double(kappa_lo),
                                            C.c_double(kappa_hi), C.c_int(p), parr, C.c_int(n)))

    def set_design_generated(self, vf, kappa_lo, kappa_hi=1.0, p=3,
                             boundary: BoundarySpec = None, seed=20240501, passes=3, radius=2,
                             return_rho=False):
        """inputs.box_filter_design generated on the device (bit-identical),
        then as set_design. Returns the whole design (x-fastest) if asked."""
        g = _DesignGen(vf, seed, passes, radius)
        parr, n = boundary._c()
        rho = np.empty(self.grid.num_cells()) if return_rho else None
        self._check(native().tmg_set_design_generated(
            self._p, C.byref(g), C.c_double(kappa_lo), C.c_double(kappa_hi), C.c_int(p), parr,
            C.c_int(n), _ptr(rho) if rho is not None else None))
        return rho

    def set_design_frozen(self, vstar, kappa_lo, kappa_hi=1.0, p=3,
                          boundary: BoundarySpec = None, seed=20240501, passes=2,
                          return_rho=False):
        """frozen_bench_design (rng.cpp:16-53) on the device, bit-identical
        to the reference's (tmg_set_design_frozen), then as set_design."""
        parr, n = boundary._c()
        rho = np.empty(self.grid.num_cells()) if return_rho else None
        self._check(native().tmg_set_design_frozen(
            self._p, C.c_double(vstar), C.c_uint64(seed), C.c_int(passes), C.c_double(kappa_lo),
            C.c_double(kappa_hi), C.c_int(p), parr, C.c_int(n),
            _ptr(rho) if rho is not None else None))
        return rho

    def set_design_tree(self, vf, kappa_lo, kappa_hi=1.0, p=3, boundary: BoundarySpec = None,
                        seed=20240501, passes=1, radius=6, dom=None, return_rho=False,
                        global_n=None, z0=0, **tree):
        """BASELINE configs[4]'s tree-like design generated on the device
        (tmg_set_design_tree; bit-identical to inputs.tree_design), then as
        set_design. dom: extents of the whole domain the tree lives in
        (default: the context's own); global_n: generate the whole design on
        that grid over dom and keep this context's z-slab from layer z0."""
        from .inputs import TREE_DEFAULTS
        t = dict(TREE_DEFAULTS)
        t.update(tree)
        g = _TreeGen(vf, seed, passes, radius, t["depth"], t["length0"], t["lshrink"],
                     t["width0"], t["wshrink"], t["spread"], t["amp"],
                     (C.c_double * 3)(*(dom or (0.0, 0.0, 0.0))),
                     (C.c_int64 * 3)(*(global_n or (0, 0, 0))), z0)
        parr, n = boundary._c()
        rho = np.empty(self.grid.num_cells()) if return_rho else None
        self._check(native().tmg_set_design_tree(
            self._p, C.byref(g), C.c_double(kappa_lo), C.c_double(kappa_hi), C.c_int(p), parr,
            C.c_int(n), _ptr(rho) if rho is not None else None))
        return rho

    def set_design_interpolated(self, rho_lo, shape_lo, kappa_lo, kappa_hi=1.0, p=3,
                                boundary: BoundarySpec = None):
        """interpolate_design (grid.cpp:220-241) of a coarser design on the
        device, then set_design."""
        r = _f64(rho_lo)
        n = (C.c_int64 * 3)(*shape_lo)
        parr, npat = boundary._c()
        self._check(native().tmg_set_design_interpolated(
            self._p, _ptr(r), n, C.c_double(kappa_lo), C.c_double(kappa_hi), C.c_int(p), parr,
            C.c_int(npat)))

    def set_x0_interpolated(self, x_lo, shape_lo):
        """Warm start for solve_resident(use_x0=True): a coarser grid's field
        prolonged on the device (interpolate_design semantics)."""
        xx = _f64(x_lo)
        n = (C.c_int64 * 3)(*shape_lo)
        self._check(native().tmg_set_x0_interpolated(self._p, _ptr(xx), n))

    def sensitivity(self, rho, t, u, kappa_lo, kappa_hi=1.0, f0=1.0, p=3):
        """sensitivity (optim.cpp:21-84) on the device: d(mean T)/d rho."""
        r, tt, uu = _f64(rho), _f64(t), _f64(u)
        out = np.empty(self.cells)
        self._check(native().tmg_sensitivity(self._p, _ptr(r), C.c_double(kappa_lo),
                                             C.c_double(kappa_hi), C.c_double(f0), C.c_int(p),
                                             _ptr(tt), _ptr(uu), _ptr(out)))
        return out

    # SIMP design loop (BASELINE configs[2]; include/topmg_b200.h tmg_simp_*)
    def simp_init(self, volfrac=0.3, rmin=1.5, move=0.2, kappa_lo=1e-6, kappa_hi=1.0, p=3,
                  source=1.0, rtol=1e-8, maxit=10000, rho0=None,
                  mmg: MmgOptions = MmgOptions(fine_blocks="coarse_cell")):
        o = _SimpOpts(volfrac, rmin, move, kappa_lo, kappa_hi, p, source, rtol, maxit)
        m = mmg._c(PrecondKind.parse("mmg"))
        r0 = _ptr(_f64(rho0)) if rho0 is not None else None
        self._check(native().tmg_simp_init(self._p, C.byref(o), C.byref(m), r0))

    def simp_step(self) -> dict:
        r = _SimpReport()
        self._check(native().tmg_simp_step(self._p, C.byref(r)))
        return {k: getattr(r, k) for k, _ in _SimpReport._fields_}

    def simp_download(self):
        """(filtered design, last state solution), x-fastest."""
        xp, t = np.empty(self.cells), np.empty(self.cells)
        self._check(native().tmg_simp_download(self._p, _ptr(xp), _ptr(t)))
        return xp, t

    # reference design loop (topmg::optimize with MMA, one level; optim.py)
    def optim_init(self, vstar=0.05, kappa_lo=1e-3, kappa_hi=1.0, f0=1.0, p=3, move_limit=0.2,
                   asy_init=0.5, asy_incr=1.2, asy_decr=0.7, rtol=1e-6, maxit=10000,
                   warm_start=False, x0=None, kind="mmg", mmg: MmgOptions = MmgOptions()):
        o = _OptimOpts(vstar, move_limit, asy_init, asy_incr, asy_decr, kappa_lo, kappa_hi, f0, p,
                       rtol, maxit, int(warm_start))
        m = mmg._c(PrecondKind.parse(kind) if isinstance(kind, str) else kind)
        xp = _ptr(_f64(x0)) if x0 is not None else None
        self._check(native().tmg_optim_init(self._p, C.byref(o), C.byref(m), xp))

    def optim_step(self) -> dict:
        r = _IterLog()
        self._check(native().tmg_optim_step(self._p, C.byref(r)))
        return {k: getattr(r, k) for k, _ in _IterLog._fields_}

    def optim_evaluate(self) -> dict:
        r = _IterLog()
        self._check(native().tmg_optim_evaluate(self._p, C.byref(r)))
        return {k: getattr(r, k) for k, _ in _IterLog._fields_}

    def optim_download(self):
        """(design, last state solution), x-fastest."""
        x, t = np.empty(self.cells), np.empty(self.cells)
        self._check(native().tmg_optim_download(self._p, _ptr(x), _ptr(t)))
        return x, t

    def assemble_rhs(self, source=None):
        out = np.empty(self.cells)
        sp = _ptr(_f64(source)) if source is not None else None
        self._check(native().tmg_assemble_rhs(self._p, sp, _ptr(out)))
        return out

    # preconditioner
    def setup(self, kind: int | str, opts: MmgOptions = MmgOptions()):
        if isinstance(kind, str):
            self.kind_name = kind
            kind = PrecondKind.parse(kind)
        else:
            self.kind_name = [k for k, v in PrecondKind._names.items() if v == kind][0]
        o = opts._c(kind)
        self._check(native().tmg_setup(self._p, C.byref(o)))

    # operators
    def apply_operator(self, x):
        xx = _f64(x)
        y = np.empty_like(xx)
        self._check(native().tmg_apply_operator(self._p, _ptr(xx), _ptr(y)))
        return y

    def apply_operator_abs(self, x):
        """|A| |x| (tmg_apply_operator_abs)."""
        xx = _f64(x)
        y = np.empty_like(xx)
        self._check(native().tmg_apply_operator_abs(self._p, _ptr(xx), _ptr(y)))
        return y

    def residual_floor(self, x, b):
        """eps ||(|A||x|)|| / ||b||: the rounding floor of any FP64 residual
        b - A x of x ("true residual")."""
        return float(np.finfo(np.float64).eps / 2 * np.linalg.norm(self.apply_operator_abs(x))
                     / np.linalg.norm(b))

    def apply_preconditioner(self, r):
        rr = _f64(r)
        z = np.empty_like(rr)
        self._check(native().tmg_apply_preconditioner(self._p, _ptr(rr), _ptr(z)))
        return z

    def pcg(self, b, rtol=1e-6, max_iterations=10000, x0=None, out=None) -> PcgResult:
        bb = _f64(b)
        if bb.size != self.cells:
            raise ValueError("pcg: rhs size mismatch")
        if x0 is not None and np.asarray(x0).size != self.cells:
            raise ValueError("pcg: initial guess size mismatch")
        x = np.empty_like(bb) if out is None else out
        hist = np.zeros(max(1, max_iterations))
        rep = _Report()
        x0p = _ptr(_f64(x0)) if x0 is not None else None
        self._check(native().tmg_pcg(self._p, _ptr(bb), x0p, C.c_double(rtol),
                                     C.c_int(max_iterations), _ptr(x), _ptr(hist),
                                     C.byref(rep)))
        return PcgResult(x, self._report(rep, hist))

    def _report(self, rep, hist=None):
        return SolveReport(self.kind_name or "", rep.iterations, bool(rep.converged),
                           hist[:rep.iterations].copy() if hist is not None else np.zeros(0),
                           rep.setup_seconds, rep.solve_seconds, rep.status,
                           rep.final_relative_residual, rep.restarts)

    # resident (bench)
    def upload_rhs(self, b):
        self._check(native().tmg_upload_rhs(self._p, _ptr(_f64(b))))

    def solve_resident(self, rtol, max_iterations, use_x0=False,
                       true_residual=False) -> SolveReport:
        """PCG on the resident rhs. The default is the reference's recurrence
        stopping rule. true_residual=True: residual replacement until
        ||b - A x|| / ||b|| <= rtol (tmg_solve_resident_ex,
        TMG_SOLVE_TRUE_RESIDUAL): converged and final_relative_residual then
        refer to the TRUE residual; status 6 = stuck at the FP64 floor."""
        rep = _Report()
        self._check(native().tmg_solve_resident_ex(self._p, C.c_double(rtol),
                                                   C.c_int(max_iterations), C.c_int(int(use_x0)),
                                                   C.c_int(1 if true_residual else 0),
                                                   C.byref(rep)))
        return self._report(rep)

    def download_solution(self):
        x = np.empty(self.cells)
        self._check(native().tmg_download_solution(self._p, _ptr(x)))
        return x

    # introspection
    def sizes(self):
        s = (C.c_int64 * 6)()
        self._check(native().tmg_get_sizes(self._p, s))
        return dict(zip(["M", "m_c", "n_c", "m_cc", "n_cc", "cells_per_coarse"], list(s)))

    def local_bases(self):
        s = self.sizes()
        lc = s["n_c"] // s["m_c"]
        phi = np.empty(s["n_c"] * s["cells_per_coarse"])
        ev = np.empty(s["n_c"])
        it = np.empty(s["m_c"], dtype=np.int32)
        self._check(native().tmg_get_local_bases(self._p, _ptr(phi), _ptr(ev),
                                                 it.ctypes.data_as(C.POINTER(C.c_int))))
        return phi.reshape(s["m_c"], lc, s["cells_per_coarse"]), ev.reshape(s["m_c"], lc), it

    def coarse_operator(self):
        n = self.sizes()["n_c"]
        a = np.empty((n, n))
        self._check(native().tmg_get_coarse_operator(self._p, _ptr(a)))
        return a

    def cc_restriction(self):
        s = self.sizes()
        a = np.empty((s["n_cc"], s["n_c"]))
        self._check(native().tmg_get_cc_restriction(self._p, _ptr(a)))
        return a

    def profile_solve(self, rtol, max_iterations):
        ms = (C.c_double * 9)()
        cnt = (C.c_int * 9)()
        self._check(native().tmg_profile_solve(self._p, C.c_double(rtol),
                                               C.c_int(max_iterations), ms, cnt))
        names = ["search", "update", "restrict", "coarse", "unused4", "unused5", "post",
                 "jacobi_step", "init"]
        return {n: (ms[i], cnt[i]) for i, n in enumerate(names)}

    def kernel_launches(self):
        return native().tmg_kernel_launches(self._p)

    def device_bytes(self):
        return native().tmg_device_bytes(self._p)

    def fine_factor_slots(self):
        """(factor slots, bricks) of the per-coarse-cell fine blocks: uniform
        interior bricks share one scaled factor."""
        a, b = C.c_int64(), C.c_int64()
        self._check(native().tmg_get_fine_factor_slots(self._p, C.byref(a), C.byref(b)))
        return a.value, b.value

    def stream(self):
        return native().tmg_stream(self._p)


def make_preconditioner(kind, grid: GridSpec, kappa, boundary: BoundarySpec, ncc, sd,
                        opts: MmgOptions = MmgOptions(), device: int = 0) -> Context:
    """make_preconditioner (solver.cpp:462-481) on the GPU: returns a context
    holding A (matrix-free from kappa) and the set-up preconditioner."""
    ctx = Context(grid, ncc, sd, device)
    ctx.set_conductivity(kappa, boundary)
    ctx.setup(kind, opts)
    return ctx


def pcg(ctx: Context, b, rtol=1e-6, max_iterations=10000, x0=None) -> PcgResult:
    """topmg::pcg (solver.cpp:483-575) with the context's operator and preconditioner."""
    return ctx.pcg(b, rtol=rtol, max_iterations=max_iterations, x0=x0)
