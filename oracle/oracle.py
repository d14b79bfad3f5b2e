"""ORACLE — test infrastructure only.

ctypes front-end for ``oracle/liboracle.so`` (the plain-C restatement of the
reference hot path, ``oracle/topmg_oracle.c``) and, when it has been built, for
``oracle/_ref/libtopmg_ref.so`` (the reference's own ``proj/core`` sources
compiled here, see ``oracle/build_ref.sh``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

I64 = C.c_int64
DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int64)

KIND = {"none": 0, "jacobi": 1, "block_jacobi": 2, "two_grid": 3, "mmg": 4}
BLOCKS = {"cc": 0, "point": 1, "cell": 2, "box2": 18, "box4": 20, "box8": 24}
FACE = {"xlo": 0, "xhi": 1, "ylo": 2, "yhi": 3, "zlo": 4, "zhi": 5}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Grid(C.Structure):
    _fields_ = [("nx", I64), ("ny", I64), ("nz", I64),
                ("lx", C.c_double), ("ly", C.c_double), ("lz", C.c_double)]


class Patch(C.Structure):
    _fields_ = [("face", C.c_int), ("u0", C.c_double), ("v0", C.c_double),
                ("u1", C.c_double), ("v1", C.c_double), ("value", C.c_double)]


class HGrid(C.Structure):
    _fields_ = [("spec", Grid), ("ncc", I64 * 3), ("sd", I64),
                ("nc", I64 * 3), ("cpc", I64 * 3)]


class Csr(C.Structure):
    _fields_ = [("rows", I64), ("cols", I64), ("off", IP), ("col", IP), ("val", DP)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int),
                ("solve_seconds", C.c_double), ("setup_seconds", C.c_double)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.check_call(["make", "-s", "-C", HERE, "liboracle.so"])
        L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_precond_op.restype = C.POINTER(Csr)
        L.orc_count_dirichlet_faces.restype = I64
        _LIB = L
    return _LIB


def _d(a):
    return a.ctypes.data_as(DP)


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def bottom_center_patch(lx=1.0, ly=1.0, side=0.2, value=0.0):
    """BoundarySpec::bottom_center_patch (proj/core/src/grid.cpp:107-119)."""
    return [(4, 0.5 * (lx - side), 0.5 * (ly - side), 0.5 * (lx + side),
             0.5 * (ly + side), value)]


def _patches(patches):
    arr = (Patch * max(1, len(patches)))()
    for i, p in enumerate(patches):
        arr[i] = Patch(*p)
    return arr, len(patches)


def grid(n, l=(1.0, 1.0, 1.0)):
    nx, ny, nz = (n, n, n) if np.isscalar(n) else n
    return Grid(nx, ny, nz, *l)


def csr_to_scipy(c):
    import scipy.sparse as sp
    nnz = c.off[c.rows]
    off = np.ctypeslib.as_array(c.off, shape=(c.rows + 1,)).copy()
    col = np.ctypeslib.as_array(c.col, shape=(nnz,)).copy() if nnz else np.zeros(0, np.int64)
    val = np.ctypeslib.as_array(c.val, shape=(nnz,)).copy() if nnz else np.zeros(0)
    return sp.csr_matrix((val, col, off), shape=(c.rows, c.cols))


def conductivity(rho, kappa_lo, kappa_hi=1.0, p=3):
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    out = np.empty_like(rho)
    _check(lib().orc_conductivity(I64(rho.size), _d(rho), C.c_double(kappa_lo),
                                  C.c_double(kappa_hi), C.c_int(p), _d(out)))
    return out


def box_filter_design(g, vf, seed=20240501, passes=3, radius=2):
    out = np.empty(g.nx * g.ny * g.nz)
    lib().orc_box_filter_design(C.byref(g), C.c_double(vf), C.c_uint64(seed),
                                C.c_int(passes), C.c_int(radius), _d(out))
    return out


def frozen_bench_design(g, vstar, seed=20240501, passes=2):
    out = np.empty(g.nx * g.ny * g.nz)
    lib().orc_frozen_bench_design(C.byref(g), C.c_double(vstar), C.c_uint64(seed),
                                  C.c_int(passes), _d(out))
    return out


class System:
    """AssembledSystem (proj/core/include/topmg/fvm.hpp:20-26)."""

    def __init__(self, g, kappa, source, patches):
        self.grid = g
        self.kappa = np.ascontiguousarray(kappa, dtype=np.float64)
        self.source = np.ascontiguousarray(source, dtype=np.float64)
        self.patches = list(patches)
        self.csr = Csr()
        self.rhs = np.empty(self.kappa.size)
        parr, np_ = _patches(self.patches)
        _check(lib().orc_assemble(C.byref(g), _d(self.kappa), _d(self.source), parr,
                                  C.c_int(np_), C.byref(self.csr), _d(self.rhs)))

    def __del__(self):
        try:
            lib().orc_csr_free(C.byref(self.csr))
        except Exception:
            pass

    @property
    def matrix(self):
        return csr_to_scipy(self.csr)

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.csr.rows)
        lib().orc_spmv(C.byref(self.csr), _d(x), _d(y))
        return y


def hierarchy(g, ncc, sd):
    h = HGrid()
    ncc3 = (I64 * 3)(*((ncc,) * 3 if np.isscalar(ncc) else ncc))
    _check(lib().orc_build_hierarchy(C.byref(g), ncc3, I64(sd), C.byref(h)))
    return h


def local_basis(h, kappa, cid, count):
    n = h.cpc[0] * h.cpc[1] * h.cpc[2]
    vals = np.empty(count)
    vecs = np.empty(count * n)
    _check(lib().orc_local_basis(C.byref(h), _d(kappa), I64(cid), I64(count),
                                 _d(vals), _d(vecs)))
    return vals, vecs.reshape(count, n)


class Precond:
    """make_preconditioner (solver.cpp:462-481) with explicit smoother blocks."""

    def __init__(self, kind, system, h=None, lc=4, lcc=8, sweeps=1,
                 fine_blocks="point", coarse_blocks="cell"):
        self.ptr = C.c_void_p()
        self.system = system
        hh = C.byref(h) if h is not None else None
        _check(lib().orc_make_preconditioner(
            C.c_int(KIND[kind]), C.byref(system.csr), hh, _d(system.kappa),
            I64(lc), I64(lcc), C.c_int(sweeps), C.c_int(BLOCKS[fine_blocks]),
            C.c_int(BLOCKS[coarse_blocks]), C.byref(self.ptr)))

    def __del__(self):
        try:
            lib().orc_precond_free(self.ptr)
        except Exception:
            pass

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty_like(r)
        _check(lib().orc_precond_apply(self.ptr, _d(r), _d(z)))
        return z

    def op(self, which):
        p = lib().orc_precond_op(self.ptr, C.c_int(which))
        return csr_to_scipy(p.contents) if p else None


@dataclass
class PcgResult:
    x: np.ndarray
    iterations: int
    converged: bool
    residual_history: np.ndarray
    solve_seconds: float


def pcg(system, b, m, rtol=1e-6, max_iterations=10000, x0=None):
    """topmg::pcg (proj/core/src/solver.cpp:483-575)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty_like(b)
    hist = np.zeros(max(1, max_iterations))
    rep = Report()
    x0p = _d(np.ascontiguousarray(x0, dtype=np.float64)) if x0 is not None else None
    _check(lib().orc_pcg(C.byref(system.csr), _d(b), m.ptr, C.c_double(rtol),
                         C.c_int(max_iterations), x0p, _d(x), _d(hist), C.byref(rep)))
    return PcgResult(x, rep.iterations, bool(rep.converged), hist[:rep.iterations].copy(),
                     rep.solve_seconds)


def syev_smallest(a, k):
    a = np.array(a, dtype=np.float64, order="C")
    n = a.shape[0]
    w = np.empty(k)
    v = np.empty((n, k))
    L = lib()
    rc = L.dla_syev_smallest(C.c_int(n), C.c_int(k), _d(a), _d(w), _d(v))
    if rc:
        raise OracleError(rc, "eigensolver failed")
    return w, v


def syev_all(a):
    a = np.array(a, dtype=np.float64, order="C")
    n = a.shape[0]
    w = np.empty(n)
    v = np.empty((n, n))
    rc = lib().dla_syev_all(C.c_int(n), _d(a), _d(w), _d(v))
    if rc:
        raise OracleError(rc, "eigensolver failed")
    return w, v


# --------------------------------------------------------------------------
# The reference itself (oracle/_ref/libtopmg_ref.so, built by build_ref.sh)
# --------------------------------------------------------------------------

REF_PATH = os.path.join(HERE, "_ref", "libtopmg_ref.so")


def ref_available():
    return os.path.exists(REF_PATH)


def ref():
    global _REF
    if _REF is None:
        R = C.CDLL(REF_PATH)
        R.ref_last_error.restype = C.c_char_p
        R.ref_ctx_create.restype = C.c_void_p
        R.ref_ctx_create.argtypes = [I64, I64, I64, DP, C.c_int, DP, C.c_int, C.c_int, C.c_int,
                                     I64, I64, C.c_int, DP]
        R.ref_ctx_create_grid.restype = C.c_void_p
        R.ref_ctx_create_grid.argtypes = [I64, I64, I64, C.c_double, C.c_double, C.c_double,
                                          I64, I64, I64, I64, DP, C.c_int, DP, C.c_int, C.c_int,
                                          C.c_int, I64, I64, C.c_int, DP]
        R.ref_sensitivity.argtypes = [I64, I64, I64, C.c_double, C.c_double, C.c_double, DP,
                                      C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, DP,
                                      DP, DP, DP]
        R.ref_ctx_pcg.argtypes = [C.c_void_p, C.c_double, C.c_int, DP, C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), DP]
        R.ref_ctx_destroy.argtypes = [C.c_void_p]
        IP = C.POINTER(C.c_int)
        R.ref_optimize.argtypes = [C.c_int, C.POINTER(I64), IP, I64, I64, C.c_double, C.c_double,
                                   C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, DP,
                                   C.c_double, C.c_int, C.c_int, IP, DP, DP, IP, IP, DP, DP, IP]
        R.ref_num_threads.restype = C.c_int
        _REF = R
    return _REF


def sensitivity(n, rho, t, u, kappa_lo, kappa_hi=1.0, f0=1.0, p=3, patches=None,
                extent=(1.0, 1.0, 1.0)):
    """Restatement of topmg::sensitivity (optim.cpp:21-84) in numpy, same
    operation order (elementwise, no contraction)."""
    nx, ny, nz = (n, n, n) if np.isscalar(n) else n
    hx, hy, hz = extent[0] / nx, extent[1] / ny, extent[2] / nz
    vol = hx * hy * hz
    cpl = (hy * hz / hx, hx * hz / hy, hx * hy / hz)
    rho3 = np.asarray(rho, dtype=float).reshape(nz, ny, nx)
    t3 = np.asarray(t, dtype=float).reshape(nz, ny, nx)
    u3 = np.asarray(u, dtype=float).reshape(nz, ny, nx)
    # material.cpp:45-74 (int_pow by repeated multiply)
    xp = np.ones_like(rho3)
    for _ in range(p):
        xp = xp * rho3
    kap = kappa_lo + xp * (kappa_hi - kappa_lo)
    xp1 = np.ones_like(rho3)
    if p >= 2:
        for _ in range(p - 1):
            xp1 = xp1 * rho3
    dk = float(p) * xp1 * (kappa_hi - kappa_lo)
    dsrc = -float(p) * xp1 * f0
    val = u3 * dsrc * vol
    on = dk != 0.0
    patches = patches if patches is not None else bottom_center_patch()
    for a in range(3):
        ax = 2 - a  # array axis of coordinate a
        n_a = (nx, ny, nz)[a]
        for side in (0, 1):
            sl_c = [slice(None)] * 3
            sl_n = [slice(None)] * 3
            if side == 0:
                sl_c[ax], sl_n[ax] = slice(1, n_a), slice(0, n_a - 1)
            else:
                sl_c[ax], sl_n[ax] = slice(0, n_a - 1), slice(1, n_a)
            sc, sn = tuple(sl_c), tuple(sl_n)
            kc, kn = kap[sc], kap[sn]
            kf = 2.0 * kc * kn / (kc + kn)
            ratio = kf / kc
            dt = 0.5 * ratio * ratio * dk[sc] * cpl[a]
            term = dt * (u3[sc] - u3[sn]) * (t3[sc] - t3[sn])
            v = val[sc]
            val[sc] = np.where(on[sc], v - term, v)
        for side in (0, 1):
            face = 2 * a + side
            sl = [slice(None)] * 3
            sl[ax] = slice(0, 1) if side == 0 else slice(n_a - 1, n_a)
            sl = tuple(sl)
            # boundary-face centres of the layer (grid.cpp:61-75)
            k_i, j_i, i_i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
            cx, cy, cz = (i_i[sl] + 0.5) * hx, (j_i[sl] + 0.5) * hy, (k_i[sl] + 0.5) * hz
            uu, vv = ((cy, cz), (cx, cz), (cx, cy))[a]
            td = np.zeros(uu.shape)
            hit = np.zeros(uu.shape, dtype=bool)
            for (f, u0, v0, u1, v1, value) in patches:
                if f != face:
                    continue
                m = (~hit) & (uu >= u0) & (uu <= u1) & (vv >= v0) & (vv <= v1)
                td[m] = value
                hit |= m
            dtd = 2.0 * cpl[a] * dk[sl]
            add = dtd * u3[sl] * (td - t3[sl])
            val[sl] = np.where(hit & on[sl], val[sl] + add, val[sl])
    return val.ravel()


def ref_sensitivity(n, rho, t, u, kappa_lo, kappa_hi=1.0, f0=1.0, p=3, patches=None,
                    extent=(1.0, 1.0, 1.0)):
    """topmg::sensitivity (optim.cpp:21-84) of the compiled reference."""
    nx, ny, nz = (n, n, n) if np.isscalar(n) else n
    patches = patches if patches is not None else bottom_center_patch()
    pa = _patch_array(patches)
    out = np.empty(nx * ny * nz)
    R = ref()
    _ref_check(R.ref_sensitivity(nx, ny, nz, *extent, _d(np.ascontiguousarray(rho, dtype=float)),
                                 kappa_lo, kappa_hi, f0, p, len(patches), _d(pa),
                                 _d(np.ascontiguousarray(t, dtype=float)),
                                 _d(np.ascontiguousarray(u, dtype=float)), _d(out)))
    return out


def ref_optimize(levels, iters, ncc, sd, vstar=0.05, convergence_dx=0.01, kappa_lo=1e-3,
                 kappa_hi=1.0, f0=1.0, p=3, patches=None, rtol=1e-6, maxit=10000):
    """topmg::optimize (optim.cpp:240-345) of the compiled reference on cubic
    levels; returns (trajectory dict of arrays, final design, final cost, failed)."""
    patches = patches if patches is not None else bottom_center_patch()
    pa = _patch_array(patches)
    nl = len(levels)
    lv = (I64 * nl)(*levels)
    it = (C.c_int * nl)(*iters)
    cap = int(sum(iters)) + 1
    costs, vols = np.zeros(cap), np.zeros(cap)
    l1, l2 = np.zeros(cap, dtype=np.int32), np.zeros(cap, dtype=np.int32)
    nlog, failed = C.c_int(0), C.c_int(0)
    fc = C.c_double(0.0)
    x = np.empty(levels[-1] ** 3)
    IP = C.POINTER(C.c_int)
    _ref_check(ref().ref_optimize(nl, lv, it, ncc, sd, vstar, convergence_dx, kappa_lo, kappa_hi,
                                  f0, p, len(patches), _d(pa), rtol, maxit, cap, C.byref(nlog),
                                  _d(costs), _d(vols), l1.ctypes.data_as(IP),
                                  l2.ctypes.data_as(IP), _d(x), C.byref(fc), C.byref(failed)))
    n = nlog.value
    traj = {"cost": costs[:n], "volume": vols[:n], "ls1": l1[:n], "ls2": l2[:n]}
    return traj, x, fc.value, bool(failed.value)


def _ref_check(rc):
    if rc != 0:
        raise OracleError(rc, ref().ref_last_error().decode())


def _patch_array(patches):
    a = np.zeros(6 * max(1, len(patches)))
    for i, p in enumerate(patches):
        a[6 * i:6 * i + 6] = p
    return a


def ref_frozen_bench_design(n, vstar, seed=20240501, passes=2):
    out = np.empty(n ** 3)
    ref().ref_frozen_bench_design(I64(n), I64(n), I64(n), C.c_double(vstar), C.c_uint64(seed),
                                  C.c_int(passes), _d(out))
    return out


def ref_conductivity(x, lo, hi=1.0, p=3):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _ref_check(ref().ref_conductivity(I64(x.size), _d(x), C.c_double(lo), C.c_double(hi),
                                      C.c_int(p), _d(out)))
    return out


def ref_assemble(n, kappa, source, patches, l=(1.0, 1.0, 1.0)):
    nx, ny, nz = (n, n, n) if np.isscalar(n) else n
    m = nx * ny * nz
    off = np.empty(m + 1, dtype=np.int64)
    col = np.empty(7 * m, dtype=np.int64)
    val = np.empty(7 * m)
    rhs = np.empty(m)
    pa = _patch_array(patches)
    _ref_check(ref().ref_assemble(I64(nx), I64(ny), I64(nz), C.c_double(l[0]), C.c_double(l[1]),
                                  C.c_double(l[2]), _d(np.ascontiguousarray(kappa, np.float64)),
                                  _d(np.ascontiguousarray(source, np.float64)), C.c_int(len(patches)),
                                  _d(pa), off.ctypes.data_as(IP), col.ctypes.data_as(IP), _d(val),
                                  _d(rhs)))
    import scipy.sparse as sp
    nnz = off[-1]
    return sp.csr_matrix((val[:nnz], col[:nnz], off), shape=(m, m)), rhs


def ref_local_basis(n, ncc, sd, kappa, cid, count):
    cpc = n // (ncc * sd)
    vals = np.empty(count)
    vecs = np.empty(count * cpc ** 3)
    _ref_check(ref().ref_local_basis(I64(n), I64(n), I64(n), I64(ncc), I64(sd),
                                     _d(np.ascontiguousarray(kappa, np.float64)), I64(cid),
                                     I64(count), _d(vals), _d(vecs)))
    return vals, vecs.reshape(count, cpc ** 3)


def ref_local_basis_grid(shape, ncc, sd, kappa, cid, count):
    """local_spectral_basis on an (nx, ny, nz) grid with per-axis ncc; boxes
    above 4096 cells run the reference's Lanczos path."""
    nx, ny, nz = shape
    ncx, ncy, ncz = (ncc,) * 3 if np.isscalar(ncc) else tuple(ncc)
    cpc = (nx // (ncx * sd)) * (ny // (ncy * sd)) * (nz // (ncz * sd))
    vals = np.empty(count)
    vecs = np.empty(count * cpc)
    _ref_check(ref().ref_local_basis_grid(I64(nx), I64(ny), I64(nz), I64(ncx), I64(ncy), I64(ncz),
                                          I64(sd), _d(np.ascontiguousarray(kappa, np.float64)),
                                          I64(cid), I64(count), _d(vals), _d(vecs)))
    return vals, vecs.reshape(count, cpc)


def ref_solve(n, ncc, sd, kappa, rhs, patches, kind="mmg", fine_blocks=None,
              coarse_blocks=None, lc=4, lcc=8, sweeps=1, rtol=1e-8, maxit=10000, x0=None):
    """Reference make_preconditioner/build_hierarchy_operators + pcg. Blocks:
    None = make_preconditioner default; 'cc' / 'point' / 'cell'."""
    m = n ** 3
    x = np.empty(m)
    hist = np.zeros(max(1, maxit))
    it = C.c_int()
    conv = C.c_int()
    ts = C.c_double()
    tv = C.c_double()
    pa = _patch_array(patches)
    fb = -1 if fine_blocks is None else BLOCKS[fine_blocks]
    cb = -1 if coarse_blocks is None else BLOCKS[coarse_blocks]
    x0p = _d(np.ascontiguousarray(x0, np.float64)) if x0 is not None else None
    _ref_check(ref().ref_solve(I64(n), I64(ncc), I64(sd),
                               _d(np.ascontiguousarray(kappa, np.float64)),
                               _d(np.ascontiguousarray(rhs, np.float64)), C.c_int(len(patches)),
                               _d(pa), C.c_int(KIND[kind]), C.c_int(fb), C.c_int(cb), I64(lc),
                               I64(lcc), C.c_int(sweeps), C.c_double(rtol), C.c_int(maxit), x0p,
                               _d(x), C.byref(it), C.byref(conv), _d(hist), C.byref(ts),
                               C.byref(tv)))
    return PcgResult(x, it.value, bool(conv.value), hist[:it.value].copy(), tv.value), ts.value


def interpolate_design(values_lo, n_lo, n_hi):
    """interpolate_design (grid.cpp:220-241): piecewise-constant prolongation."""
    v = np.ascontiguousarray(values_lo, dtype=np.float64)
    glo, ghi = grid(n_lo), grid(n_hi)
    out = np.empty(ghi.nx * ghi.ny * ghi.nz)
    _check(lib().orc_interpolate_design(_d(v), C.byref(glo), C.byref(ghi), _d(out)))
    return out


class RefContext:
    """The reference's set-up kept alive (oracle/_ref, ref_ctx_*): one
    make_preconditioner / build_hierarchy_operators, then any number of
    pcg() calls with any rhs and x0 (solver.cpp:483-575). fine_blocks None =
    the reference's make_preconditioner default (fine_blocks_by_cc)."""

    def __init__(self, shape, ncc, sd, kappa, patches=None, kind="mmg", fine_blocks="cell",
                 coarse_blocks="cc", lc=4, lcc=8, sweeps=1, extent=None, threads=0):
        nx, ny, nz = (shape,) * 3 if np.isscalar(shape) else tuple(shape)
        ncx, ncy, ncz = (ncc,) * 3 if np.isscalar(ncc) else tuple(ncc)
        ext = extent or (1.0, 1.0, 1.0)
        R = ref()
        R.ref_set_num_threads(threads)
        R.ref_ctx_solve.argtypes = [C.c_void_p, DP, DP, C.c_double, C.c_int, DP, DP,
                                    C.POINTER(C.c_int), C.POINTER(C.c_int), DP]
        R.ref_ctx_apply.argtypes = [C.c_void_p, DP, DP]
        self.m = nx * ny * nz
        pa = _patch_array(patches if patches is not None else bottom_center_patch())
        ts = C.c_double()
        fb = -1 if fine_blocks is None else BLOCKS[fine_blocks]
        cb = -1 if coarse_blocks is None else BLOCKS[coarse_blocks]
        self.ptr = R.ref_ctx_create_grid(nx, ny, nz, ext[0], ext[1], ext[2], ncx, ncy, ncz, sd,
                                         _d(np.ascontiguousarray(kappa, np.float64)),
                                         len(pa) // 6, _d(pa), KIND[kind], fb, cb, lc, lcc,
                                         sweeps, C.byref(ts))
        if not self.ptr:
            raise OracleError(4, R.ref_last_error().decode())
        self.setup_seconds = ts.value
        self.threads = R.ref_num_threads()

    def solve(self, b=None, rtol=1e-8, maxit=10000, x0=None):
        x = np.empty(self.m)
        hist = np.zeros(max(1, maxit))
        it, cv, sv = C.c_int(), C.c_int(), C.c_double()
        bp = _d(np.ascontiguousarray(b, np.float64)) if b is not None else None
        xp = _d(np.ascontiguousarray(x0, np.float64)) if x0 is not None else None
        _ref_check(ref().ref_ctx_solve(self.ptr, bp, xp, C.c_double(rtol), C.c_int(maxit), _d(x),
                                       _d(hist), C.byref(it), C.byref(cv), C.byref(sv)))
        return PcgResult(x, it.value, bool(cv.value), hist[:it.value].copy(), sv.value)

    def apply(self, x):
        y = np.empty(self.m)
        _ref_check(ref().ref_ctx_apply(self.ptr, _d(np.ascontiguousarray(x, np.float64)), _d(y)))
        return y

    def close(self):
        if getattr(self, "ptr", None):
            ref().ref_ctx_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
