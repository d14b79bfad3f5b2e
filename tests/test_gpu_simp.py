"""SIMP design loop on the device (BASELINE
configs[2]). The filter and OC rules are builder-defined (M5) and checked
against the numpy restatements below; the solves and the sensitivity inside
one design iteration are checked against the compiled reference ("only
per-solve parity is pinned")."""
import numpy as np
import pytest

import oracle as O
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, inputs

pytestmark = pytest.mark.gpu

BC = BoundarySpec.bottom_center_patch(1.0, 1.0, 0.2, 0.0)
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def np_filter(x, n, r, mode, W=None):
    """Linear-hat density filter (csrc/simp.cu k_density_filter), numpy."""
    nx, ny, nz = n
    R = int(np.floor(r))
    x3 = np.zeros((nz, ny, nx)) if x is None else x.reshape(nz, ny, nx)
    W3 = None if W is None else W.reshape(nz, ny, nx)
    out = np.zeros((nz, ny, nx))
    for dk in range(-R, R + 1):
        for dj in range(-R, R + 1):
            for di in range(-R, R + 1):
                w = r - np.sqrt(di * di + dj * dj + dk * dk)
                if w <= 0:
                    continue
                src = [slice(max(0, d), n_ + min(0, d)) for d, n_ in ((dk, nz), (dj, ny), (di, nx))]
                dst = [slice(max(0, -d), n_ + min(0, -d)) for d, n_ in ((dk, nz), (dj, ny), (di, nx))]
                if mode == 0:
                    out[tuple(dst)] += w
                elif mode == 1:
                    out[tuple(dst)] += w * x3[tuple(src)]
                else:
                    out[tuple(dst)] += w * x3[tuple(src)] / W3[tuple(src)]
    if mode == 1:
        out /= W3
    return out.ravel()


def np_oc(x, dc, dv, volfrac, move, n, r, W):
    lo, hi = 1e-40, 1e40
    for _ in range(200):
        if hi / lo <= 1 + 1e-10:
            break
        mid = np.sqrt(lo * hi)
        xn = np.clip(x * np.sqrt(np.maximum(0, -dc) / (mid * dv)), np.maximum(0, x - move),
                     np.minimum(1, x + move))
        if np_filter(xn, n, r, 1, W).mean() > volfrac:
            lo = mid
        else:
            hi = mid
    return np.clip(x * np.sqrt(np.maximum(0, -dc) / (hi * dv)), np.maximum(0, x - move),
                   np.minimum(1, x + move))


@needs_ref
def test_simp_step_matches_reference_pieces():
    n, kmin, vf, rmin = 32, 1e-3, 0.3, 1.5
    nn = (n, n, n)
    rng = np.random.default_rng(50)
    rho0 = np.clip(0.3 + 0.2 * rng.standard_normal(n ** 3), 0.0, 1.0)
    c = Context(GridSpec(n, n, n), 2, 2)
    c.set_design(rho0, kmin, 1.0, 3, BC)
    c.simp_init(volfrac=vf, rmin=rmin, move=0.2, kappa_lo=kmin, rtol=1e-10, rho0=rho0)
    rep = c.simp_step()
    xphys_after, T = c.simp_download()
    # filter (mode 1) of the initial design = the densities the step solved on
    W = np_filter(None, nn, rmin, 0)
    xphys = np_filter(rho0, nn, rmin, 1, W)
    # state solve: the reference PCG on the same system (per-solve parity)
    kap = inputs.conductivity(xphys, kmin)
    s = O.System(O.grid(n), kap, np.ones(n ** 3), O.bottom_center_patch())
    ref = O.pcg(s, s.rhs, O.Precond("mmg", s, O.hierarchy(O.grid(n), 2, 2), fine_blocks="cell",
                                    coarse_blocks="cc"), rtol=1e-10)
    assert abs(rep["ls1_iterations"] - ref.iterations) <= max(1, 0.1 * ref.iterations)
    np.testing.assert_allclose(T, ref.x, rtol=1e-7, atol=1e-7 * abs(ref.x).max())
    assert abs(rep["cost"] - ref.x.mean()) <= 1e-7 * abs(ref.x.mean())
    assert abs(rep["volume"] - xphys.mean()) <= 1e-13
    # the OC step moves the design by at most the move limit
    assert 0.0 < rep["change"] <= 0.2 + 1e-12
    assert abs(xphys_after.mean() - vf) <= 1e-6


def test_simp_sensitivity_and_oc_restated():
    """The step's dc (filter transpose of the reference sensitivity) and the
    OC update, restated in numpy, reproduce the device design update."""
    n, kmin, vf, rmin = 16, 1e-3, 0.3, 1.5
    nn = (n, n, n)
    rho0 = np.full(n ** 3, vf)
    c = Context(GridSpec(n, n, n), 1, 2)
    c.set_design(rho0, kmin, 1.0, 3, BC)
    c.simp_init(volfrac=vf, rmin=rmin, move=0.2, kappa_lo=kmin, rtol=1e-12, rho0=rho0)
    c.simp_step()
    xphys1, T = c.simp_download()
    # adjoint by a dense solve on the same design
    W = np_filter(None, nn, rmin, 0)
    xphys0 = np_filter(rho0, nn, rmin, 1, W)
    s = O.System(O.grid(n), inputs.conductivity(xphys0, kmin), np.ones(n ** 3),
                 O.bottom_center_patch())
    A = s.matrix.toarray()
    T_exact = np.linalg.solve(A, s.rhs)
    np.testing.assert_allclose(T, T_exact, rtol=1e-9, atol=1e-9 * abs(T_exact).max())
    U = np.linalg.solve(A, np.full(n ** 3, 1.0 / n ** 3))
    dcp = O.ref_sensitivity(n, xphys0, T_exact, U, kmin, 1.0, 0.0, 3)
    dc = np_filter(dcp, nn, rmin, 2, W)
    dv = np_filter(np.full(n ** 3, 1.0 / n ** 3), nn, rmin, 2, W)
    x1 = np_oc(rho0, dc, dv, vf, 0.2, nn, rmin, W)
    np.testing.assert_allclose(xphys1, np_filter(x1, nn, rmin, 1, W), rtol=1e-6, atol=1e-6)


def test_simp_loop_configs2_shape():
    """configs[2]-style loop (uniform start, r = 1.5, move 0.2) at 32^3: the
    cost falls, the volume holds, warm-started solves converge."""
    n = 32
    c = Context(GridSpec(n, n, n), 2, 2)
    c.set_design(np.full(n ** 3, 0.3), 1e-6, 1.0, 3, BC)
    c.simp_init(volfrac=0.3, rmin=1.5, move=0.2, kappa_lo=1e-6, rtol=1e-8)
    reps = [c.simp_step() for _ in range(6)]
    costs = [r["cost"] for r in reps]
    assert costs[-1] < 0.5 * costs[0]
    assert all(abs(r["volume"] - 0.3) < 1e-6 for r in reps[1:])
    assert all(r["ls1_iterations"] > 0 and r["ls2_iterations"] > 0 for r in reps)
    xphys, T = c.simp_download()
    assert xphys.min() >= 0.0 and xphys.max() <= 1.0
