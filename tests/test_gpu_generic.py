"""Any coarse-cell shape: the generic kernels
(csrc/generic.cu) against the oracle's restatement, the compiled reference
(oracle/_ref, including its Lanczos path above 4096 cells per box) and, for
4^3 / 8^3 bricks forced onto the generic kernels (TMG_FORCE_GENERIC=1), the
tuned templated kernels.

Bars as everywhere (BASELINE.json north_star): the TPFA apply and rhs are
bitwise; PCG iterations within 10% (+-1), relative solution error <= 1e-6;
local bases span the reference's eigenspaces (principal angles)."""
import os

import numpy as np
import pytest
import scipy.linalg as sla

import oracle as O
from paper_2410_06850_b200 import (BoundarySpec, Context, GridSpec, MmgOptions, inputs)

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

BC = BoundarySpec.bottom_center_patch(1.0, 1.0, 0.2, 0.0)
PATCH = O.bottom_center_patch()
CELL = MmgOptions(fine_blocks="coarse_cell")


def iters_close(a, b):
    return abs(a - b) <= max(1, int(0.1 * b))


def design(shape, kmin, vf=0.3, seed=20240501):
    """seeded box-filter design on any (nx, ny, nz) grid (inputs.py generator)"""
    rho = inputs.box_filter_design(shape, vf, seed=seed)
    return rho, inputs.conductivity(rho, kmin)


def ctx(shape, ncc, sd, kappa, slabs=1, generic=None):
    old = os.environ.get("TMG_FORCE_GENERIC")
    if generic:
        os.environ["TMG_FORCE_GENERIC"] = "1"
    try:
        c = Context(GridSpec(*shape), ncc, sd, slabs=slabs)
    finally:
        if generic:
            if old is None:
                del os.environ["TMG_FORCE_GENERIC"]
            else:
                os.environ["TMG_FORCE_GENERIC"] = old
    c.set_conductivity(kappa, BC)
    return c


def span_close(a, b, cos_min=1 - 1e-8):
    """principal angles between the row spaces of a and b (M-orthonormal
    bases compared after orthonormalising in the Euclidean metric)"""
    qa, _ = np.linalg.qr(a.T)
    qb, _ = np.linalg.qr(b.T)
    s = sla.svdvals(qa.T @ qb)
    return s.min() >= cos_min, s.min()


# --------------------------------------------------- forced generic vs tuned

@pytest.mark.parametrize("n,ncc,sd", [(32, 2, 2), (32, 4, 2)])
def test_forced_generic_matches_tuned(n, ncc, sd):
    """8^3 and 4^3 bricks through the generic kernels: the operator is
    bitwise the tuned one, the MMG solves agree to the solver tolerance."""
    shape = (n, n, n)
    _, kappa = design(shape, 1e-6)
    t = ctx(shape, ncc, sd, kappa)
    g = ctx(shape, ncc, sd, kappa, generic=True)
    x = np.random.default_rng(1).standard_normal(n ** 3)
    np.testing.assert_array_equal(g.apply_operator(x), t.apply_operator(x))
    b = t.assemble_rhs(np.ones(n ** 3))
    np.testing.assert_array_equal(g.assemble_rhs(np.ones(n ** 3)), b)
    for kind, opts in [("jacobi", MmgOptions()), ("mmg", CELL), ("mmg", MmgOptions()),
                       ("two_grid", CELL), ("mmg", MmgOptions(fine_blocks="coarse_cell",
                                                              smoother_sweeps=2))]:
        t.setup(kind, opts)
        g.setup(kind, opts)
        rt = t.pcg(b, rtol=1e-8, max_iterations=20000)
        rg = g.pcg(b, rtol=1e-8, max_iterations=20000)
        assert rt.report.converged and rg.report.converged, kind
        # Jacobi-PCG at contrast 1e6 runs ~1800 rounding-sensitive iterations
        # (the dot products' summation order differs): the usual 10% bar
        close = (iters_close if kind == "jacobi" else
                 lambda a, b: abs(a - b) <= 1)(rg.report.iterations, rt.report.iterations)
        assert close, (kind, rt.report.iterations, rg.report.iterations)
        assert np.linalg.norm(rg.x - rt.x) <= 1e-6 * np.linalg.norm(rt.x), kind
    # local bases: same eigenspaces per coarse cell
    t.setup("mmg", CELL)
    g.setup("mmg", CELL)
    pt, et, _ = t.local_bases()
    pg, eg, _ = g.local_bases()
    np.testing.assert_allclose(eg, et, rtol=1e-6, atol=1e-10)
    for cid in range(0, pt.shape[0], max(1, pt.shape[0] // 7)):
        ok, cmin = span_close(pt[cid], pg[cid], 1 - 1e-7)
        assert ok, (cid, cmin)


# ------------------------------------------- general shapes vs the oracle

SHAPES = [
    ((24, 16, 32), (2, 2, 2), 2),   # c = (6, 4, 8): non-cubic
    ((24, 24, 24), (4, 4, 4), 2),   # c = 3
    ((16, 16, 16), (4, 4, 4), 2),   # c = 2 (8 cells: the whole box is the subspace)
    ((20, 12, 16), (2, 3, 2), 2),   # c = (5, 2, 4)
]


@pytest.mark.parametrize("shape,ncc,sd", SHAPES)
def test_generic_apply_and_rhs_bitwise(shape, ncc, sd):
    m = int(np.prod(shape))
    rng = np.random.default_rng(m)
    kappa = 10.0 ** rng.uniform(-6, 0, m)
    source = rng.random(m)
    s = O.System(O.grid(shape), kappa, source, PATCH)
    c = ctx(shape, ncc, sd, kappa)
    x = rng.standard_normal(m)
    np.testing.assert_array_equal(c.apply_operator(x), s.apply(x))
    np.testing.assert_array_equal(c.assemble_rhs(source), s.rhs)


@pytest.mark.parametrize("shape,ncc,sd", SHAPES)
@pytest.mark.parametrize("kind,fine", [("mmg", "cell"), ("mmg", "cc"), ("two_grid", "cell"),
                                       ("block_jacobi", "cc"), ("jacobi", None)])
def test_generic_pcg_vs_oracle(shape, ncc, sd, kind, fine):
    _, kappa = design(shape, 1e-3)
    s = O.System(O.grid(shape), kappa, np.ones(int(np.prod(shape))), PATCH)
    h = O.hierarchy(O.grid(shape), ncc, sd)
    lc = min(4, int(np.prod([n // (k * sd) for n, k in zip(shape, ncc)])))
    if kind == "jacobi":
        m = O.Precond("jacobi", s)
    elif kind == "block_jacobi":
        m = O.Precond("block_jacobi", s, h, fine_blocks="cc")
    else:
        m = O.Precond(kind, s, h, lc=lc, fine_blocks=fine, coarse_blocks="cc")
    ref = O.pcg(s, s.rhs, m, rtol=1e-8, max_iterations=20000)
    c = ctx(shape, ncc, sd, kappa)
    c.setup(kind, MmgOptions(num_local_basis=lc,
                             fine_blocks="cc" if fine == "cc" else "coarse_cell"))
    r = c.pcg(s.rhs, rtol=1e-8, max_iterations=20000)
    assert r.report.converged and ref.converged
    assert iters_close(r.report.iterations, ref.iterations), (r.report.iterations, ref.iterations)
    assert np.linalg.norm(r.x - ref.x) <= 1e-6 * np.linalg.norm(ref.x)


@pytest.mark.parametrize("shape,ncc,sd", SHAPES[:2])
def test_generic_local_bases_vs_oracle(shape, ncc, sd):
    _, kappa = design(shape, 1e-6)
    c = ctx(shape, ncc, sd, kappa)
    c.setup("mmg", CELL)
    phi, ev, it = c.local_bases()
    assert np.all(it >= 0)
    h = O.hierarchy(O.grid(shape), ncc, sd)
    for cid in range(0, phi.shape[0], max(1, phi.shape[0] // 5)):
        vals, vecs = O.local_basis(h, kappa, cid, 4)
        np.testing.assert_allclose(ev[cid], vals, rtol=1e-6, atol=1e-9 * vals.max())
        ok, cmin = span_close(phi[cid], vecs, 1 - 1e-7)
        assert ok, (cid, cmin)


def test_generic_slabs_match_single():
    """the partitioned path (in-process z-slabs) on a generic shape"""
    shape, ncc, sd = (24, 16, 32), (2, 2, 4), 2
    _, kappa = design(shape, 1e-3)
    one = ctx(shape, ncc, sd, kappa)
    two = ctx(shape, ncc, sd, kappa, slabs=2)
    x = np.random.default_rng(5).standard_normal(int(np.prod(shape)))
    np.testing.assert_array_equal(two.apply_operator(x), one.apply_operator(x))
    b = one.assemble_rhs(np.ones(int(np.prod(shape))))
    for opts in (CELL, MmgOptions()):
        one.setup("mmg", opts)
        two.setup("mmg", opts)
        r1 = one.pcg(b, rtol=1e-8)
        r2 = two.pcg(b, rtol=1e-8)
        assert r1.report.converged and r2.report.converged
        assert abs(r1.report.iterations - r2.report.iterations) <= 1
        assert np.linalg.norm(r2.x - r1.x) <= 1e-8 * np.linalg.norm(r1.x)


@pytest.mark.parametrize("kind", ["mmg", "block_jacobi"])
def test_tuned_bricks_with_box_fine_blocks(kind):
    """4^3 bricks (tuned kernels) with sd = 3: the reference's cc-element fine
    blocks of 12^3 cells are outside the tuned block_jacobi.cu sizes and run
    the generic box block Thomas"""
    n, ncc, sd = 24, 2, 3
    _, kappa = design((n, n, n), 1e-3)
    s = O.System(O.grid(n), kappa, np.ones(n ** 3), PATCH)
    h = O.hierarchy(O.grid(n), ncc, sd)
    m = (O.Precond("block_jacobi", s, h, fine_blocks="cc") if kind == "block_jacobi" else
         O.Precond("mmg", s, h, fine_blocks="cc", coarse_blocks="cc"))
    ref = O.pcg(s, s.rhs, m, rtol=1e-8, max_iterations=20000)
    c = ctx((n, n, n), ncc, sd, kappa)
    c.setup(kind)
    r = c.pcg(s.rhs, rtol=1e-8, max_iterations=20000)
    assert r.report.converged and ref.converged
    assert iters_close(r.report.iterations, ref.iterations), (r.report.iterations, ref.iterations)
    assert np.linalg.norm(r.x - ref.x) <= 1e-6 * np.linalg.norm(ref.x)


@pytest.mark.parametrize("n,ncc,sd,lc,lcc", [(24, 2, 3, 1, 4),    # q = 27 (odd, warp Jacobi)
                                              (24, 2, 3, 3, 8),    # q = 81 (batched tensor-core GJ)
                                              (16, 4, 1, 3, 2)])   # q = 3
def test_any_coarse_block_size(n, ncc, sd, lc, lcc):
    """cc elements of q = sd^3 L_c coarse unknowns of any size: odd q <= 64
    (round-robin Jacobi with a bye) and q > 64 not a multiple of 64"""
    _, kappa = design((n, n, n), 1e-3)
    s = O.System(O.grid(n), kappa, np.ones(n ** 3), PATCH)
    h = O.hierarchy(O.grid(n), ncc, sd)
    m = O.Precond("mmg", s, h, lc=lc, lcc=lcc, fine_blocks="cell", coarse_blocks="cc")
    ref = O.pcg(s, s.rhs, m, rtol=1e-8, max_iterations=20000)
    c = ctx((n, n, n), ncc, sd, kappa)
    c.setup("mmg", MmgOptions(num_local_basis=lc, num_cc_basis=lcc, fine_blocks="coarse_cell"))
    r = c.pcg(s.rhs, rtol=1e-8, max_iterations=20000)
    assert r.report.converged and ref.converged
    assert iters_close(r.report.iterations, ref.iterations), (r.report.iterations, ref.iterations)
    assert np.linalg.norm(r.x - ref.x) <= 1e-6 * np.linalg.norm(ref.x)


# ------------------------------- against the compiled reference (oracle/_ref)

@needs_ref
def test_generic_default_preconditioner_vs_reference():
    """make_preconditioner(Mmg) of the reference itself (fine_blocks_by_cc,
    solver.cpp:387-399) on a non-cubic hierarchy"""
    shape, ncc, sd = (24, 16, 32), (2, 2, 2), 2
    _, kappa = design(shape, 1e-6)
    rc = O.RefContext(shape, ncc, sd, kappa, fine_blocks=None, coarse_blocks=None)
    c = ctx(shape, ncc, sd, kappa)
    b = c.assemble_rhs(np.ones(int(np.prod(shape))))
    ref = rc.solve(b, rtol=1e-8)
    c.setup("mmg")
    r = c.pcg(b, rtol=1e-8)
    assert r.report.converged and ref.converged
    assert iters_close(r.report.iterations, ref.iterations), (r.report.iterations, ref.iterations)
    assert np.linalg.norm(r.x - ref.x) <= 1e-6 * np.linalg.norm(ref.x)


@needs_ref
def test_lanczos_boxes_vs_reference():
    """17^3 = 4913-cell coarse cells: above SpectralOptions::dense_threshold
    (coarse_space.hpp:37-42) the reference switches to lanczos_smallest
    (coarse_space.cpp:61-198), which returns the pairs in descending order.
    The GPU's bases keep that order, span the same eigenspaces, and the MMG
    solve matches the reference's."""
    n, ncc, sd = 34, 1, 2
    shape = (n, n, n)
    _, kappa = design(shape, 1e-3)
    c = ctx(shape, ncc, sd, kappa)
    c.setup("mmg", MmgOptions(fine_blocks="coarse_cell", num_cc_basis=8))
    phi, ev, it = c.local_bases()
    assert phi.shape == (8, 4, 17 ** 3) and np.all(it >= 0)
    for cid in (0, 5):
        vals, vecs = O.ref_local_basis_grid(shape, ncc, sd, kappa, cid, 4)
        assert np.all(np.diff(vals) <= 0)  # descending, as the reference returns them
        np.testing.assert_allclose(ev[cid], vals, rtol=1e-6, atol=1e-9 * vals.max())
        for a in range(4):  # pairwise (simple eigenvalues here)
            cosang = abs(phi[cid, a] @ vecs[a]) / (np.linalg.norm(phi[cid, a]) *
                                                  np.linalg.norm(vecs[a]))
            assert cosang >= 1 - 1e-6, (cid, a, cosang)
    rc = O.RefContext(shape, ncc, sd, kappa, fine_blocks="cell", coarse_blocks="cc")
    b = c.assemble_rhs(np.ones(n ** 3))
    ref = rc.solve(b, rtol=1e-8)
    r = c.pcg(b, rtol=1e-8)
    assert r.report.converged and ref.converged
    assert iters_close(r.report.iterations, ref.iterations), (r.report.iterations, ref.iterations)
    assert np.linalg.norm(r.x - ref.x) <= 1e-6 * np.linalg.norm(ref.x)
