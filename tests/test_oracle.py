"""CPU tests of the oracle (oracle/, test infrastructure): it is pinned against
the spec's known answers, the golden fixtures produced by the reference itself
(tests/golden/make_golden.py), and — when oracle/_ref has been built here — the
compiled reference directly. Also checks the product-side input generator
against the oracle's C generator (bit-identical)."""
import glob
import os

import numpy as np
import pytest

import oracle as O
from paper_2410_06850_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
PATCH = O.bottom_center_patch()


# ------------------------------------------------------------- known answers

def test_kat_conductivity():
    # kappa(0.5; p=3, kappa_lo=1, kappa_hi=1e6) = 125000.875
    assert O.conductivity(np.array([0.5]), 1.0, 1e6, 3)[0] == 125000.875


def test_kat_conductivity_rejects_bad_material():
    with pytest.raises(O.OracleError):
        O.conductivity(np.array([0.5]), 0.0, 1.0, 3)
    with pytest.raises(O.OracleError):
        O.conductivity(np.array([0.5]), 2.0, 1.0, 3)


def test_kat_two_cell_column():
    # 1x1x2 cells of unit size -> A = [[1,-1],[-1,1]] (Neumann);
    # Dirichlet T_D = 100 on z = 0 adds 2*kappa*area/h = 2 to a_00 and 200 to b_0.
    g = O.grid((1, 1, 2), (1.0, 1.0, 2.0))
    with pytest.raises(O.OracleError, match="no Dirichlet face"):
        O.System(g, np.ones(2), np.ones(2), [])
    s = O.System(g, np.ones(2), np.array([3.0, 5.0]), [(4, 0.0, 0.0, 1.0, 1.0, 100.0)])
    np.testing.assert_array_equal(s.matrix.toarray(), [[3.0, -1.0], [-1.0, 1.0]])
    np.testing.assert_array_equal(s.rhs, [200.0 + 3.0, 5.0])


def test_kat_local_basis_constant_kappa():
    # constant kappa: smallest eigenvalue 0 with a constant vector,
    # then the 3-fold cluster mu_1 (SURVEY.md §7 hard part 3).
    g = O.grid(16)
    h = O.hierarchy(g, 2, 2)
    vals, vecs = O.local_basis(h, np.ones(16 ** 3), 0, 4)
    assert abs(vals[0]) < 1e-10 * vals[1]
    v0 = vecs[0] / vecs[0][0]
    np.testing.assert_allclose(v0, np.ones_like(v0), rtol=1e-10)
    np.testing.assert_allclose(vals[1:], vals[1], rtol=1e-10)
    # M-orthonormal: Phi^T M Phi = I with M = kappa * vol
    vol = (1 / 16) ** 3
    np.testing.assert_allclose(vecs @ (vol * vecs.T), np.eye(4), atol=1e-10)


def test_kat_jacobi_diagonal_one_iteration():
    # Jacobi on a diagonal operator converges in one iteration:
    # a 1-cell-thick slab with Dirichlet on every cell's z-lo face and no x/y
    # couplings (nx = ny = 1 column has couplings; use nz = 1 plane of 1 cell).
    g = O.grid((1, 1, 1))
    s = O.System(g, np.array([2.0]), np.array([1.0]), [(4, 0.0, 0.0, 1.0, 1.0, 0.0)])
    m = O.Precond("jacobi", s)
    r = O.pcg(s, s.rhs, m, rtol=1e-12)
    assert r.converged and r.iterations == 1


def test_kat_galerkin_two_paths():
    # R A R^T computed as (R A) R^T equals R (A R^T)
    g = O.grid(16)
    kappa = inputs.conductivity(inputs.box_filter_design(16, 0.3), 1e-3)
    s = O.System(g, kappa, np.ones(16 ** 3), PATCH)
    m = O.Precond("mmg", s, O.hierarchy(g, 2, 2), fine_blocks="cell", coarse_blocks="cc")
    A, Rc, Ac = m.op(0), m.op(1), m.op(3)
    other = (Rc @ (A @ Rc.T)).toarray()
    np.testing.assert_allclose(Ac.toarray(), other, rtol=1e-11, atol=1e-11 * abs(other).max())


def test_preconditioner_symmetric_positive():
    # <M r1, r2> = <r1, M r2>, <r, M r> > 0
    g = O.grid(16)
    kappa = inputs.conductivity(inputs.box_filter_design(16, 0.3), 1e-6)
    s = O.System(g, kappa, np.ones(16 ** 3), PATCH)
    m = O.Precond("mmg", s, O.hierarchy(g, 2, 2), fine_blocks="cell", coarse_blocks="cc")
    rng = np.random.default_rng(3)
    r1, r2 = rng.standard_normal((2, 16 ** 3))
    a, b = m.apply(r1) @ r2, r1 @ m.apply(r2)
    assert abs(a - b) <= 1e-10 * abs(a)
    assert r1 @ m.apply(r1) > 0


# -------------------------------------------------------- dense eigensolver

@pytest.mark.parametrize("n,k", [(10, 3), (64, 4), (200, 8), (300, 16)])
def test_eigensolver_vs_numpy(n, k):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    a = a + a.T
    w, v = O.syev_smallest(a, k)
    we, ve = np.linalg.eigh(a)
    np.testing.assert_allclose(w, we[:k], atol=1e-12 * abs(we).max())
    np.testing.assert_allclose(a @ v, v * w, atol=1e-11 * abs(we).max())
    np.testing.assert_allclose(v.T @ v, np.eye(k), atol=1e-12)


def test_eigensolver_degenerate_cluster():
    # 8^3 Neumann Laplacian: eigenvalues 0, mu1 (x3), 2 mu1 (x3), 3 mu1
    n1 = 8
    T = np.diag(np.r_[1, 2 * np.ones(n1 - 2), 1]) - np.eye(n1, k=1) - np.eye(n1, k=-1)
    I = np.eye(n1)
    L = np.kron(np.kron(T, I), I) + np.kron(np.kron(I, T), I) + np.kron(np.kron(I, I), T)
    w, v = O.syev_smallest(L, 8)
    mu1 = 2 * (1 - np.cos(np.pi / 8))
    np.testing.assert_allclose(w, [0, mu1, mu1, mu1, 2 * mu1, 2 * mu1, 2 * mu1, 3 * mu1],
                               atol=1e-12)
    np.testing.assert_allclose(v.T @ v, np.eye(8), atol=1e-12)


# ---------------------------------------------------------------- generators

@pytest.mark.parametrize("n,r,vf", [(16, 2, 0.3), (24, 1, 0.3), ((8, 12, 16), 2, 0.2),
                                    (64, 2, 0.3)])
def test_product_generator_matches_oracle(n, r, vf):
    g = O.grid(n)
    a = O.box_filter_design(g, vf, passes=3, radius=r)
    b = inputs.box_filter_design(n, vf, passes=3, radius=r)
    np.testing.assert_array_equal(a, b)


def test_generator_solid_count_config0():
    # N=64, vf=0.3 -> exactly 78,644 solid cells
    assert inputs.box_filter_design(64, 0.3).sum() == 78644


def test_lcg_uniforms_match_reference_constants():
    # Lcg64 (rng.hpp:17-25) by direct recurrence
    s = 20240501
    ref = []
    for _ in range(5):
        s = (6364136223846793005 * s + 1442695040888963407) % 2 ** 64
        ref.append((s >> 11) * 2.0 ** -53)
    np.testing.assert_array_equal(inputs.lcg_uniforms(5, 20240501), ref)


# ------------------------------------------------------------ golden vectors

def _golden_cases():
    return sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.npz")) if "local_basis" not in p)


@pytest.mark.parametrize("path", _golden_cases(), ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_matches_reference_golden(path):
    z = np.load(path)
    n, ncc, sd = int(z["n"]), int(z["ncc"]), int(z["sd"])
    if n > 16 and str(z["kind"]) == "jacobi":
        pytest.skip("large jacobi golden is exercised on the GPU")
    rho = inputs.box_filter_design(n, float(z["vf"]), passes=int(z["passes"]),
                                   radius=int(z["radius"]))
    assert rho.sum() == z["rho_sum"]
    kappa = O.conductivity(rho, float(z["kmin"]))
    g = O.grid(n)
    s = O.System(g, kappa, np.ones(n ** 3), PATCH)
    np.testing.assert_array_equal(s.rhs, z["rhs"])
    np.testing.assert_array_equal(s.apply(z["apply_in"]), z["apply_out"])
    fb = str(z["fine_blocks"])
    cb = str(z["coarse_blocks"])
    m = O.Precond(str(z["kind"]), s, O.hierarchy(g, ncc, sd),
                  fine_blocks="cc" if fb == "None" else fb,
                  coarse_blocks="cc" if cb == "None" else cb)
    r = O.pcg(s, s.rhs, m, rtol=float(z["rtol"]), max_iterations=20000)
    assert r.converged
    assert r.iterations == int(z["iterations"])
    rel = np.linalg.norm(r.x - z["x"]) / np.linalg.norm(z["x"])
    assert rel <= 1e-9, rel
    np.testing.assert_allclose(r.residual_history, z["history"], rtol=1e-6)


def test_oracle_local_basis_matches_reference_golden():
    z = np.load(os.path.join(GOLDEN, "local_basis_n16_cell5.npz"))
    n = int(z["n"])
    kappa = O.conductivity(inputs.box_filter_design(n, 0.3), float(z["kmin"]))
    h = O.hierarchy(O.grid(n), int(z["ncc"]), int(z["sd"]))
    vals, vecs = O.local_basis(h, kappa, int(z["cid"]), 4)
    np.testing.assert_allclose(vals, z["values"], atol=1e-9 * abs(z["values"]).max())
    # same spans (M-orthonormal bases): singular values of the overlap = 1
    qa = np.linalg.qr(vecs.T)[0]
    qb = np.linalg.qr(z["vectors"].T)[0]
    np.testing.assert_allclose(np.linalg.svd(qa.T @ qb)[1], 1.0, atol=1e-9)


# ------------------------------------------------- the reference, run live

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_live_reference_assembly_bitwise():
    n = 16
    kappa = inputs.conductivity(inputs.box_filter_design(n, 0.3), 1e-6)
    A, rhs = O.ref_assemble(n, kappa, np.ones(n ** 3), PATCH)
    s = O.System(O.grid(n), kappa, np.ones(n ** 3), PATCH)
    B = s.matrix
    np.testing.assert_array_equal(A.indptr, B.indptr)
    np.testing.assert_array_equal(A.indices, B.indices)
    np.testing.assert_array_equal(A.data, B.data)
    np.testing.assert_array_equal(rhs, s.rhs)


@needs_ref
def test_live_reference_design_and_conductivity_bitwise():
    np.testing.assert_array_equal(O.ref_frozen_bench_design(16, 0.3),
                                  O.frozen_bench_design(O.grid(16), 0.3))
    x = np.random.default_rng(1).random(1000)
    np.testing.assert_array_equal(O.ref_conductivity(x, 1e-3), O.conductivity(x, 1e-3))


@needs_ref
@pytest.mark.parametrize("kind,fb,cb", [("jacobi", None, None), ("mmg", "cell", "cc"),
                                        ("mmg", None, None), ("mmg", "point", "cell"),
                                        ("two_grid", None, None), ("block_jacobi", None, None)])
def test_live_reference_solve(kind, fb, cb):
    n = 16
    kappa = inputs.conductivity(inputs.box_filter_design(n, 0.3), 1e-3)
    s = O.System(O.grid(n), kappa, np.ones(n ** 3), PATCH)
    r, _ = O.ref_solve(n, 2, 2, kappa, s.rhs, PATCH, kind, fb, cb, rtol=1e-8)
    m = O.Precond(kind, s, O.hierarchy(O.grid(n), 2, 2), fine_blocks=fb or "cc",
                  coarse_blocks=cb or "cc")
    o = O.pcg(s, s.rhs, m, rtol=1e-8)
    assert r.iterations == o.iterations
    assert np.linalg.norm(r.x - o.x) <= 1e-10 * np.linalg.norm(r.x)


@needs_ref
def test_lanczos_restatement_vs_reference():
    """Boxes above dense_threshold = 4096 cells (17^3 = 4913): the restated
    lanczos_smallest (coarse_space.cpp:61-198) against the reference's own,
    same Lcg64 start, same descending slot order"""
    n = 34
    kappa = inputs.conductivity(inputs.box_filter_design(n, 0.3), 1e-3)
    v_ref, V_ref = O.ref_local_basis_grid((n, n, n), 1, 2, kappa, 3, 4)
    v, V = O.local_basis(O.hierarchy(O.grid(n), 1, 2), kappa, 3, 4)
    assert np.all(np.diff(v_ref) <= 0) and np.all(np.diff(v) <= 0)
    np.testing.assert_allclose(v, v_ref, rtol=0, atol=1e-9 * v_ref.max())
    for a in range(4):
        cosang = abs(V[a] @ V_ref[a]) / (np.linalg.norm(V[a]) * np.linalg.norm(V_ref[a]))
        assert cosang >= 1 - 1e-9, (a, cosang)


@needs_ref
def test_live_reference_warm_start_x0():
    # pcg(..., x0) (solver.cpp:485,515-516): same x0 -> same iterations
    n = 16
    kappa = inputs.conductivity(inputs.box_filter_design(n, 0.3), 1e-3)
    s = O.System(O.grid(n), kappa, np.ones(n ** 3), PATCH)
    x0 = np.random.default_rng(5).random(n ** 3)
    r, _ = O.ref_solve(n, 2, 2, kappa, s.rhs, PATCH, "jacobi", rtol=1e-8, x0=x0)
    o = O.pcg(s, s.rhs, O.Precond("jacobi", s), rtol=1e-8, x0=x0)
    assert r.iterations == o.iterations
    np.testing.assert_array_equal(r.x, o.x)


def test_interpolate_design_mean_preserving():
    # grid.cpp:220-241: piecewise-constant prolongation preserves the mean
    lo = np.random.default_rng(2).random(8 ** 3)
    hi = O.interpolate_design(lo, 8, 16)
    assert hi.size == 16 ** 3 and abs(hi.mean() - lo.mean()) < 1e-15
    assert hi[0] == lo[0] and hi[1] == lo[0] and hi[2] == lo[1]


# ---------------------------------------------------------- sensitivity (§8(f))

@needs_ref
@pytest.mark.parametrize("n,p,f0", [(8, 3, 1.0), ((6, 8, 10), 1, 0.5), (12, 2, 0.0)])
def test_sensitivity_restatement_bitwise_vs_reference(n, p, f0):
    nx, ny, nz = (n, n, n) if np.isscalar(n) else n
    m = nx * ny * nz
    rng = np.random.default_rng(30)
    rho = rng.random(m)
    rho[rng.random(m) < 0.2] = 0.0  # dk == 0 cells (p >= 2)
    t, u = rng.standard_normal(m), rng.standard_normal(m)
    patches = [(4, 0.2, 0.2, 0.8, 0.8, 1.5), (1, 0.0, 0.0, 0.5, 1.0, -0.5)]
    ref = O.ref_sensitivity(n, rho, t, u, 1e-3, 1.0, f0, p, patches)
    mine = O.sensitivity(n, rho, t, u, 1e-3, 1.0, f0, p, patches)
    np.testing.assert_array_equal(mine, ref)


@needs_ref
def test_sensitivity_matches_finite_differences():
    """d(mean T)/d rho_c from the adjoint formula vs central differences of
    the exactly solved system (grid 6^3, dense solves)."""
    n, klo, f0, p = 6, 1e-2, 1.0, 3
    m = n ** 3
    rng = np.random.default_rng(31)
    rho = 0.2 + 0.6 * rng.random(m)
    patches = O.bottom_center_patch(side=0.5)

    def mean_t(r):
        kap = inputs.conductivity(r, klo)
        src = f0 * (1.0 - r ** p)  # heat_source (material.cpp:52-58)
        s = O.System(O.grid(n), kap, src, patches)
        A = s.matrix.toarray()
        return np.linalg.solve(A, s.rhs), A

    t, A = mean_t(rho)
    u = np.linalg.solve(A.T, np.full(m, 1.0 / m))  # adjoint_rhs (optim.cpp:16-19)
    grad = O.ref_sensitivity(n, rho, t, u, klo, 1.0, f0, p, patches)
    for c in rng.choice(m, 6, replace=False):
        h = 1e-6
        rp, rm = rho.copy(), rho.copy()
        rp[c] += h
        rm[c] -= h
        fd = (mean_t(rp)[0].mean() - mean_t(rm)[0].mean()) / (2 * h)
        assert abs(fd - grad[c]) <= 1e-5 * abs(grad[c]) + 1e-12


def test_interpolate_design_matches_oracle():
    from paper_2410_06850_b200 import GridSpec, interpolate_design
    rng = np.random.default_rng(5)
    lo = rng.random(4 * 6 * 8)
    hi = interpolate_design(lo, GridSpec(4, 6, 8), GridSpec(8, 12, 24))
    np.testing.assert_array_equal(hi, O.interpolate_design(lo, (4, 6, 8), (8, 12, 24)))


def test_tree_segments_deterministic_and_rooted():
    """configs[4]'s tree generator (inputs.tree_segments; the device builds
    the same list in csrc/abi.cu): root at the z = 0 face centre heading +z,
    2^depth - 1 segments, children start where their parent ends."""
    from paper_2410_06850_b200 import inputs
    s = inputs.tree_segments(20240501, depth=6)
    assert s.shape == (63, 7)
    np.testing.assert_array_equal(s, inputs.tree_segments(20240501, depth=6))
    assert tuple(s[0, :3]) == (0.5, 0.5, 0.0) and s[0, 3:5].tolist() == [0.5, 0.5]
    for k in range(1, 63):
        parent = (k - 1) // 2
        np.testing.assert_array_equal(s[k, :3], s[parent, 3:6])
    assert not np.array_equal(s, inputs.tree_segments(7, depth=6))
