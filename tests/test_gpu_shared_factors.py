"""Shared fine-smoother factors: interior bricks whose cells
and face halo carry one conductivity k share the canonical factor A_hat^-1
of a unit-conductivity brick, scaled by 1 / face_t(k, k) (A_II = face_t(k, k)
A_hat); bricks of one conductivity inside get their local bases in closed
form. Checked against the oracle's exact per-coarse-cell blocks and
eigensolver, and against the unshared paths (TMG_G_SHARE=0,
TMG_EIG_SHARE=0)."""
import os

import numpy as np
import pytest

import oracle as O
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs

pytestmark = pytest.mark.gpu
BC = BoundarySpec.bottom_center_patch(1.0, 1.0, 0.2, 0.0)
CELL = MmgOptions(fine_blocks="coarse_cell")


def iters_close(a, b):
    return abs(a - b) <= max(1, int(0.1 * b))


def setup(ctx, share, opts=CELL):
    old = os.environ.get("TMG_G_SHARE")
    os.environ["TMG_G_SHARE"] = "1" if share else "0"
    try:
        ctx.setup("mmg", opts)
    finally:
        if old is None:
            del os.environ["TMG_G_SHARE"]
        else:
            os.environ["TMG_G_SHARE"] = old


@pytest.mark.parametrize("n,ncc,sd,kmin", [(64, 4, 2, 1e-6), (64, 2, 4, 1e-3)])
def test_shared_factors_match_oracle_and_unshared(n, ncc, sd, kmin):
    rho = inputs.box_filter_design(n, 0.2, radius=4)
    kappa = inputs.conductivity(rho, kmin)
    c = Context(GridSpec(n, n, n), ncc, sd)
    c.set_conductivity(kappa, BC)
    b = c.assemble_rhs(np.ones(n ** 3))
    setup(c, True, MmgOptions(fine_blocks="coarse_cell", num_cc_basis=8 if sd == 2 else 12))
    slots, bricks = c.fine_factor_slots()
    assert bricks == (n // 8) ** 3 and slots < 0.9 * bricks, (slots, bricks)
    rs = c.pcg(b, rtol=1e-8)
    setup(c, False, MmgOptions(fine_blocks="coarse_cell", num_cc_basis=8 if sd == 2 else 12))
    assert c.fine_factor_slots() == (bricks, bricks)
    ru = c.pcg(b, rtol=1e-8)
    assert rs.report.converged and ru.report.converged
    assert abs(rs.report.iterations - ru.report.iterations) <= 1
    assert np.linalg.norm(rs.x - ru.x) <= 1e-8 * np.linalg.norm(ru.x)
    s = O.System(O.grid(n), kappa, np.ones(n ** 3), O.bottom_center_patch())
    m = O.Precond("mmg", s, O.hierarchy(O.grid(n), ncc, sd), lcc=8 if sd == 2 else 12,
                  fine_blocks="cell", coarse_blocks="cc")
    ref = O.pcg(s, s.rhs, m, rtol=1e-8)
    assert iters_close(rs.report.iterations, ref.iterations), (rs.report.iterations, ref.iterations)
    assert np.linalg.norm(rs.x - ref.x) <= 1e-6 * np.linalg.norm(ref.x)


def test_shared_factor_preconditioner_is_the_exact_block_solve():
    """One V-cycle with shared factors equals the unshared one to rounding."""
    n = 32
    kappa = np.full(n ** 3, 0.5)
    kappa[: n ** 3 // 3] = 1e-3  # two uniform slabs of conductivity
    c = Context(GridSpec(n, n, n), 2, 2)
    c.set_conductivity(kappa, BC)
    r = np.random.default_rng(3).standard_normal(n ** 3)
    setup(c, True)
    slots, bricks = c.fine_factor_slots()
    assert slots < bricks
    zs = c.apply_preconditioner(r)
    setup(c, False)
    zu = c.apply_preconditioner(r)
    assert np.linalg.norm(zs - zu) <= 1e-12 * np.linalg.norm(zu)


def test_shared_local_eigensolves_match_individual():
    """Bricks of one conductivity inside take closed-form bases (separable
    DCT-II modes, M-orthonormal); they match solving every brick
    (TMG_EIG_SHARE=0) and the oracle's dense eigensolver."""
    n = 32
    rho = inputs.box_filter_design(n, 0.2, radius=4)
    kappa = inputs.conductivity(rho, 1e-3)
    c = Context(GridSpec(n, n, n), 2, 2)
    c.set_conductivity(kappa, BC)
    c.setup("mmg", CELL)
    ps, es, its = c.local_bases()
    old = os.environ.get("TMG_EIG_SHARE")
    os.environ["TMG_EIG_SHARE"] = "0"
    try:
        c.setup("mmg", CELL)
    finally:
        if old is None:
            del os.environ["TMG_EIG_SHARE"]
        else:
            os.environ["TMG_EIG_SHARE"] = old
    pu, eu, _ = c.local_bases()
    np.testing.assert_allclose(es, eu, rtol=1e-7, atol=1e-9 * eu.max())
    k3 = kappa.reshape(n, n, n)
    uniform = [b for b in range(64)
               if np.ptp(k3[8 * (b // 16):8 * (b // 16) + 8, 8 * (b // 4 % 4):8 * (b // 4 % 4) + 8,
                            8 * (b % 4):8 * (b % 4) + 8]) == 0]
    assert len(uniform) >= 2
    h = O.hierarchy(O.grid(n), 2, 2)
    for b in uniform[:3] + [0, 37]:
        qa, _ = np.linalg.qr(ps[b].T)
        qb, _ = np.linalg.qr(pu[b].T)
        assert np.linalg.svd(qa.T @ qb)[1].min() >= 1 - 1e-8, b
        vals, vecs = O.local_basis(h, kappa, b, 4)
        np.testing.assert_allclose(es[b], vals, rtol=1e-6, atol=1e-9 * vals.max())
        # M-orthonormal in the brick's own mass (the scaling is exact)
        m = kappa[np.array(O_cells(n, b))] / n ** 3
        g = (ps[b] * m) @ ps[b].T
        np.testing.assert_allclose(g, np.eye(4), atol=1e-8)


def O_cells(n, b):
    """x-fastest global ids of brick b's cells (cells_of_coarse order)"""
    nb = n // 8
    bi, bj, bk = b % nb, (b // nb) % nb, b // (nb * nb)
    return [(8 * bi + i) + n * ((8 * bj + j) + n * (8 * bk + k))
            for k in range(8) for j in range(8) for i in range(8)]


def test_search_from_kappa_is_bitwise_the_coefficient_search():
    """k_search_kappa (coefficients recomputed from kappa, 40 B/cell) and
    k_search (stored coefficients, 64 B/cell) give bitwise the same PCG
    (TMG_SEARCH_KAPPA is read once per process: two processes)."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs\n"
        "n = 32; kappa = inputs.conductivity(inputs.box_filter_design(n, 0.3), 1e-6)\n"
        "c = Context(GridSpec(n, n, n), 2, 2)\n"
        "c.set_conductivity(kappa, BoundarySpec.bottom_center_patch(1, 1, 0.2, 0))\n"
        "c.setup('mmg', MmgOptions(fine_blocks='coarse_cell'))\n"
        "r = c.pcg(c.assemble_rhs(np.ones(n ** 3)), rtol=1e-10)\n"
        "sys.stdout.write(r.x.tobytes().hex()[:4000] + ' ' + r.report.residual_history.tobytes().hex())\n"
    ) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = []
    for v in ("1", "0"):  # kappa-based (opt-in) and the default
        env = dict(os.environ, TMG_SEARCH_KAPPA=v)
        out.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                  text=True, check=True).stdout)
    assert out[0] == out[1]
