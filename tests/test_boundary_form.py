"""The boundary form of the V-cycle's fine steps, checked on the
CPU with the oracle's assembled matrix: with one exact block solve per brick
(r1_I = A_II^{-1} r_I),

  R_c (r - A r1)        ==  sum over brick faces of Phi_I(c_f) T_f r1_nb(f)
  r2 + S(r - A r2)      ==  S(r + t),  t_c = sum over surface faces of T_f r2_nb(f)

for any per-brick basis Phi (r2 = r1 + R_c^T ec). k_restrict_bnd and
k_post_bnd compute the right-hand sides; the reference computes the left
(solver.cpp:285-289, 322-333). Test infrastructure: the oracle is the checker.
"""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle as O
from paper_2410_06850_b200 import inputs


def _bricks(n, c):
    nb = n // c
    out = []
    for bk in range(nb):
        for bj in range(nb):
            for bi in range(nb):
                loc = np.arange(c ** 3)
                i, j, k = loc % c, (loc // c) % c, loc // (c * c)
                out.append((bi * c + i) + n * ((bj * c + j) + n * (bk * c + k)))
    return out


@pytest.mark.parametrize("n,c,kmin", [(16, 4, 1e-2), (16, 8, 1e-3), (24, 4, 1e-1)])
def test_boundary_form_matches_literal_vcycle_steps(n, c, kmin):
    g = O.grid(n)
    rho = inputs.box_filter_design(n, 0.3)
    kappa = inputs.conductivity(rho, kmin)
    A = O.System(g, kappa, np.ones(n ** 3), O.bottom_center_patch()).matrix.tocsr()
    bricks = _bricks(n, c)
    owner = np.empty(n ** 3, dtype=np.int64)
    for b, cells in enumerate(bricks):
        owner[cells] = b
    rng = np.random.default_rng(4)
    L = 4
    phi = [rng.standard_normal((len(cells), L)) for cells in bricks]
    lu = [spla.splu(A[cells][:, cells].tocsc()) for cells in bricks]

    def S(v):  # exact block-Jacobi, one block per brick
        out = np.empty_like(v)
        for cells, f in zip(bricks, lu):
            out[cells] = f.solve(v[cells])
        return out

    def surface_sum(v):  # t_c = sum over faces to other bricks of T_f v_nb = -A_{c,nb} v_nb
        Acoo = A.tocoo()
        cross = owner[Acoo.row] != owner[Acoo.col]
        off = sp.csr_matrix((Acoo.data[cross], (Acoo.row[cross], Acoo.col[cross])), shape=A.shape)
        return -(off @ v)

    r = rng.standard_normal(n ** 3)
    r1 = S(r)
    # restriction
    lit = np.concatenate([p.T @ (r - A @ r1)[cells] for p, cells in zip(phi, bricks)])
    t1 = surface_sum(r1)
    bnd = np.concatenate([p.T @ t1[cells] for p, cells in zip(phi, bricks)])
    assert np.linalg.norm(lit - bnd) <= 1e-10 * np.linalg.norm(lit)
    # only surface cells carry the pre-smoothed residual
    interior = np.ones(n ** 3, dtype=bool)
    interior[np.nonzero(surface_sum(np.ones(n ** 3)) != 0)[0]] = False
    assert np.abs(t1[interior]).max() == 0.0
    # post-smoothing
    ec = rng.standard_normal(len(bricks) * L)
    r2 = r1.copy()
    for b, (p, cells) in enumerate(zip(phi, bricks)):
        r2[cells] += p @ ec[b * L:(b + 1) * L]
    z_lit = r2 + S(r - A @ r2)
    z_bnd = S(r + surface_sum(r2))
    assert np.linalg.norm(z_lit - z_bnd) <= 1e-10 * np.linalg.norm(z_lit)
