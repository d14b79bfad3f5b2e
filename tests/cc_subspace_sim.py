"""Design note for the large-element cc eigensolver (csrc/coarse_large.cu):
numpy model of its subspace iteration (shifted inverse, two SVQB passes,
Rayleigh-Ritz on H) run on the oracle's projected matrices H = Rc S_E Rc^T of a
32^3 / sd = 4 hierarchy, sweeping the shift. Prints the steps to reach a
1e-13 residual and the best residual reached. Not collected by pytest.

    python tests/cc_subspace_sim.py
"""
import os
import sys

import numpy as np

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
sys.path.insert(0, os.path.join(R, "oracle"))
import oracle as O  # noqa: E402
from paper_2410_06850_b200 import inputs  # noqa: E402
n = 32
def getH(kmin, radius):
    rho = inputs.box_filter_design(n, 0.3, radius=radius)
    kappa = inputs.conductivity(rho, kmin)
    s = O.System(O.grid(n), kappa, np.ones(n ** 3), O.bottom_center_patch())
    m = O.Precond("mmg", s, O.hierarchy(O.grid(n), 1, 4), fine_blocks="cell", coarse_blocks="cc")
    A = s.matrix.tocsr(); Rc = m.op(1).toarray()
    off = A.copy(); off.setdiag(0); off.eliminate_zeros()
    S = off.toarray(); S -= np.diag(S.sum(1))
    H = Rc @ S @ Rc.T; return 0.5 * (H + H.T)
def svqb(Y):
    G = Y.T @ Y; d = 1 / np.sqrt(np.maximum(np.diag(G), 1e-300)); G = d[:, None] * G * d[None, :]
    lam, W = np.linalg.eigh(G); return Y @ (d[:, None] * W / np.sqrt(np.maximum(lam, 1e-24)))
def run(H, srel, K=16, lcc=8, tol=1e-13):
    q = H.shape[0]; md = H.diagonal().max()
    Hs = np.linalg.inv(H + srel * md * np.eye(q))
    rng = np.random.default_rng(0)
    Y = rng.uniform(-.5, .5, (q, K)); Y[:, 0] = 1
    best = 1
    for it in range(100):
        X = svqb(svqb(Y))
        T = X.T @ H @ X; T = 0.5 * (T + T.T); th, W = np.linalg.eigh(T); X = X @ W
        res = (np.linalg.norm(H @ X - X * th, axis=0)[:lcc] / md).max()
        best = min(best, res)
        if res < tol: return it + 1, res
        Y = Hs @ X
    return 100, best
for kmin, radius in [(1e-3, 2), (1e-6, 2), (1e-6, 4)]:
    H = getH(kmin, radius); w = np.linalg.eigvalsh(H) / H.diagonal().max()
    print(f"kmin {kmin} r {radius}: lam8 {w[7]:.2e} lam17 {w[16]:.2e}")
    for srel in [1e-10, 1e-8, 1e-6, 1e-5, 1e-4, 1e-3]:
        print("   sigma", srel, run(H, srel))
