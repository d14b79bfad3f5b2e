"""Rounding sensitivity of block_jacobi PCG at contrast 1e6 (32^3, c = 8,
sd = 2): the reference's own preconditioner (oracle) inside a restatement of
pcg() (solver.cpp:483-575), with z perturbed by relative noise of size eps.
Measured: 286 iterations unperturbed; 205-286 at eps = 1e-14 and 1e-12; so
an iteration count within 10% is not a reproducible target for this case
(tests/test_gpu_parity.py::test_block_jacobi_vs_oracle). Not collected by
pytest.

    python tests/bj_sensitivity.py
"""
import os
import sys

import numpy as np

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
sys.path.insert(0, os.path.join(R, "oracle"))
import oracle as O  # noqa: E402
from paper_2410_06850_b200 import inputs  # noqa: E402
n, kmin = 32, 1e-6
rho = inputs.box_filter_design(n, 0.3, radius=2); kappa = inputs.conductivity(rho, kmin)
s = O.System(O.grid(n), kappa, np.ones(n ** 3), O.bottom_center_patch())
m = O.Precond("block_jacobi", s, O.hierarchy(O.grid(n), 2, 2), fine_blocks="cc")
A = s.matrix.tocsr(); b = s.rhs
def pcg(prec, rtol=1e-8, maxit=5000):
    x = np.zeros_like(b); r = b.copy(); bn = np.linalg.norm(b)
    z = prec(r); p = z.copy(); rz = r @ z
    for it in range(1, maxit + 1):
        q = A @ p; a = rz / (p @ q); x += a * p; r -= a * q
        if np.linalg.norm(r) / bn <= rtol: return it
        z = prec(r); rz2 = r @ z; p = z + (rz2 / rz) * p; rz = rz2
    return maxit
print("oracle pcg", O.pcg(s, b, m, rtol=1e-8).iterations)
print("numpy pcg, exact z", pcg(m.apply))
rng = np.random.default_rng(0)
for eps in [1e-14, 1e-12, 1e-10, 1e-8]:
    its = [pcg(lambda r: m.apply(r) * (1 + eps * rng.standard_normal(r.size))) for _ in range(3)]
    print("perturbed", eps, its)
