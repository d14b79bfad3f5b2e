"""Diagnostics for the generic local eigensolver: iterations, eigenvalues and
spans against the oracle on one generic shape (build variant with
-DTMG_EIG_DEBUG for per-step traces of brick 0)."""
import sys, os
import numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "oracle"))
import oracle as O
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs
shape, ncc, sd = (24, 16, 32), (2, 2, 2), 2
rho = inputs.box_filter_design(shape, 0.3)
kappa = inputs.conductivity(rho, 1e-6)
c = Context(GridSpec(*shape), ncc, sd)
c.set_conductivity(kappa, BoundarySpec.bottom_center_patch(1, 1, 0.2, 0))
c.setup("mmg", MmgOptions(fine_blocks="coarse_cell"))
phi, ev, it = c.local_bases()
print("iters", it[:16])
h = O.hierarchy(O.grid(shape), ncc, sd)
for cid in range(4):
    vals, vecs = O.local_basis(h, kappa, cid, 4)
    qa, _ = np.linalg.qr(phi[cid].T); qb, _ = np.linalg.qr(vecs.T)
    print(cid, "gpu", ev[cid], "orc", vals, "cos", np.linalg.svd(qa.T @ qb)[1].min())
