"""Repeat the generic local eigensolver on one shape in one process, after
other contexts, and report the iteration counts (state / race diagnosis)."""
import sys, os
import numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "oracle"))
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs
BC = BoundarySpec.bottom_center_patch(1, 1, 0.2, 0)
def run(shape, ncc, sd, kmin, opts, kind="mmg"):
    rho = inputs.box_filter_design(shape, 0.3)
    kappa = inputs.conductivity(rho, kmin)
    c = Context(GridSpec(*shape), ncc, sd)
    c.set_conductivity(kappa, BC)
    c.setup(kind, opts)
    if kind in ("mmg", "two_grid"):
        phi, ev, it = c.local_bases()
        print(shape, kind, "nonconv", int((it < 0).sum()), "of", len(it), "iters", it[:12], flush=True)
    c.close()
shape0 = (24, 16, 32)
for rep in range(3):
    run(shape0, (2, 2, 2), 2, 1e-6, MmgOptions(fine_blocks="coarse_cell"))
for sh, ncc in [((24, 24, 24), (4, 4, 4)), ((16, 16, 16), (4, 4, 4)), ((20, 12, 16), (2, 3, 2))]:
    run(sh, ncc, 2, 1e-3, MmgOptions(fine_blocks="coarse_cell"))
    run(sh, ncc, 2, 1e-3, MmgOptions(fine_blocks="cc"))
for rep in range(3):
    run(shape0, (2, 2, 2), 2, 1e-6, MmgOptions(fine_blocks="coarse_cell"))
