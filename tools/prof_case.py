"""One MMG-PCG case for profiling (default: BASELINE configs[1], 128^3, kmin 1e-6)."""
import argparse, os, sys
import numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--ncc", type=int, default=8)
ap.add_argument("--sd", type=int, default=2)
ap.add_argument("--kmin", type=float, default=1e-6)
ap.add_argument("--kind", default="mmg")
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--setups", type=int, default=1)
ap.add_argument("--slabs", type=int, default=1)
ap.add_argument("--lcc", type=int, default=8)
a = ap.parse_args()
n = a.n
rho = inputs.box_filter_design(n, 0.3)
kappa = inputs.conductivity(rho, a.kmin)
ctx = Context(GridSpec(n, n, n), a.ncc, a.sd, slabs=a.slabs)
ctx.set_conductivity(kappa, BoundarySpec.bottom_center_patch(1, 1, 0.2, 0))
b = ctx.assemble_rhs(np.ones(n ** 3))
import time
for _ in range(a.setups):
    t0 = time.perf_counter()
    ctx.setup(a.kind, MmgOptions(num_cc_basis=a.lcc, fine_blocks="coarse_cell"))
    print("setup wall ms %.2f" % ((time.perf_counter() - t0) * 1e3))
ctx.upload_rhs(b)
for _ in range(a.solves):
    rep = ctx.solve_resident(1e-8, 5000)
print("iterations", rep.iterations, "solve ms", rep.solve_seconds * 1e3)
if os.environ.get("TMG_PROFILE") and a.slabs == 1:
    prof = ctx.profile_solve(1e-8, 5000)
    for k, (ms, cnt) in prof.items():
        if cnt:
            print("  %-12s %8.3f ms total %5d launches %8.1f us/launch" % (k, ms, cnt, 1e3 * ms / cnt))
