"""Per-kernel device times of a profiled solve (tmg_profile_solve: events
around every phase) at BASELINE configs[K]; TMG_LIB selects a library build
(A/B of build variants)."""
import argparse, os, sys
import numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--maxit", type=int, default=12)
a = ap.parse_args()
cfg = dict(inputs.CONFIGS[a.config])
n = cfg["n"]
c = Context(GridSpec(n, n, n), cfg["ncc"], cfg["sd"])
c.set_design_generated(cfg["vf"], cfg["kmin"], 1.0, 3, BoundarySpec.bottom_center_patch(1, 1, 0.2, 0),
                       passes=cfg["passes"], radius=cfg["radius"])
b = c.assemble_rhs(np.ones(n ** 3))
c.setup("mmg", MmgOptions(fine_blocks="coarse_cell", num_cc_basis=cfg.get("lcc", 8)))
c.upload_rhs(b)
prof = c.profile_solve(1e-8, a.maxit)
for k, (ms, cnt) in prof.items():
    if cnt:
        print("  %-12s %8.3f ms total %5d launches %8.1f us/launch" % (k, ms, cnt, 1e3 * ms / cnt))
