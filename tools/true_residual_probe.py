"""Diagnostics: recurrence vs true residual of the device PCG, and residual
replacement restarts (configs[3] generator/hierarchy at n^3).

    python tools/true_residual_probe.py [--n 256] [--restarts 6]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--restarts", type=int, default=6)
ap.add_argument("--cfg", type=int, default=3)
a = ap.parse_args()
cfg = inputs.CONFIGS[a.cfg]
n = a.n
ncc = n // (8 * cfg["sd"])
ctx = Context(GridSpec(n, n, n), ncc, cfg["sd"])
bc = BoundarySpec.bottom_center_patch(1, 1, 0.2, 0)
ctx.set_design_generated(cfg["vf"], cfg["kmin"], 1.0, 3, bc, passes=cfg["passes"],
                         radius=cfg["radius"])
b = ctx.assemble_rhs(np.ones(n ** 3))
ctx.setup("mmg", MmgOptions(num_cc_basis=cfg.get("lcc", 8, fine_blocks="coarse_cell")))
bn = np.linalg.norm(b)
r = ctx.pcg(b, rtol=1e-8)
x = r.x
print(f"n={n}: {r.report.iterations} it, recurrence {r.report.residual_history[-1]:.3e}, "
      f"true {np.linalg.norm(b - ctx.apply_operator(x)) / bn:.3e}, |x|max {np.abs(x).max():.3e}")
print("history:", " ".join(f"{h:.2e}" for h in r.report.residual_history))
for k in range(a.restarts):
    r = ctx.pcg(b, rtol=1e-8, x0=x)
    x = r.x
    t = np.linalg.norm(b - ctx.apply_operator(x)) / bn
    print(f"restart {k}: {r.report.iterations} it, reported {r.report.final_relative_residual:.3e}"
          f", true {t:.3e}; history {' '.join(f'{h:.2e}' for h in r.report.residual_history)}")
ctx.upload_rhs(b)
v = ctx.solve_resident(1e-8, 10000, true_residual=True)
xv = ctx.download_solution()
print("solve_resident(true_residual):", v.iterations, v.restarts, v.status,
      v.final_relative_residual, np.linalg.norm(b - ctx.apply_operator(xv)) / bn,
      "FP64 floor eps|A||x|/|b|:", ctx.residual_floor(xv, b))
