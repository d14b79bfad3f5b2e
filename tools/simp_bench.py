"""BASELINE configs[2] on the device: 128^3, SIMP loop of 10 design
iterations from uniform rho = 0.3, density filter r = 1.5, OC move 0.2,
kmin = 1e-6, each solve warm-started from the previous one. Prints one JSON
line per design iteration and a summary (wall time per design iteration,
set-up / LS1 / LS2 shares).

    python tools/simp_bench.py [--n 128] [--iters 10]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--out", default=None)
a = ap.parse_args()
n = a.n
ncc = n // 16
c = Context(GridSpec(n, n, n), ncc, 2)
c.set_design(np.full(n ** 3, 0.3), 1e-6, 1.0, 3, BoundarySpec.bottom_center_patch(1, 1, 0.2, 0))
c.simp_init(volfrac=0.3, rmin=1.5, move=0.2, kappa_lo=1e-6, rtol=1e-8)
reps = []
t0 = time.perf_counter()
for _ in range(a.iters):
    r = c.simp_step()
    reps.append(r)
    print(json.dumps(r), flush=True)
wall = time.perf_counter() - t0
summary = {
    "workload": f"BASELINE configs[2]: {n}^3, {a.iters} SIMP iterations (filter r=1.5, OC move 0.2, "
                "kmin 1e-6, warm-started LS1/LS2, rtol 1e-8)",
    "seconds_per_design_iteration": wall / a.iters,
    "setup_s": sum(r["setup_seconds"] for r in reps) / a.iters,
    "ls1_s": sum(r["ls1_seconds"] for r in reps) / a.iters,
    "ls2_s": sum(r["ls2_seconds"] for r in reps) / a.iters,
    "ls1_iterations": [r["ls1_iterations"] for r in reps],
    "ls2_iterations": [r["ls2_iterations"] for r in reps],
    "cost": [r["cost"] for r in reps],
}
print(json.dumps(summary))
if a.out:
    with open(a.out, "w") as f:
        json.dump(summary, f, indent=1)
