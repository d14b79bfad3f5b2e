"""The reference's design loop (topmg::optimize with MMA) on the device at
BASELINE configs[2]'s size: 128^3, vstar 0.3, kmin 1e-6, 10 MMA iterations,
rtol 1e-8. Reference semantics (cold set-up, solves from zero) and the
warm-started variant; one JSON line each with per-iteration set-up / LS1 / LS2
and the wall time per design iteration.

    python tools/optim_bench.py [--n 128] [--iters 10] [--out file.json]
"""
import argparse
import json
import os
import sys
import time

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
from paper_2410_06850_b200 import (BoundarySpec, GridSpec, MaterialModel, OptimConfig,  # noqa: E402
                                   optimize)

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--out", default=None)
a = ap.parse_args()
n = a.n
# warm-up: CUDA context, module loading, buffer pools (not timed)
optimize(OptimConfig(vstar=0.3, schedule=[GridSpec(n, n, n)], iters_per_level=[1],
                     ncc=(n // 16,) * 3, sd=2, rtol=1e-8),
         MaterialModel(1e-6, 1.0, 1.0, 3), BoundarySpec.bottom_center_patch(1, 1, 0.2, 0))
rows = []
for warm in (False, True):
    def run(iters):
        cfg = OptimConfig(vstar=0.3, schedule=[GridSpec(n, n, n)], iters_per_level=[iters],
                          convergence_dx=0.0, ncc=(n // 16,) * 3, sd=2, rtol=1e-8, warm_start=warm)
        t0 = time.perf_counter()
        r = optimize(cfg, MaterialModel(1e-6, 1.0, 1.0, 3),
                     BoundarySpec.bottom_center_patch(1, 1, 0.2, 0))
        return r, time.perf_counter() - t0
    _, wall1 = run(1)
    res, wall = run(a.iters)
    tr = res.trajectory
    row = {"workload": f"topmg::optimize semantics (MMA, 1 level), {n}^3, vstar 0.3, kmin 1e-6, "
                       f"{a.iters} iterations, rtol 1e-8",
           "warm_start": warm, "failed": res.failed,
           # wall of one optimize() call / iterations: includes the context's
           # creation, the final evaluation solve and tmg_destroy (~0.45 s)
           "seconds_per_design_iteration": wall / max(1, len(tr)),
           # marginal cost of a design iteration: (wall(iters) - wall(1)) / (iters - 1)
           "marginal_seconds_per_design_iteration": (wall - wall1) / max(1, len(tr) - 1),
           "setup_s": sum(t.setup_seconds for t in tr) / len(tr),
           "ls1_s": sum(t.ls1_seconds for t in tr) / len(tr),
           "ls2_s": sum(t.ls2_seconds for t in tr) / len(tr),
           "ls1_iterations": [t.ls1_iters for t in tr], "ls2_iterations": [t.ls2_iters for t in tr],
           "cost": [t.cost for t in tr], "final_cost": res.final_cost}
    rows.append(row)
    print(json.dumps(row), flush=True)
if a.out:
    with open(a.out, "w") as f:
        json.dump(rows, f, indent=1)
