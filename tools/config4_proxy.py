"""configs[4] single-GPU proxy: one rank's slab of the 1024^3 tree problem.

BASELINE configs[4] is 1024^3 cells on 8 B200 in z-slabs of 1024 x 1024 x 128.
This runs one such slab on one GPU as a standalone problem: the bottom slab
of the global 1024^3 tree design (tmg_set_design_tree generates the whole
design on the device, global_n = 1024^3, and keeps the slab), cells of the
global size (extent 1 x 1 x 0.125), the
Dirichlet patch of the global problem on its z = 0 face, Neumann on top
(where the distributed run has the next slab's ghost layer). It measures
what one GPU of the 8-GPU run holds and moves: device memory, set-up time,
time per PCG iteration and MDoF*iter/s. Its iteration count is the slab
problem's, not the global one's.

    python tools/config4_proxy.py [--nz 128] [--out f.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--nz", type=int, default=128)
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg = inputs.CONFIGS[4]
n, nz, sd = a.n, a.nz, cfg["sd"]
ncc = (n // (8 * sd), n // (8 * sd), nz // (8 * sd))
lz = nz / n
c = Context(GridSpec(n, n, nz, 1.0, 1.0, lz), ncc, sd)
bc = BoundarySpec.bottom_center_patch(1, 1, 0.2, 0)
t0 = time.perf_counter()
# the global 1024^3 design (its filter and volume-fraction threshold), of
# which this context keeps the bottom slab
c.set_design_tree(cfg["vf"], cfg["kmin"], 1.0, 3, bc, passes=cfg["passes"], radius=cfg["radius"],
                  dom=(1.0, 1.0, 1.0), global_n=(n, n, n), z0=0)
t_gen = time.perf_counter() - t0
b = c.assemble_rhs(np.ones(n * n * nz))
opts = MmgOptions(num_cc_basis=cfg["lcc"], fine_blocks="coarse_cell")
t0 = time.perf_counter()
c.setup("mmg", opts)
t_setup_cold = time.perf_counter() - t0
t0 = time.perf_counter()
c.setup("mmg", opts)
t_setup = time.perf_counter() - t0
c.upload_rhs(b)
reps = [c.solve_resident(1e-8, 20000) for _ in range(a.solves)]
rep = reps[-1]
x = c.download_solution()
bn = np.linalg.norm(b)
true_rel = float(np.linalg.norm(b - c.apply_operator(x)) / bn)
prof = c.profile_solve(1e-8, 20000)
out = {
    "workload": f"BASELINE configs[4] single-GPU proxy: one z-slab {n}x{n}x{nz} of the {n}^3 "
                f"tree design (vf {cfg['vf']}, radius {cfg['radius']}, kmin {cfg['kmin']:g}), "
                "rtol 1e-8, standalone slab problem",
    "hierarchy": f"c=8 sd={sd} ncc={ncc} L_c=4 L_cc={cfg['lcc']} (n_cc={np.prod(ncc) * cfg['lcc']})",
    "cells": n * n * nz, "iterations": rep.iterations, "converged": rep.converged,
    "solve_s": rep.solve_seconds, "setup_s": t_setup, "setup_cold_s": t_setup_cold,
    "setup_device_s": rep.setup_seconds,
    "mdof_iter_per_s": n * n * nz * rep.iterations / rep.solve_seconds / 1e6,
    "ms_per_iteration": 1e3 * rep.solve_seconds / rep.iterations,
    "true_relative_residual": true_rel, "fp64_residual_floor": c.residual_floor(x, b),
    "device_gb": c.device_bytes() / 1e9, "design_generation_s": t_gen,
    "kernel_ms_per_launch": {k: round(v[0] / v[1], 4) for k, v in prof.items() if v[1]},
}
print(json.dumps(out))
if a.out:
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
