"""BASELINE configs[3] on one B200: 512^3 cells (~1.34e8 DoF), seeded box-filter
design (vf 0.2, radius 4, 3 passes), kmin 1e-6, MMG-PCG to rtol 1e-8.

Hierarchy: c = n / (ncc sd) cells per coarse cell, L_c = 4. Defaults: sd = 4,
ncc = n / 32 (c = 8, q = sd^3 L_c = 256: the large-element coarse level of
coarse_large.cu) and L_cc = 12, so n_cc = 12 ncc^3 (49152 at 512^3: the
dense A_cc^-1 takes 19 GB). At 512^3, L_cc = 8 needs 372 iterations and
L_cc = 12 needs 49 (profiles/r05_config3_512*.json). SURVEY.md suggests sd = 8 / ncc = 8 (q = 2048), which
needs a block-sparse coarse level.

    python tools/config3.py [--n 512] [--ncc 16] [--sd 4] [--lcc 12] [--solves 2] [--out f.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--lcc", type=int, default=12)
ap.add_argument("--sd", type=int, default=4)
ap.add_argument("--ncc", type=int, default=0)
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--out", default=None)
ap.add_argument("--host-gen", action="store_true", help="generate the design with numpy")
a = ap.parse_args()
n = a.n
sd = a.sd
ncc = a.ncc or n // (8 * sd)
c = Context(GridSpec(n, n, n), ncc, sd)
bc = BoundarySpec.bottom_center_patch(1, 1, 0.2, 0)
t0 = time.perf_counter()
if a.host_gen:
    rho = inputs.box_filter_design(n, 0.2, passes=3, radius=4)
    c.set_conductivity(inputs.conductivity(rho, 1e-6), bc)
    del rho
else:  # on the device (gen.cu), bit-identical
    c.set_design_generated(0.2, 1e-6, 1.0, 3, bc, passes=3, radius=4)
t_gen = time.perf_counter() - t0
b = c.assemble_rhs(np.ones(n ** 3))
t0 = time.perf_counter()
c.setup("mmg", MmgOptions(num_cc_basis=a.lcc, fine_blocks="coarse_cell"))
t_setup = time.perf_counter() - t0
c.upload_rhs(b)
reps = [c.solve_resident(1e-8, 20000) for _ in range(a.solves)]
rep = reps[-1]
x = c.download_solution()
true_rel = float(np.linalg.norm(b - c.apply_operator(x)) / np.linalg.norm(b))
out = {
    "workload": f"BASELINE configs[3]-style: {n}^3 cells, vf 0.2, radius 4, kmin 1e-6, rtol 1e-8",
    "hierarchy": f"c={n // (ncc * sd)} sd={sd} ncc={ncc} L_c=4 L_cc={a.lcc} "
                 f"(n_cc={ncc ** 3 * a.lcc})",
    "cells": n ** 3, "iterations": rep.iterations, "converged": rep.converged,
    "solve_s": rep.solve_seconds, "setup_s": t_setup,
    "mdof_iter_per_s": n ** 3 * rep.iterations / rep.solve_seconds / 1e6,
    "ms_per_iteration": 1e3 * rep.solve_seconds / rep.iterations,
    "true_relative_residual": true_rel, "device_gb": c.device_bytes() / 1e9,
    "design_generation_s": t_gen, "design_generator": "host numpy" if a.host_gen else "device",
}
print(json.dumps(out))
if a.out:
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
