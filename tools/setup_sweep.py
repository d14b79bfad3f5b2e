"""Set-up cost vs local-eigensolver settings (diagnostics): for each
(eig_tol, eig_degree) the warm set-up time (second set-up, buffers pooled),
PCG iterations and solve time at BASELINE configs[K]. Run with
TMG_SETUP_PROFILE=1 for the per-phase device times on stderr.

    python tools/setup_sweep.py [--config 3] [--settings "1e-11:32,1e-9:32,1e-9:24"]
"""
import argparse
import json
import os
import sys

import numpy as np

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--settings", default="1e-11:32,1e-10:32,1e-9:32,1e-8:32,1e-11:24,1e-9:24,1e-9:16")
a = ap.parse_args()
cfg = dict(inputs.CONFIGS[a.config])
n = cfg["n"]
ctx = Context(GridSpec(n, n, n), cfg["ncc"], cfg["sd"], device=0)
ctx.set_design_generated(cfg["vf"], cfg["kmin"], 1.0, 3,
                         BoundarySpec.bottom_center_patch(1.0, 1.0, 0.2, 0.0),
                         passes=cfg["passes"], radius=cfg["radius"])
b = ctx.assemble_rhs(np.ones(n ** 3))
ctx.upload_rhs(b)
for item in a.settings.split(","):
    tol, deg = item.split(":")
    o = MmgOptions(eig_tol=float(tol), eig_degree=int(deg), num_cc_basis=cfg.get("lcc", 8),
                   fine_blocks="coarse_cell")
    ctx.setup("mmg", o)
    print(f"--- eig_tol {tol} degree {deg} (warm set-up below)", file=sys.stderr, flush=True)
    ctx.setup("mmg", o)
    ctx.upload_rhs(b)
    rep = ctx.solve_resident(1e-8, 5000)
    extra = {}
    if n <= 256:  # local-eigensolver rounds (downloads the bases)
        _, _, its = ctx.local_bases()
        extra = {"eig_rounds_mean": float(np.mean(np.abs(its))), "eig_rounds_max": int(np.max(its)),
                 "eig_unconverged": int(np.sum(its < 0))}
    print(json.dumps({"config": a.config, "eig_tol": float(tol), "eig_degree": int(deg),
                      "setup_ms": rep.setup_seconds * 1e3, "iterations": rep.iterations,
                      "solve_ms": rep.solve_seconds * 1e3, "converged": rep.converged, **extra}),
          flush=True)
