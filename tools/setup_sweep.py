"""Set-up cost vs local-eigensolver settings at BASELINE configs[1] (diagnostics):
for each (eig_tol, eig_degree) the set-up time (second set-up, buffers pooled),
PCG iterations and solve time. Prints one JSON line per setting.

    python tools/setup_sweep.py
"""
import json
import os
import sys

import numpy as np

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs  # noqa: E402

cfg = dict(inputs.CONFIGS[1])
n = cfg["n"]
rho = inputs.box_filter_design(n, cfg["vf"], passes=cfg["passes"], radius=cfg["radius"])
kappa = inputs.conductivity(rho, cfg["kmin"])
ctx = Context(GridSpec(n, n, n), cfg["ncc"], cfg["sd"], device=0)
ctx.set_conductivity(kappa, BoundarySpec.bottom_center_patch(1.0, 1.0, 0.2, 0.0))
b = ctx.assemble_rhs(np.ones(n ** 3))
settings = [(0.0, 0), (1e-10, 0), (1e-9, 0), (1e-8, 0), (1e-7, 0), (0.0, 24), (0.0, 16), (1e-9, 24), (1e-8, 16)]
for tol, deg in settings:
    o = MmgOptions(eig_tol=tol, eig_degree=deg)
    ctx.setup("mmg", o)
    ctx.setup("mmg", o)
    res = ctx.pcg(b, rtol=1e-8, max_iterations=1000)
    rep = res.report
    print(json.dumps({"eig_tol": tol or 1e-11, "eig_degree": deg or 32, "setup_ms": rep.setup_seconds * 1e3,
                      "iterations": rep.iterations, "solve_ms": rep.solve_seconds * 1e3,
                      "converged": rep.converged}), flush=True)
