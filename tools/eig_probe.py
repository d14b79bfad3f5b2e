"""Local eigensolver outer-iteration counts per coarse cell (diagnostics).

    python tools/eig_probe.py [--n 256] [--cfg 3]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--cfg", type=int, default=3)
a = ap.parse_args()
cfg = inputs.CONFIGS[a.cfg]
n = a.n
c = Context(GridSpec(n, n, n), n // (8 * cfg["sd"]), cfg["sd"])
c.set_design_generated(cfg["vf"], cfg["kmin"], 1.0, 3, BoundarySpec.bottom_center_patch(1, 1, 0.2, 0),
                       passes=cfg["passes"], radius=cfg["radius"])
for tol in (1e-11, 1e-9):
    o = MmgOptions(num_cc_basis=cfg.get("lcc", 8), fine_blocks="coarse_cell", eig_tol=tol)
    c.setup("mmg", o)
    t = time.perf_counter()
    c.setup("mmg", o)
    dt = time.perf_counter() - t
    _, ev, it = c.local_bases()
    h = np.bincount(np.abs(it))
    print(f"tol {tol:g}: set-up {dt * 1e3:.0f} ms; outer iterations mean {np.abs(it).mean():.2f} "
          f"max {np.abs(it).max()} nonconverged {(it < 0).sum()}; histogram {h.tolist()}")
