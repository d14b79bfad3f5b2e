"""Small solves of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): tools/gpu/sanitize.sh runs each case
under each tool and profiles/ keeps the summaries.

    python tools/sanitize_cases.py <case>
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_06850_b200 import (BoundarySpec, Context, GridSpec, MaterialModel, MmgOptions,  # noqa
                                   inputs)

BC = BoundarySpec.bottom_center_patch(1, 1, 0.2, 0)
CELL = MmgOptions(fine_blocks="coarse_cell")


def solve(n, ncc, sd, kind="mmg", opts=CELL, slabs=1, kmin=1e-3, iters=3):
    k = inputs.conductivity(inputs.box_filter_design(n, 0.3), kmin)
    c = Context(GridSpec(n, n, n), ncc, sd, slabs=slabs)
    c.set_conductivity(k, BC)
    c.setup(kind, opts)
    b = c.assemble_rhs(np.ones(n ** 3))
    r = c.pcg(b, rtol=1e-8, max_iterations=iters)  # graph chunks + history
    c.upload_rhs(b)
    c.solve_resident(1e-8, iters, true_residual=True)
    c.apply_preconditioner(b)
    print(kind, n, ncc, sd, slabs, r.report.iterations)


CASES = {
    # TMA ring (k_update / k_post_bnd), grid tickets, cooperative k_coarse_fused
    "mmg_cell": lambda: solve(32, 2, 2),
    # cc-element fine blocks, E = 16 (k_bj_apply) and E = 32 (k_bj32_*)
    "mmg_cc16": lambda: solve(32, 2, 2, opts=MmgOptions()),
    "mmg_cc32": lambda: solve(32, 1, 4, opts=MmgOptions()),
    # large coarse elements (coarse_large.cu), dense A_cc inverse + symv
    "mmg_large_q": lambda: solve(32, 1, 4),
    "two_grid": lambda: solve(32, 2, 2, kind="two_grid"),
    "block_jacobi": lambda: solve(32, 2, 2, kind="block_jacobi", opts=MmgOptions()),
    "jacobi": lambda: solve(32, 2, 2, kind="jacobi"),
    # A_cc by the block Thomas over cc-element planes
    "acc_planes": lambda: (os.environ.__setitem__("TMG_ACC_PLANES", "1"), solve(32, 4, 1)),
    # partitioned path: ghost exchanges, cross-slab reductions, k_finalize
    "slabs": lambda: solve(32, 2, 2, slabs=2),
    # device generator (radix select) and the MMA design loop (cooperative dual)
    "gen_optim": lambda: _gen_optim(),
    "simp": lambda: _simp(),
}


def _gen_optim():
    from paper_2410_06850_b200.optim import OptimConfig, optimize
    c = Context(GridSpec(32, 32, 32), 2, 2)
    c.set_design_generated(0.3, 1e-3, 1.0, 3, BC, passes=2, radius=2)
    cfg = OptimConfig(vstar=0.3, schedule=[GridSpec(16, 16, 16)], iters_per_level=[2],
                      ncc=(1, 1, 1), sd=2, rtol=1e-6)
    cfg.mmg = CELL
    res = optimize(cfg, MaterialModel(1e-3), BC)
    print("optim", len(res.trajectory))


def _simp():
    c = Context(GridSpec(32, 32, 32), 2, 2)
    c.set_design(np.full(32 ** 3, 0.3), 1e-6, 1.0, 3, BC)
    c.simp_init(volfrac=0.3, rmin=1.5, move=0.2, kappa_lo=1e-6, rtol=1e-6)
    print("simp", c.simp_step()["ls1_iterations"])


if __name__ == "__main__":
    CASES[sys.argv[1]]()
