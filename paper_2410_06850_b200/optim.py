"""The reference's design loop, host side (topmg::optimize, optim.cpp:240-345;
types optim.hpp:27-96). Each resolution level runs on the device through the
C ABI (tmg_optim_*: conductivity and heat source, preconditioner set-up, LS1
and LS2, sensitivity, MMA update); this module keeps the level schedule, the
design prolongation between levels (interpolate_design, grid.cpp:220-241),
the per-level budgets and the ||dx||_inf stop, and the final evaluation solve.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from .solver import BoundarySpec, Context, GridSpec, MmgOptions, SolverError


@dataclass
class MmaOptions:
    """MmaOptions (optim.hpp:27-32)."""
    move_limit: float = 0.2
    asy_init: float = 0.5
    asy_incr: float = 1.2
    asy_decr: float = 0.7


@dataclass
class MaterialModel:
    """MaterialModel (material.hpp; material.cpp:8-16): kappa = lo + x^p (hi - lo),
    f = f0 (1 - x^p)."""
    kappa_lo: float
    kappa_hi: float = 1.0
    f0: float = 1.0
    p: int = 3


@dataclass
class OptimConfig:
    """OptimConfig (optim.hpp:58-72). precond: a PrecondKind name."""
    vstar: float = 0.05
    schedule: List[GridSpec] = field(default_factory=list)
    iters_per_level: List[int] = field(default_factory=list)
    convergence_dx: float = 0.01
    mma: MmaOptions = field(default_factory=MmaOptions)
    ncc: Tuple[int, int, int] = (2, 2, 2)
    sd: int = 2
    mmg: MmgOptions = field(default_factory=MmgOptions)
    precond: str = "mmg"
    rtol: float = 1e-6
    maxit: int = 10000
    warm_start: bool = False  # not in the reference: warm set-up / solves between iterations


@dataclass
class IterationLog:
    """IterationLog (optim.hpp:74-84) plus the update's ||dx||_inf and multiplier."""
    level: int = 0
    iter: int = 0
    cost: float = 0.0
    volume: float = 0.0
    ls1_iters: int = 0
    ls2_iters: int = 0
    setup_seconds: float = 0.0
    ls1_seconds: float = 0.0
    ls2_seconds: float = 0.0
    dx_inf: float = 0.0
    lam: float = 0.0


@dataclass
class OptimizeResult:
    """OptimizeResult (optim.hpp:86-96)."""
    design: np.ndarray = None
    grid: GridSpec = None
    temperature: np.ndarray = None
    final_cost: float = 0.0
    trajectory: List[IterationLog] = field(default_factory=list)
    failed: bool = False
    failure_message: str = ""
    total_linear_iterations: int = 0


def interpolate_design(values_lo: np.ndarray, grid_lo: GridSpec, grid_hi: GridSpec) -> np.ndarray:
    """Piecewise-constant prolongation by an integer factor per axis
    (interpolate_design, grid.cpp:220-241)."""
    n_lo = (grid_lo.nx, grid_lo.ny, grid_lo.nz)
    n_hi = (grid_hi.nx, grid_hi.ny, grid_hi.nz)
    if np.size(values_lo) != grid_lo.num_cells():
        raise ValueError("interpolate_design: field size does not match grid")
    if any(h % l for h, l in zip(n_hi, n_lo)):
        raise ValueError("interpolate_design: non-integer refinement factor")
    f = [h // l for h, l in zip(n_hi, n_lo)]
    v = np.asarray(values_lo, dtype=np.float64).reshape(n_lo[2], n_lo[1], n_lo[0])
    v = np.repeat(np.repeat(np.repeat(v, f[2], axis=0), f[1], axis=1), f[0], axis=2)
    return np.ascontiguousarray(v).ravel()


def _log(level: int, d: dict) -> IterationLog:
    return IterationLog(level=level, iter=d["iter"], cost=d["cost"], volume=d["volume"],
                        ls1_iters=d["ls1_iters"], ls2_iters=d["ls2_iters"],
                        setup_seconds=d["setup_seconds"], ls1_seconds=d["ls1_seconds"],
                        ls2_seconds=d["ls2_seconds"], dx_inf=d["dx_inf"], lam=d["lambda"])


def optimize(cfg: OptimConfig, material: MaterialModel, boundary: BoundarySpec,
             device: int = 0) -> OptimizeResult:
    """topmg::optimize (optim.cpp:240-345): uniform x = vstar, then per level
    form kappa -> preconditioner -> LS1, LS2 -> sensitivity -> MMA update until
    the level budget or ||dx||_inf < convergence_dx, prolongate to the next
    level; one evaluation solve of the final design. A linear solve that does
    not converge ends the run with failed = True and the partial trajectory."""
    if not cfg.schedule:
        raise ValueError("optimize: empty resolution schedule")
    if len(cfg.schedule) != len(cfg.iters_per_level):
        raise ValueError("optimize: schedule and iteration budgets disagree")
    if not (0.0 < cfg.vstar <= 1.0):
        raise ValueError("optimize: vstar must lie in (0, 1]")
    res = OptimizeResult()
    x = None
    ctx = None
    m = cfg.mma

    def init(level_ctx, x0):
        level_ctx.optim_init(vstar=cfg.vstar, kappa_lo=material.kappa_lo,
                             kappa_hi=material.kappa_hi, f0=material.f0, p=material.p,
                             move_limit=m.move_limit, asy_init=m.asy_init, asy_incr=m.asy_incr,
                             asy_decr=m.asy_decr, rtol=cfg.rtol, maxit=cfg.maxit,
                             warm_start=cfg.warm_start, x0=x0, kind=cfg.precond, mmg=cfg.mmg)

    for level, grid in enumerate(cfg.schedule):
        x0 = (np.full(grid.num_cells(), cfg.vstar) if level == 0
              else interpolate_design(x, cfg.schedule[level - 1], grid))
        ctx = Context(grid, cfg.ncc, cfg.sd, device=device)
        ctx.set_design(x0, material.kappa_lo, material.kappa_hi, material.p, boundary)
        init(ctx, x0)
        for _ in range(cfg.iters_per_level[level]):
            try:
                d = ctx.optim_step()
            except SolverError as e:
                if "did not converge" not in str(e):
                    raise
                res.failed, res.failure_message = True, str(e)
                res.design, res.grid = ctx.optim_download()[0], grid
                return res
            lg = _log(level, d)
            res.trajectory.append(lg)
            res.total_linear_iterations += lg.ls1_iters + lg.ls2_iters
            if lg.dx_inf < cfg.convergence_dx:
                break
        x = ctx.optim_download()[0]
    try:
        d = ctx.optim_evaluate()
    except SolverError as e:
        if "did not converge" not in str(e):
            raise
        res.failed, res.failure_message = True, str(e)
        res.design, res.grid = x, cfg.schedule[-1]
        return res
    res.final_cost = d["cost"]
    res.design, res.temperature = ctx.optim_download()
    res.grid = cfg.schedule[-1]
    return res
