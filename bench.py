"""Benchmark: FP64 PCG + multiscale-MG solve throughput on B200.

Workload (BASELINE.json configs[1], the single-GPU configuration the metric is
quoted on): 128^3 cells, seeded box-filter design (vf 0.3, 3 passes, radius 2),
SIMP p = 3, kmin = 1e-6, unit source, T = 0 on the centred 0.2 x 0.2 patch of
z = 0, PCG to ||r||/||b|| <= 1e-8 with the multiscale V-cycle (L_c = 4,
L_cc = 8, c = 8, sd = 2, ncc = 8). One step = one full PCG solve from x0 = 0
on the resident system. value = DoF * iterations / solve time (MDoF*iter/s).
With N > 1 ranks (torchrun) the solve is partitioned: one configs[1] slab of
128^3 cells per GPU stacked along z (weak scaling), ghost exchanges and CG
reductions over NCCL, time = max over ranks, value = all DoF of the job.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--impl reference times the reference's own CPU implementation of the path
(oracle/_ref: proj/core compiled unmodified) on the same
config with all host threads; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG solve MDoF*iter/s (FP64, rtol 1e-8, multiscale-MG V-cycle)"
UNIT = "MDoF*iter/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
RTOL = 1e-8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)  # ~0.55 s timed: enough clock samples
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-side-by-side", action="store_true",
                    help="skip the LS2 row and the config-1 side-by-side preconditioners")
    ap.add_argument("--ref-iters", type=int, default=8,
                    help="PCG iterations per reference step (bounded sample)")
    return ap.parse_args()


def workload(cfg_id, world=1):
    """configs[cfg_id] design; with world > 1 the weak-scaling grid of the
    partitioned runs: world slabs of n^3 cells stacked along z."""
    from paper_2410_06850_b200 import inputs
    cfg = dict(inputs.CONFIGS[cfg_id])
    n = cfg["n"]
    shape = n if world == 1 else (n, n, n * world)
    rho = inputs.box_filter_design(shape, cfg["vf"], passes=cfg["passes"], radius=cfg["radius"])
    kappa = inputs.conductivity(rho, cfg["kmin"])
    return cfg, kappa


def config_json(cfg, cfg_id, extra=None, world=1):
    n = cfg["n"]
    if world == 1:
        d = {"workload": f"BASELINE configs[{cfg_id}]: {n}^3 cells, kmin={cfg['kmin']:g}, "
                         f"MMG-PCG rtol={RTOL:g}",
             "cells": n ** 3,
             "hierarchy": f"c={n // (cfg['ncc'] * cfg['sd'])} sd={cfg['sd']} ncc={cfg['ncc']} "
                          f"L_c=4 L_cc={cfg.get('lcc', 8)} nu=1"}
    else:
        d = {"workload": f"{world} x BASELINE configs[{cfg_id}] slabs: {n}x{n}x{n * world} cells, "
                         f"kmin={cfg['kmin']:g}, MMG-PCG rtol={RTOL:g}",
             "cells": n ** 3 * world,
             "hierarchy": f"c={n // (cfg['ncc'] * cfg['sd'])} sd={cfg['sd']} "
                          f"ncc={cfg['ncc']}x{cfg['ncc']}x{cfg['ncc'] * world} L_c=4 "
                          f"L_cc={cfg.get('lcc', 8)} nu=1"}
    d.update({"kmin": cfg["kmin"], "rtol": RTOL,
              "smoother": "exact block-Jacobi per coarse cell (fine) / per cc element (coarse)",
              "l2": "no flush: one solve streams ~1.7 GB/iteration per GPU through the 126 MB L2"})
    if extra:
        d.update(extra)
    return d


# ------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clocks and throttle reasons
    during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clocks_setting"}

    def __init__(self, device):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------- reference

def reference_context(cfg, kappa, world=1):
    """The reference (proj/core, oracle/_ref) on the bench workload: configs[1]
    for N = 1, the N-slab elongated grid of the partitioned runs for N > 1."""
    import ctypes as C
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # bench's reference / cpu-baseline leg only
    R = O.ref()
    R.ref_set_num_threads(0)
    pa = O._patch_array(O.bottom_center_patch())
    ts = C.c_double()
    n = cfg["n"]
    ctx = R.ref_ctx_create_grid(n, n, n * world, 1.0, 1.0, float(world), cfg["ncc"], cfg["ncc"],
                                cfg["ncc"] * world, cfg["sd"], O._d(kappa), 1, O._d(pa), 4,
                                O.BLOCKS["cell"], O.BLOCKS["cc"], 4, 8, 1, C.byref(ts))
    if not ctx:
        raise RuntimeError(R.ref_last_error().decode())
    return O, R, ctx, ts.value, R.ref_num_threads()


def reference_steps(O, R, ctx, n, steps, iters):
    import ctypes as C
    it, cv, sv = C.c_int(), C.c_int(), C.c_double()
    tot_it, tot_s = 0, 0.0
    for _ in range(steps):
        rc = R.ref_ctx_pcg(ctx, C.c_double(RTOL), C.c_int(iters), None, C.byref(it), C.byref(cv),
                           C.byref(sv))
        if rc:
            raise RuntimeError(R.ref_last_error().decode())
        tot_it += it.value
        tot_s += sv.value
    return tot_it, tot_s


def cpu_baseline(cfg, kappa, iters):
    O, R, ctx, setup_s, threads = reference_context(cfg, kappa)
    try:
        its, secs = reference_steps(O, R, ctx, cfg["n"], 1, iters)
    finally:
        R.ref_ctx_destroy(ctx)
    return {"value": cfg["n"] ** 3 * its / secs / 1e6, "unit": UNIT, "cores": threads,
            "kind": "reference",
            "sample": f"reference proj/core (oracle/_ref) on {cfg['n']}^3 configs[1]: "
                      f"set-up ({setup_s:.1f} s, untimed) + one PCG of {its} iterations",
            "setup_seconds": setup_s}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    cfg, kappa = workload(args.config, world)
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libtopmg_ref.so")):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtopmg_ref.so not built "
                          "(run bash oracle/build_ref.sh where /root/reference exists)"}))
        return 0
    O, R, ctx, setup_s, threads = reference_context(cfg, kappa, world)
    # bounded sample: the N-slab grid is N times larger, so fewer iterations
    # per step keep the whole run within minutes (the metric is per iteration)
    ref_iters = max(2, args.ref_iters // world)
    try:
        reference_steps(O, R, ctx, cfg["n"], args.warmup, ref_iters)
        t0 = time.perf_counter()
        its, secs = reference_steps(O, R, ctx, cfg["n"], args.steps, ref_iters)
        wall = time.perf_counter() - t0
    finally:
        R.ref_ctx_destroy(ctx)
    value = kappa.size * its / secs / 1e6
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE configs[1])",
            "config": config_json(cfg, args.config, {"reference_setup_seconds": setup_s,
                                                     "iterations_per_step": its // args.steps},
                                  world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{args.steps} steps x {ref_iters} PCG iterations "
                                       f"of the reference on {kappa.size} cells (set-up untimed)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# -------------------------------------------------------------------- ours

# Algorithmic bytes per fine cell of the iteration kernels:
# unique data that must move between HBM and the SMs once per launch. The
# boundary-form kernels touch Phi and r1 only on the 296 of 512 cells of each
# brick that lie on its surface (SURF), plus the face T's (3 B).
#  k_post  : r 8 + coef_z 8 + G 288 + z 8 + (Phi 32 + r1 8)*SURF + T 3 = 338.1
#  k_update: x 16 + p 8 + q 8 + r 16 + coef_z 8 + G 288 + r1 8*SURF     = 348.6
#  k_restrict: (Phi 32 + r1 8)*SURF + T 3                              = 26.1
#  k_search: coef 32 + z 8 + p 16 + q 8                                 = 64
SURF = 296 / 512
KERNEL_BYTES_PER_CELL = {"post": 312 + 40 * SURF + 3, "update": 344 + 8 * SURF, "search": 64,
                         "restrict": 40 * SURF + 3}
ITER_BYTES_PER_CELL = sum(KERNEL_BYTES_PER_CELL.values())  # + coarse levels (~0.1%)


def ncu_traffic(kernel):
    path = os.path.join(ROOT, "profiles", "ncu_summary_latest.json")
    try:
        with open(path) as f:
            d = json.load(f)
        ks = d["kernels"]
        for name in ("k_" + kernel + "_bnd", "k_" + kernel):  # boundary-form kernels first
            if name in ks:
                return ks[name]["dram_bytes_per_launch"]
        return None
    except Exception:
        return None


def side_by_side(ctx, b, M):
    """SURVEY.md §8(d) second rows, one device-timed solve each on the bench
    design: LS2 (adjoint rhs 1/M, optim.cpp:16-19) on the resident MMG
    hierarchy, then config 1's side-by-side preconditioners (M6: the
    reference kinds jacobi / block_jacobi / two_grid, and mmg with the
    reference's own fine blocks, one per cc element)."""
    def row(rep, setup_s=None):
        return {"iterations": rep.iterations, "converged": rep.converged,
                "solve_ms": 1e3 * rep.solve_seconds,
                "setup_ms": 1e3 * (rep.setup_seconds if setup_s is None else setup_s),
                "mdof_iter_per_s": M * rep.iterations / rep.solve_seconds / 1e6
                if rep.solve_seconds > 0 else None}
    out = {}
    ctx.upload_rhs(np.full(M, 1.0 / M))
    out["ls2"] = row(ctx.solve_resident(RTOL, 20000))
    from paper_2410_06850_b200 import MmgOptions
    rows = {}
    for name, kind, opts in [("jacobi", "jacobi", MmgOptions()),
                             ("block_jacobi", "block_jacobi", MmgOptions()),
                             ("two_grid", "two_grid", MmgOptions()),
                             ("mmg_reference_fine_blocks", "mmg", MmgOptions(fine_blocks="cc"))]:
        try:
            ctx.setup(kind, opts)
            ctx.upload_rhs(b)
            rows[name] = row(ctx.solve_resident(RTOL, 20000))
        except Exception as e:  # reported, not fatal
            rows[name] = {"unavailable": str(e)[:160]}
    out["side_by_side"] = rows
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, inputs
    from paper_2410_06850_b200 import dist as D
    n = inputs.CONFIGS[args.config]["n"]
    patch = BoundarySpec.bottom_center_patch(1.0, 1.0, 0.2, 0.0)
    cfg, kappa = workload(args.config, world)
    if world == 1:
        grid = GridSpec(n, n, n)
        ctx = Context(grid, cfg["ncc"], cfg["sd"], device=local)
        kappa_local = kappa
    else:
        # weak scaling: one configs[1] slab (n^3 cells) per GPU, stacked along z
        # into an n x n x (n * world) grid with cubic cells (lz = world); the
        # design is the same generator on the whole grid.
        grid = GridSpec(n, n, n * world, 1.0, 1.0, float(world))
        ncc = (cfg["ncc"], cfg["ncc"], cfg["ncc"] * world)
        ctx = D.dist_context(grid, ncc, cfg["sd"], dist, local)
        kappa_local = D.slab(kappa, D.partition(grid, ncc, cfg["sd"], world, rank))
    M_local = ctx.cells
    M = grid.num_cells()
    ctx.set_conductivity(kappa_local, patch)
    b = ctx.assemble_rhs(np.ones(M_local))
    barrier()
    t0 = time.perf_counter()
    from paper_2410_06850_b200 import MmgOptions
    mopts = MmgOptions(num_cc_basis=cfg.get("lcc", 8))
    ctx.setup("mmg", mopts)  # first set-up: includes module loading and allocations
    setup_cold_wall = max_over_ranks(time.perf_counter() - t0)
    barrier()
    t0 = time.perf_counter()
    ctx.setup("mmg", mopts)  # re-set-up (a design iteration's cost; buffers pooled)
    setup_wall = max_over_ranks(time.perf_counter() - t0)
    ctx.upload_rhs(b)
    for _ in range(max(3, args.warmup)):
        rep = ctx.solve_resident(RTOL, 10000)
    stream = torch.cuda.ExternalStream(ctx.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.kernel_launches()
    torch.cuda.synchronize()
    barrier()
    its = []
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            rep = ctx.solve_resident(RTOL, 10000)
            its.append(rep.iterations)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = ctx.kernel_launches() - launches0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    iters = int(np.mean(its))
    value = M * iters / (ms * 1e-3) / 1e6

    # e2e through the C ABI with pinned host buffers (H2D b, solve, D2H x)
    b_pin = torch.from_numpy(b).pin_memory().numpy()
    x_pin = torch.empty(M_local, dtype=torch.float64).pin_memory().numpy()
    ctx.pcg(b_pin, rtol=RTOL, out=x_pin)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    e2e_its = 0
    for _ in range(args.steps):
        e2e_its += ctx.pcg(b_pin, rtol=RTOL, out=x_pin).report.iterations
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
    e2e_value = M * (e2e_its / args.steps) / e2e_s / 1e6
    res2 = sum_over_ranks(float(np.sum((b - ctx.apply_operator(x_pin)) ** 2)))
    b2 = sum_over_ranks(float(np.sum(b ** 2)))
    true_rel = float(np.sqrt(res2 / b2))

    peak = None
    peak_src = "fallback 6650 GB/s (B200_PROFILING.md)"
    try:
        with open(PEAKS) as f:
            peak = float(json.load(f)["hbm_gbs"])
            peak_src = "measured MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        peak = 6650.0
    iter_achieved = ITER_BYTES_PER_CELL * M_local * iters / (ms * 1e-3) / 1e9  # per GPU
    if world == 1:
        # per-kernel CUDA-event times during one live solve (roofline)
        prof = ctx.profile_solve(RTOL, 10000)
        per = {k: (v[0] / v[1] if v[1] else 0.0) for k, v in prof.items()}
        dominant = max(("post", "update", "search", "restrict"), key=lambda k: prof[k][0])
        bytes_launch = KERNEL_BYTES_PER_CELL[dominant] * M
        achieved = bytes_launch / (per[dominant] * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": ncu_traffic(dominant),
                "algorithmic_bytes_per_launch": bytes_launch, "peak_source": peak_src}
    else:
        per = {}
        roof = {"bound": "hbm", "kernel": "whole iteration, per GPU (incl. exchanges)",
                "achieved": iter_achieved, "peak": peak, "unit": "GB/s",
                "frac": iter_achieved / peak, "traffic": None,
                "algorithmic_bytes_per_launch": ITER_BYTES_PER_CELL * M_local,
                "peak_source": peak_src}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    extra = {
        "iterations": iters, "setup_ms": 1e3 * rep.setup_seconds,
        "setup_wall_ms": 1e3 * setup_wall, "setup_cold_wall_ms": 1e3 * setup_cold_wall,
        "time_to_solution_ms": 1e3 * rep.setup_seconds + ms,
        "true_relative_residual": true_rel,
        "parallelism": f"z-slabs x{world} over NCCL (one {n}^3 slab per GPU)" if world > 1
                       else "single-gpu",
        "kernel_ms_per_launch": {k: round(v, 4) for k, v in per.items() if v},
        "iteration_hbm_gbs_algorithmic_per_gpu": iter_achieved,
        "device_bytes": ctx.device_bytes()}
    cj = config_json(cfg, args.config, extra, world)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded box-filter design, BASELINE configs[1])",
        "config": cj,
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * M_local,
                "d2h_bytes_per_step": 8 * M_local},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_side_by_side and args.config == 1:  # M6: config 1's rows
        line.update(side_by_side(ctx, b, M))
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, kappa, args.ref_iters)
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "unavailable": str(e)[:200]}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
