"""The reference's design loop (topmg::optimize with MMA, optim.cpp:240-345) on
the device against the compiled reference (oracle/_ref ref_optimize): same
schedule, material, boundary and preconditioner partition (the reference's
fine blocks, one per cc element). Bars: per-iteration cost and volume, linear
iteration counts within 10%, the final design and cost."""
import numpy as np
import pytest

import oracle as O
from paper_2410_06850_b200 import (BoundarySpec, GridSpec, MaterialModel, MmgOptions,
                                   OptimConfig, optimize)

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
BC = BoundarySpec.bottom_center_patch(1.0, 1.0, 0.2, 0.0)


def close_iters(a, b):
    return abs(a - b) <= max(1, int(0.1 * b))


@needs_ref
@pytest.mark.parametrize("levels,iters,vstar,kmin", [([16], [6], 0.3, 1e-3),
                                                     ([16, 32], [4, 3], 0.2, 1e-3),
                                                     # three levels: 2^3 coarse cells at 8^3
                                                     # (generic kernels)
                                                     ([8, 16, 32], [3, 2, 2], 0.3, 1e-3)])
def test_optimize_matches_reference(levels, iters, vstar, kmin):
    ref, x_ref, fc_ref, failed = O.ref_optimize(levels, iters, 2, 2, vstar=vstar, kappa_lo=kmin)
    assert not failed
    cfg = OptimConfig(vstar=vstar, schedule=[GridSpec(n, n, n) for n in levels],
                      iters_per_level=iters, ncc=(2, 2, 2), sd=2,
                      mmg=MmgOptions(fine_blocks="cc"))
    res = optimize(cfg, MaterialModel(kmin, 1.0, 1.0, 3), BC)
    assert not res.failed
    n = len(ref["cost"])
    assert len(res.trajectory) == n
    for k, lg in enumerate(res.trajectory):
        assert abs(lg.cost - ref["cost"][k]) <= 1e-6 * abs(ref["cost"][k]), (k, lg.cost, ref["cost"][k])
        assert abs(lg.volume - ref["volume"][k]) <= 1e-9, k
        assert close_iters(lg.ls1_iters, ref["ls1"][k]), (k, lg.ls1_iters, ref["ls1"][k])
        assert close_iters(lg.ls2_iters, ref["ls2"][k]), (k, lg.ls2_iters, ref["ls2"][k])
    assert np.max(np.abs(res.design - x_ref)) <= 1e-6
    assert abs(res.final_cost - fc_ref) <= 1e-6 * abs(fc_ref)


def test_optimize_gpu_default_blocks_and_warm_start():
    """The default (reference) fine blocks, one per cc element, and the
    warm-started variant follow the same design trajectory (the solves agree
    to rtol)."""
    cfg = OptimConfig(vstar=0.3, schedule=[GridSpec(32, 32, 32)], iters_per_level=[5],
                      ncc=(2, 2, 2), sd=2, rtol=1e-8)
    a = optimize(cfg, MaterialModel(1e-3), BC)
    cfg.warm_start = True
    b = optimize(cfg, MaterialModel(1e-3), BC)
    assert not a.failed and not b.failed
    costs = [t.cost for t in a.trajectory]
    assert costs[-1] < costs[0]
    for ta, tb in zip(a.trajectory, b.trajectory):
        assert abs(ta.cost - tb.cost) <= 1e-6 * abs(ta.cost)
    assert np.max(np.abs(a.design - b.design)) <= 1e-5
    assert abs(a.design.mean() - 0.3) < 0.02


def test_optimize_nonconvergence_is_a_partial_result():
    cfg = OptimConfig(vstar=0.3, schedule=[GridSpec(16, 16, 16)], iters_per_level=[3],
                      ncc=(2, 2, 2), sd=2, maxit=2)
    res = optimize(cfg, MaterialModel(1e-3), BC)
    assert res.failed and "did not converge within 2 iterations" in res.failure_message
    assert res.trajectory == []
