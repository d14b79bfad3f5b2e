import sys, time, numpy as np
import os; R=os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0,R); sys.path.insert(0,R+'/oracle')
import oracle as O
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, MmgOptions, inputs
def run(n, ncc, sd, kmin, kinds=('jacobi','mmg')):
    rho = inputs.box_filter_design(n, 0.3); kappa = inputs.conductivity(rho, kmin)
    bc = BoundarySpec.bottom_center_patch(1.0, 1.0, 0.2, 0.0)
    ctx = Context(GridSpec(n, n, n), ncc, sd)
    ctx.set_conductivity(kappa, bc)
    b = ctx.assemble_rhs(np.ones(n**3))
    g = O.grid(n); sysm = O.System(g, kappa, np.ones(n**3), O.bottom_center_patch())
    print('rhs equal', np.array_equal(b, sysm.rhs), flush=True)
    x = np.random.default_rng(0).standard_normal(n**3)
    y = ctx.apply_operator(x); yr = sysm.apply(x)
    print('apply bitwise', np.array_equal(y, yr), np.abs(y-yr).max(), flush=True)
    for kind in kinds:
        t=time.time(); ctx.setup(kind, MmgOptions()); ts=time.time()-t
        res = ctx.pcg(b, rtol=1e-8, max_iterations=3000)
        if kind=='mmg':
            m = O.Precond('mmg', sysm, O.hierarchy(g, ncc, sd), fine_blocks='cell', coarse_blocks='cc')
        else:
            m = O.Precond(kind, sysm)
        ref = O.pcg(sysm, sysm.rhs, m, rtol=1e-8, max_iterations=3000)
        rel = np.linalg.norm(res.x-ref.x)/np.linalg.norm(ref.x)
        print(n, kind, 'gpu it', res.report.iterations, res.report.converged, 'oracle it', ref.iterations, 'rel', rel,
              'setup %.3fs solve %.2fms'%(ts, res.report.solve_seconds*1e3), flush=True)
        if kind=='mmg':
            phi, ev, it = ctx.local_bases()
            print('  eig iters min/max', it.min(), it.max(), 'evals[0]', ev[0])
            # repeat solve timing
            for _ in range(3):
                r2 = ctx.pcg(b, rtol=1e-8, max_iterations=3000)
            print('  repeat solve ms', r2.report.solve_seconds*1e3, r2.report.iterations)
run(16, 2, 2, 1e-3)
run(32, 2, 2, 1e-6)
run(64, 4, 2, 1e-3)
# config 1: 128^3, kmin 1e-6, GPU only (true residual check)
n=128; rho = inputs.box_filter_design(n, 0.3); kappa = inputs.conductivity(rho, 1e-6)
ctx = Context(GridSpec(n, n, n), 8, 2); ctx.set_conductivity(kappa, BoundarySpec.bottom_center_patch(1,1,0.2,0))
b = ctx.assemble_rhs(np.ones(n**3))
for kind in ['mmg']:
    t=time.time(); ctx.setup(kind); ts=time.time()-t
    for _ in range(3): res = ctx.pcg(b, rtol=1e-8, max_iterations=5000)
    tr = np.linalg.norm(b-ctx.apply_operator(res.x))/np.linalg.norm(b)
    print(128, kind, res.report.iterations, res.report.converged, 'true rel res', tr, 'setup %.3fs (dev %.3fs) solve %.2fms'%(ts, res.report.setup_seconds, res.report.solve_seconds*1e3), flush=True)
    ctx.upload_rhs(b)
    for _ in range(3): rep = ctx.solve_resident(1e-8, 5000)
    print(' resident solve ms', rep.solve_seconds*1e3, rep.iterations, 'MDoF.it/s', n**3*rep.iterations/rep.solve_seconds/1e6)
    prof = ctx.profile_solve(1e-8, 5000)
    for k,(ms,cnt) in prof.items():
        if cnt: print('  %-12s %8.3f ms total %5d launches %8.1f us/launch'%(k, ms, cnt, 1e3*ms/cnt))
