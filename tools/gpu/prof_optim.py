import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
from paper_2410_06850_b200 import OptimConfig, MaterialModel, GridSpec, BoundarySpec, optimize
n = 128
mk = lambda it: OptimConfig(vstar=0.3, schedule=[GridSpec(n, n, n)], iters_per_level=[it], convergence_dx=0.0, ncc=(n // 16,) * 3, sd=2, rtol=1e-8)
optimize(mk(1), MaterialModel(1e-6, 1.0, 1.0, 3), BoundarySpec.bottom_center_patch(1, 1, 0.2, 0))
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
optimize(mk(10), MaterialModel(1e-6, 1.0, 1.0, 3), BoundarySpec.bottom_center_patch(1, 1, 0.2, 0))
pr.disable()
print("wall", time.perf_counter() - t0)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
