"""B200-native PCG + multiscale-multigrid solve path of arXiv 2410.06850.

The compute lives in ``libtopmg_b200.so`` (hand-written sm_100a CUDA behind the
C ABI ``include/topmg_b200.h``); ``solver`` is a thin Python mirror of the
reference's solver interface used by the tests and the benchmark.
"""
from .solver import (BoundarySpec, ConfigError, Context, DirichletPatch, GridSpec, MmgOptions,
                     NotSupportedError, PcgResult, PrecondKind, SolveReport, SolverError,
                     make_preconditioner, native, pcg)
from .optim import (IterationLog, MaterialModel, MmaOptions, OptimConfig, OptimizeResult,
                    interpolate_design, optimize)

__all__ = ["BoundarySpec", "ConfigError", "Context", "DirichletPatch", "GridSpec", "MmgOptions",
           "NotSupportedError", "PcgResult", "PrecondKind", "SolveReport", "SolverError",
           "make_preconditioner", "native", "pcg", "IterationLog", "MaterialModel", "MmaOptions",
           "OptimConfig", "OptimizeResult", "interpolate_design", "optimize"]
