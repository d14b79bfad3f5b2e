/*
 * topmg_b200 — C ABI of the B200 PCG + multiscale-multigrid solve path.
 *
 * This is the drop-in boundary for the reference's linear-solve hot path
 * (/root/reference/proj/core). Each entry point cites the reference interface
 * it replaces. Plain pointers and sizes only; every host array is in the
 * reference's x-fastest cell order i + nx*(j + ny*k) (grid.hpp:27-29,44-46).
 * All arithmetic is FP64. Errors follow the reference's three exception
 * classes (grid.hpp:16-24, solver.cpp:486-492) as return codes; the message
 * is available from tmg_last_error(). Non-convergence is not an error
 * (solver.hpp:179-182): it is reported through tmg_report.converged = 0.
 *
 * A context owns one GPU's device memory, one CUDA stream and the captured
 * iteration graph. It is thread-compatible, not thread-safe.
 */
#ifndef TOPMG_B200_H
#define TOPMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes. */
#define TMG_OK 0
#define TMG_ECONFIG 1 /* topmg::ConfigError   (grid.hpp:16-19)        */
#define TMG_ESOLVER 2 /* topmg::SolverError   (grid.hpp:21-24)        */
#define TMG_EARG 3    /* std::invalid_argument (solver.cpp:486-492)   */
#define TMG_ECUDA 4   /* CUDA runtime failure                          */
#define TMG_ENOTSUP 5 /* configuration outside what the GPU path builds */

/* PrecondKind (solver.hpp:160). */
#define TMG_PRECOND_NONE 0
#define TMG_PRECOND_JACOBI 1
#define TMG_PRECOND_BLOCK_JACOBI 2 /* cc-element blocks of 8^3 / 16^3 cells */
#define TMG_PRECOND_TWO_GRID 3     /* R_cc = I; sd^3 L_c <= 256             */
#define TMG_PRECOND_MMG 4

/* Faces, topmg::Face (grid.hpp:57). */
#define TMG_FACE_XLO 0
#define TMG_FACE_XHI 1
#define TMG_FACE_YLO 2
#define TMG_FACE_YHI 3
#define TMG_FACE_ZLO 4
#define TMG_FACE_ZHI 5

typedef struct tmg_ctx tmg_ctx;

/* GridSpec (grid.hpp:30-55) + build_hierarchy(spec, ncc, sd) (grid.hpp:127-129). */
typedef struct {
  int64_t nx, ny, nz;
  double lx, ly, lz;
  int64_t ncc[3];
  int64_t sd;
} tmg_grid;

/* DirichletPatch (grid.hpp:61-66). */
typedef struct {
  int face;
  double u0, v0, u1, v1, value;
} tmg_patch;

/* MmgOptions (solver.hpp:141-146) + PrecondKind. Zero eig_* fields select
 * the defaults of the batched local eigensolver. */
typedef struct {
  int kind;
  int64_t num_local_basis; /* L_c  (reference default 4) */
  int64_t num_cc_basis;    /* L_cc (reference default 8) */
  int smoother_sweeps;     /* nu   (reference default 1) */
  double eig_tol;      /* residual tolerance relative to ||B||, 0 -> 1e-9 */
  int eig_degree;      /* Chebyshev filter degree, 0 -> 32 */
  int eig_max_outer;   /* filter/Rayleigh-Ritz rounds, 0 -> 60 */
  int warm_start;      /* 1: start the local eigensolver from the previous set-up's
                          bases (same context; a design iteration's re-set-up) */
  int fine_blocks;     /* fine smoother partition (mmg, two_grid):
                          TMG_FINE_BLOCKS_CC (0, the default: build_mmg's
                          fine_blocks_by_cc, solver.cpp:353-361, one exact block per
                          cc element: 8^3, 16^3 or 32^3 cells with cubic 4^3 / 8^3
                          coarse cells, any element whose z planes hold <= 4096
                          cells otherwise; TMG_ENOTSUP beyond, or when the block
                          factors exceed device memory) or TMG_FINE_BLOCKS_COARSE_CELL (1, opt-in: one
                          block per coarse cell, the fast GPU partition of
                          DESIGN.md §2; the reference builds it through
                          build_hierarchy_operators, solver.hpp:132-135) */
} tmg_mmg_options;

#define TMG_FINE_BLOCKS_CC 0
#define TMG_FINE_BLOCKS_COARSE_CELL 1

/* SolveReport (solver.hpp:15-22). */
typedef struct {
  int iterations;
  int converged;
  int status; /* 0 running,1 converged,2 max iterations,3 zero rhs,4 indefinite,5 non-finite,
                 6 true residual at the FP64 floor (TMG_SOLVE_TRUE_RESIDUAL) */
  double setup_seconds;
  double solve_seconds;
  double final_relative_residual; /* ||r||/||b|| of the recurrence residual */
  int restarts;                   /* residual replacements (TMG_SOLVE_TRUE_RESIDUAL) */
} tmg_report;

/* Context ------------------------------------------------------------------ */

/* Validates the hierarchy like build_hierarchy (grid.cpp:196-218; ConfigError
 * on non-divisible axes) and allocates the context on CUDA device `device`.
 * Any coarse-cell shape cells_per_c = n / (ncc sd) per axis is accepted up to
 * 2^20 fine cells per coarse cell (TMG_ENOTSUP above): cubic 4^3 / 8^3 run
 * the tuned kernels, every other shape (non-cubic, 2^3, 12^3, 17^3 with the
 * reference's Lanczos-path ordering above 4096 cells, ...) the generic ones
 * (csrc/generic.cu); TMG_FORCE_GENERIC=1 in the environment forces the
 * generic kernels for 4^3 / 8^3 too (A/B tests). */
int tmg_create(const tmg_grid* grid, int device, tmg_ctx** out);
void tmg_destroy(tmg_ctx* ctx);

/* Partitioned solves; no reference counterpart (the
 * reference is shared-memory only). The grid is split along z into slabs of
 * whole cc-element layers (the slab count must divide ncc[2]); a slab keeps
 * one ghost brick layer per neighbour, refreshed by halo exchanges, and the
 * CG dot products / the coarse-coarse right-hand side are reduced across
 * slabs. Iteration counts match the single-slab solve (the smoother blocks
 * never straddle slabs); dot products differ only in summation order.
 *
 * tmg_create_slabs: `nslabs` slabs in one process on one device, exchanged
 *   by device copies (the partitioned data path on a single GPU). Host arrays
 *   stay global.
 * tmg_create_dist: slab `rank` of `nranks`, one process per GPU, exchanges
 *   and reductions over NCCL. `nccl_id` = the bytes of tmg_nccl_unique_id()
 *   made on rank 0 and broadcast by the caller. Every host array passed to
 *   this context is the rank's own slab: cells x-fastest with z in
 *   [out[0], out[1]) of tmg_partition(). */
int tmg_create_slabs(const tmg_grid* grid, int device, int nslabs, tmg_ctx** out);
int tmg_nccl_unique_id(void* id, int bytes); /* bytes >= 128 */
int tmg_create_dist(const tmg_grid* grid, int device, int rank, int nranks, const void* nccl_id,
                    tmg_ctx** out);
/* Host-only: slab `rank` of `nranks`. out[10] = {first fine z, end fine z,
 * first brick, bricks, first cc element, cc elements, first x-fastest cell,
 * cells, has neighbour below, has neighbour above}. */
int tmg_partition(const tmg_grid* grid, int nranks, int rank, int64_t* out);
/* The halo exchange of slab `rank` as exchange() issues it over NCCL:
 * returns the number of operations (<= 4, or -error), each 4 int64 in ops:
 * {1 = send / 0 = receive, peer rank, first global unit, units}, units =
 * bricks (elem = 0) or cc elements (elem = 1), one z-layer per neighbour.
 * Host-only (no GPU). */
int tmg_halo_plan(const tmg_grid* grid, int nranks, int rank, int elem, int64_t* ops,
                  int max_ops);
/* Message of the last failed call on this context (or of tmg_create when ctx
 * is NULL). */
const char* tmg_last_error(const tmg_ctx* ctx);

/* Problem ------------------------------------------------------------------ */

/* Conductivity per cell + Dirichlet patches: the inputs of assemble_system
 * (fvm.cpp:33-51: ConfigError on kappa <= 0, bad patches, or no Dirichlet
 * face). The operator A is then applied matrix-free from kappa. */
int tmg_set_conductivity(tmg_ctx* ctx, const double* kappa, const tmg_patch* patches,
                         int npatches);
/* SIMP design (rho per cell) -> kappa on the device, MaterialModel +
 * conductivity (material.cpp:8-15,45-59). */
/* Seeded synthetic design (SURVEY.md §8(d) "Synthetic inputs", §8(f) rank 3):
 * Lcg64(seed) uniforms (rng.hpp:17-25), `passes` box means of radius `radius`
 * over the clipped (2r+1)^3 window, the ceil(vf M) largest -> 1 with ties by
 * lower index (rng.cpp:39-51). Bit-identical to inputs.box_filter_design. */
typedef struct {
  double vf;
  uint64_t seed;
  int passes;
  int radius;
} tmg_design_gen;

/* Generates the design on the device (every rank of a partitioned solve
 * generates the whole field and keeps its slab), then as tmg_set_design.
 * rho_out (nullable): the whole design, x-fastest, on the host. */
int tmg_set_design_generated(tmg_ctx* ctx, const tmg_design_gen* gen, double kappa_lo,
                             double kappa_hi, int p, const tmg_patch* patches, int npatch,
                             double* rho_out);

/* frozen_bench_design (rng.cpp:16-53, the reference's bench design) on the
 * device: Lcg64(seed) uniforms, `passes` 7-point averaging sweeps, the
 * ceil(vstar M) largest -> 1 (ties by lower index); bit-identical to the
 * reference's. Then as tmg_set_design; rho_out (nullable) gets the design. */
int tmg_set_design_frozen(tmg_ctx* ctx, double vstar, uint64_t seed, int passes, double kappa_lo,
                          double kappa_hi, int p, const tmg_patch* patches, int npatch,
                          double* rho_out);

/* BASELINE configs[4]'s "seeded tree-like binary field" (no reference
 * generator exists, inputs.tree_design restates it): a binary
 * tree of `depth` levels of capsule segments rooted at the centre of the z = 0
 * face, built from Lcg64(seed ^ 0x9E3779B97F4A7C15) in breadth-first order in
 * the frame of the domain [0, dom]^3 (dom = 0: the context's own extents);
 * field = max over segments of (1 - distance / width)_+ + amp * u (u the
 * design generator's LCG noise), then `passes` box means of `radius` and the
 * ceil(vf M) largest -> 1 (ties by lower index, rng.cpp:39-51). The cell
 * centres are the context's own, so a slab context whose domain is the bottom
 * of dom (e.g. 1024 x 1024 x 128 cells of extent 1 x 1 x 0.125 in the unit
 * cube) gets the bottom slab of the tree; with global_n the design is the
 * global one's slab exactly (its threshold is the whole domain's). */
typedef struct {
  double vf;
  uint64_t seed;
  int passes;
  int radius;
  int depth;       /* tree levels: 2^depth - 1 segments (<= 12) */
  double length0;  /* root segment length (domain units); level k: length0 * lshrink^k */
  double lshrink;
  double width0;   /* root capsule radius; level k: width0 * wshrink^k */
  double wshrink;
  double spread;   /* child direction = normalize(parent + spread * (u - 1/2)^3) */
  double amp;      /* noise amplitude */
  double dom[3];   /* extents of the whole domain the tree lives in (0: own) */
  int64_t global_n[3]; /* nonzero: generate the whole design on global_n cells over
                          dom (field, filter and top-k threshold of the global
                          problem) and keep z-layers [z0, z0 + nz) */
  int64_t z0;
} tmg_tree_gen;

int tmg_set_design_tree(tmg_ctx* ctx, const tmg_tree_gen* gen, double kappa_lo, double kappa_hi,
                        int p, const tmg_patch* patches, int npatch, double* rho_out);

int tmg_set_design(tmg_ctx* ctx, const double* rho, double kappa_lo, double kappa_hi, int p,
                   const tmg_patch* patches, int npatches);
/* interpolate_design (grid.cpp:220-241) on the device: piecewise-constant
 * prolongation of a field on a coarser grid n_lo[3] (x-fastest; every axis
 * an integer factor of the context's grid, else TMG_ECONFIG).
 * tmg_set_x0_interpolated: into the resident x, the warm start of the next
 *   tmg_solve_resident(..., use_x0 = 1) (a coarse solve's T as initial guess).
 * tmg_set_design_interpolated: prolongs rho, then as tmg_set_design (the
 *   continuation step of optimize, optim.cpp:288-295). */
int tmg_set_x0_interpolated(tmg_ctx* ctx, const double* x_lo, const int64_t* n_lo);
int tmg_set_design_interpolated(tmg_ctx* ctx, const double* rho_lo, const int64_t* n_lo,
                                double kappa_lo, double kappa_hi, int p,
                                const tmg_patch* patches, int npatches);

/* sensitivity (optim.cpp:21-84) on the device: the adjoint gradient of the
 * mean temperature per cell for design rho, state t and adjoint u (the LS2
 * solution with rhs adjoint_rhs = 1/M, optim.cpp:16-19), with the
 * MaterialModel (kappa_lo, kappa_hi, f0, p) and the context's conductivity
 * and Dirichlet patches. Bitwise equal to the reference. */
int tmg_sensitivity(tmg_ctx* ctx, const double* rho, double kappa_lo, double kappa_hi, double f0,
                    int p, const double* t, const double* u, double* grad);

/* The rhs of assemble_system (fvm.cpp:63-112): f*vol + Dirichlet terms.
 * source may be NULL (f = 0). */
int tmg_assemble_rhs(tmg_ctx* ctx, const double* source, double* rhs_out);

/* SIMP design loop on the device (BASELINE configs[2]) ------
 * One design iteration = density filter (linear hat, radius rmin cells) ->
 * kappa = MaterialModel(kappa_lo, kappa_hi, p) -> make_preconditioner ->
 * state solve LS1 (source f = `source` per cell) and adjoint solve LS2
 * (rhs 1/M, optim.cpp:16-19), each warm-started from its previous solution ->
 * sensitivity (optim.cpp:21-84, design-independent source) -> filter
 * transpose -> optimality-criteria update (move limit `move`, bisection on
 * the volume multiplier for mean(filtered x) = volfrac). The filter and OC
 * rules are builder-defined (the reference's outer loop uses MMA,
 * optim.cpp:121-345). Single-slab contexts; the problem's patches are those
 * of the last tmg_set_conductivity / tmg_set_design call. */
typedef struct {
  double volfrac;    /* target mean of the filtered design */
  double rmin;       /* filter radius in cells (configs[2]: 1.5) */
  double move;       /* OC move limit (configs[2]: 0.2) */
  double kappa_lo, kappa_hi;
  int p;             /* SIMP penalisation */
  double source;     /* uniform heat source f */
  double rtol;       /* PCG tolerance of LS1 / LS2 */
  int maxit;
} tmg_simp_options;

typedef struct {
  int iteration;
  double cost;       /* mean temperature of LS1 (mean_temperature, optim.cpp:10-14) */
  double volume;     /* mean filtered design before the update */
  double change;     /* ||x_new - x||_inf */
  int ls1_iterations, ls2_iterations;
  double setup_seconds, ls1_seconds, ls2_seconds, step_seconds;
} tmg_simp_report;

/* rho0 = initial design (x-fastest, NULL -> uniform volfrac). */
int tmg_simp_init(tmg_ctx* ctx, const tmg_simp_options* opts, const tmg_mmg_options* mmg,
                  const double* rho0);
int tmg_simp_step(tmg_ctx* ctx, tmg_simp_report* report);
/* filtered design ("physical" densities) and the last state solution */
int tmg_simp_download(tmg_ctx* ctx, double* xphys, double* temperature);

/* The reference's design loop (topmg::optimize, optim.cpp:240-345) on one
 * resolution level, resident on the device: per iteration the design's
 * conductivity and heat source (material.cpp:45-66), a preconditioner set-up
 * (mmg options as given; the reference rebuilds it from scratch), LS1 and LS2
 * (adjoint_rhs) from zero, mean temperature, sensitivity (optim.cpp:21-84)
 * and the single-constraint MMA update (mma_update, :121-220) clamped to
 * [0, 1]. The level schedule and design prolongation between levels
 * (interpolate_design, grid.cpp:220-241) stay with the host caller
 * (paper_2410_06850_b200/optim.py mirrors optimize()). */
typedef struct {
  double vstar;                /* OptimConfig::vstar (reference default 0.05) */
  double move_limit, asy_init, asy_incr, asy_decr; /* MmaOptions: 0.2, 0.5, 1.2, 0.7 */
  double kappa_lo, kappa_hi, f0; /* MaterialModel */
  int p;
  double rtol;                 /* OptimConfig::rtol (1e-6) */
  int maxit;                   /* OptimConfig::maxit (10000) */
  int warm_start;              /* 0: as the reference (cold set-up, x0 = 0); 1: warm-started
                                  local eigensolver and solves from the previous T / U */
} tmg_optim_options;

/* IterationLog (optim.hpp:74-84) plus the update's ||dx||_inf and multiplier. */
typedef struct {
  int iter;
  double cost, volume;
  int ls1_iters, ls2_iters;
  double setup_seconds, ls1_seconds, ls2_seconds;
  double dx_inf, lambda, step_seconds;
} tmg_iteration_log;

/* x0: initial design (x-fastest); NULL -> uniform vstar. Resets the MMA
 * state (MmaState, optim.hpp:35-40). The context's boundary patches are used. */
int tmg_optim_init(tmg_ctx* ctx, const tmg_optim_options* opts, const tmg_mmg_options* mmg,
                   const double* x0);
/* One MMA iteration. A state/adjoint solve that does not converge returns
 * TMG_ESOLVER with the reference's failure message; the design is unchanged. */
int tmg_optim_step(tmg_ctx* ctx, tmg_iteration_log* log);
/* Evaluation solve of the current design (LS1 only): log->cost = final cost. */
int tmg_optim_evaluate(tmg_ctx* ctx, tmg_iteration_log* log);
/* current design and the last state solution (x-fastest; either nullable) */
int tmg_optim_download(tmg_ctx* ctx, double* x, double* temperature);

/* Preconditioner set-up: make_preconditioner (solver.cpp:462-481). */
int tmg_setup(tmg_ctx* ctx, const tmg_mmg_options* opts);

/* Solve -------------------------------------------------------------------- */

/* topmg::pcg (solver.cpp:483-575): same stopping rule ||r||/||b|| <= rtol on
 * the recurrence residual, same failure (pAp <= 0 -> TMG_ESOLVER), x0 may be
 * NULL (zero start). history (nullable) receives max_iterations entries at
 * most, the relative residual after each iteration. Host buffers. */
int tmg_pcg(tmg_ctx* ctx, const double* b, const double* x0, double rtol, int max_iterations,
            double* x_out, double* history, tmg_report* report);

/* y = A x, SparseOperator::apply on the assembled TPFA matrix (sparse.cpp:71-84). */
int tmg_apply_operator(tmg_ctx* ctx, const double* x, double* y);
/* y = |A| |x| (every stencil term made nonnegative; no reference
 * counterpart): eps ||(|A||x|)|| / ||b|| is the rounding floor of any FP64
 * residual b - A x of x. */
int tmg_apply_operator_abs(tmg_ctx* ctx, const double* x, double* y);
/* z = M r, Preconditioner::apply (solver.hpp:28). */
int tmg_apply_preconditioner(tmg_ctx* ctx, const double* r, double* z);

/* Device-resident variant used by the benchmark: b stays in HBM between
 * solves; tmg_solve_resident times only the device solve. */
int tmg_upload_rhs(tmg_ctx* ctx, const double* b);
int tmg_upload_x0(tmg_ctx* ctx, const double* x0);
int tmg_solve_resident(tmg_ctx* ctx, double rtol, int max_iterations, int use_x0,
                       tmg_report* report);
/* tmg_solve_resident with flags. TMG_SOLVE_TRUE_RESIDUAL (no reference
 * counterpart; the reference stops on the recurrence residual,
 * solver.cpp:549-560): after the recurrence meets rtol, the true residual
 * b - A x is formed on the device and, while it exceeds rtol, the solve
 * restarts from it (residual replacement): at most 4 restarts, and none once
 * a restart no longer halves it (the FP64 floor eps |A||x| / |b| of the
 * problem is above rtol: status 6). report->converged then
 * means TRUE residual <= rtol; final_relative_residual is the true relative
 * residual of the returned x; iterations and solve_seconds cover every
 * restart; restarts counts them. The history buffer holds the last restart. */
#define TMG_SOLVE_TRUE_RESIDUAL 1
int tmg_solve_resident_ex(tmg_ctx* ctx, double rtol, int max_iterations, int use_x0, int flags,
                          tmg_report* report);
int tmg_download_solution(tmg_ctx* ctx, double* x);

/* Introspection / measurement ------------------------------------------- */

/* Fine smoother factor slots after tmg_setup (per-coarse-cell fine blocks):
 * interior bricks whose cells and face halo carry one conductivity share one
 * scaled factor, so slots <= bricks ("shared factors"). */
int tmg_get_fine_factor_slots(tmg_ctx* ctx, int64_t* slots, int64_t* bricks);
/* Local bases in the reference's R_c row order: phi[(I*Lc + a)*cells + i] is
 * entry i (cells_of_coarse order) of basis a of coarse cell I; evals[I*Lc+a]. */
int tmg_get_local_bases(tmg_ctx* ctx, double* phi, double* evals, int* eig_iterations);
/* Dense coarse operator A_c (n_c x n_c, n_c = L_c * m_c, R_c row order). */
int tmg_get_coarse_operator(tmg_ctx* ctx, double* ac_dense);
/* R_cc as dense (n_cc x n_c). */
int tmg_get_cc_restriction(tmg_ctx* ctx, double* rcc_dense);
/* Sizes: [M, m_c, n_c, m_cc, n_cc, cells_per_coarse]. */
int tmg_get_sizes(tmg_ctx* ctx, int64_t* sizes6);
/* One solve launching every kernel separately with CUDA events around each
 * (names: search, update, restrict, coarse_down, gemv, coarse_up, post,
 * jacobi_step, init). ms_total[k] / count[k] per kernel k (9 slots). */
int tmg_profile_solve(tmg_ctx* ctx, double rtol, int max_iterations, double* ms_total,
                      int* count);
/* Bytes of device memory held by the context. */
int64_t tmg_device_bytes(const tmg_ctx* ctx);
/* Kernels enqueued by this context's solves so far (graph nodes included,
 * kernels that exit early after convergence included). */
int64_t tmg_kernel_launches(const tmg_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) for external event timing. */
void* tmg_stream(tmg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
