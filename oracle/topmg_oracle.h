/*
 * ORACLE — test infrastructure only.
 *
 * A plain-C CPU restatement of the reference's linear-solve hot path
 * (proj/core/src/{grid,material,fvm,sparse,coarse_space,solver}.cpp). Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it,
 * and only as the checker. The product path (paper_2410_06850_b200/) never
 * links or calls it.
 *
 * Pinned against the reference compiled here (oracle/_ref, see
 * oracle/build_ref.sh and DESIGN.md "Oracle") and against the spec's known
 * answers (tests/test_oracle.py).
 */
#ifndef TOPMG_ORACLE_H
#define TOPMG_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef int64_t orc_index;

enum { ORC_OK = 0, ORC_ECONFIG = 1, ORC_ESOLVER = 2, ORC_EARG = 3 };

/* GridSpec (proj/core/include/topmg/grid.hpp:30-55) */
typedef struct {
  orc_index nx, ny, nz;
  double lx, ly, lz;
} orc_grid;

/* DirichletPatch (grid.hpp:61-66); face: 0 XLo,1 XHi,2 YLo,3 YHi,4 ZLo,5 ZHi */
typedef struct {
  int face;
  double u0, v0, u1, v1, value;
} orc_patch;

/* SparseOperator CSR (sparse.hpp:21-74); int64 indices, sorted columns */
typedef struct {
  orc_index rows, cols;
  orc_index* off;
  orc_index* col;
  double* val;
} orc_csr;

/* HierarchicalGrid (grid.hpp:93-134) */
typedef struct {
  orc_grid spec;
  orc_index ncc[3];
  orc_index sd;
  orc_index nc[3];
  orc_index cpc[3]; /* cells_per_c */
} orc_hgrid;

/* Preconditioner kinds: PrecondKind (solver.hpp:160) + smoother partition.
 * fine/coarse block partition for the MMG smoothers:
 *   ORC_BLOCKS_CC    — reference default: one block per cc element
 *                      (fine_blocks_by_cc / coarse_blocks_by_cc, solver.cpp:353-374)
 *   ORC_BLOCKS_POINT — singleton fine blocks (point Jacobi)
 *   ORC_BLOCKS_CELL  — one L_c x L_c block per coarse cell (coarse level)
 * The pinned GPU variant is fine=POINT, coarse=CELL. */
enum { ORC_NONE = 0, ORC_JACOBI = 1, ORC_BLOCK_JACOBI = 2, ORC_TWO_GRID = 3, ORC_MMG = 4 };
enum { ORC_BLOCKS_CC = 0, ORC_BLOCKS_POINT = 1, ORC_BLOCKS_CELL = 2, ORC_BLOCKS_BOX0 = 16 /* + b: b^3 boxes */ };

typedef struct orc_precond orc_precond;

typedef struct {
  int iterations;
  int converged;
  double solve_seconds;
  double setup_seconds;
} orc_report;

/* ---- last error text (thread-local) ---- */
const char* orc_last_error(void);

/* ---- grid / boundary (grid.cpp) ---- */
int orc_build_hierarchy(const orc_grid* g, const orc_index ncc[3], orc_index sd,
                        orc_hgrid* out);
int orc_dirichlet_value(const orc_grid* g, const orc_patch* p, int np,
                        orc_index i, orc_index j, orc_index k, int face,
                        double* value);
orc_index orc_count_dirichlet_faces(const orc_grid* g, const orc_patch* p, int np);
int orc_interpolate_design(const double* lo, const orc_grid* glo,
                           const orc_grid* ghi, double* hi);

/* ---- material / inputs ---- */
int orc_conductivity(orc_index n, const double* x, double kappa_lo,
                     double kappa_hi, int p, double* kappa);
/* rng.cpp:16-53 (reference frozen_bench_design) */
void orc_frozen_bench_design(const orc_grid* g, double vstar, uint64_t seed,
                             int passes, double* rho);
/* BASELINE.json generator (new, M4): LCG uniforms, `passes` box-mean filters
 * of radius r over the clipped (2r+1)^3 window, top ceil(vf*M) -> 1. */
void orc_box_filter_design(const orc_grid* g, double vf, uint64_t seed,
                           int passes, int radius, double* rho);

/* ---- assembly (fvm.cpp:33-166) ---- */
int orc_assemble(const orc_grid* g, const double* kappa, const double* source,
                 const orc_patch* p, int np, orc_csr* a, double* rhs);
void orc_csr_free(orc_csr* a);
void orc_spmv(const orc_csr* a, const double* x, double* y);

/* ---- coarse spaces (coarse_space.cpp) ---- */
/* local_spectral_basis: values[count], vectors column-major (cells x count). */
int orc_local_basis(const orc_hgrid* h, const double* kappa, orc_index coarse_id,
                    orc_index count, double* values, double* vectors);
/* cc basis: projected matrix eigenpairs; vectors column-major (q x count). */
int orc_cc_basis(const orc_hgrid* h, const double* kappa, const orc_csr* rc,
                 orc_index cc_id, orc_index count, double* values,
                 double* vectors);
int orc_build_coarse_spaces(const orc_hgrid* h, const double* kappa,
                            orc_index lc, orc_index lcc, orc_csr* rc,
                            orc_csr* rcc);
/* Galerkin R A R^T (sparse.cpp:261-270) */
int orc_galerkin(const orc_csr* r, const orc_csr* a, orc_csr* out);

/* ---- preconditioners + PCG (solver.cpp) ---- */
int orc_make_preconditioner(int kind, const orc_csr* a, const orc_hgrid* h,
                            const double* kappa, orc_index lc, orc_index lcc,
                            int sweeps, int fine_blocks, int coarse_blocks,
                            orc_precond** out);
void orc_precond_free(orc_precond* m);
int orc_precond_apply(const orc_precond* m, const double* r, double* z);
/* Access the hierarchy's operators (NULL if not MMG/two-grid). */
const orc_csr* orc_precond_op(const orc_precond* m, int which); /* 0 A,1 Rc,2 Rcc,3 Ac,4 Acc */

int orc_pcg(const orc_csr* a, const double* b, const orc_precond* m,
            double rtol, int max_iterations, const double* x0 /*nullable*/,
            double* x, double* history /*nullable, max_iterations*/,
            orc_report* rep);

#ifdef __cplusplus
}
#endif
#endif
