// Host-visible launchers of the device kernels (one translation unit each).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <map>
#include <vector>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <cuda_runtime.h>

#include "common.cuh"

namespace tmg {

// Boundary forms of the fine restriction / post-smoothing;
// build with -DTMG_RESTRICT_BND=0 / -DTMG_POST_BND=0 for the literal kernels.
// The boundary kernels read r1 only on the brick face layers (r1f); the full
// r1 is written and exchanged only when a literal kernel needs it.
#ifndef TMG_RESTRICT_BND
#define TMG_RESTRICT_BND 1
#endif
#ifndef TMG_POST_BND
#define TMG_POST_BND 1
#endif
#define TMG_R1_FULL (!(TMG_RESTRICT_BND && TMG_POST_BND))

// PDL on unless TMG_NO_PDL is set (A/B diagnostics)
inline bool pdl_enabled() {
  static const bool on = getenv("TMG_NO_PDL") == nullptr;
  return on;
}

// A failed launch throws; the C ABI's guard() turns it into TMG_ECUDA with
// the message (the launchers run inside every tmg_* entry point's guard).
inline void launch_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                             cudaGetErrorString(e) + ")");
}

// SM count of the current device (cached per device ordinal).
inline int device_sm_count() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  launch_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 0;
  launch_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev),
               "cudaDeviceGetAttribute");
  cache[dev] = sms;
  return sms;
}

// Raise `kernel`'s dynamic shared-memory limit on the current device to at
// least `smem` (the attribute is per device and per function; it is never
// lowered, so launches of the same kernel with different sizes all stay
// valid).
template <typename K>
inline void ensure_dyn_smem(K kernel, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> limit;
  if (smem <= 48 * 1024) return;
  int dev = 0;
  launch_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = limit[std::make_pair(dev, (const void*)kernel)];
  if (smem <= cur) return;
  launch_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "cudaFuncSetAttribute");
  cur = smem;
}

// Resident CTAs per SM of `kernel` with `smem` dynamic bytes on the current
// device (after ensure_dyn_smem). Cached per (device, kernel, threads, smem).
template <typename K>
inline int device_occupancy(K kernel, int threads, size_t smem) {
  ensure_dyn_smem(kernel, smem);
  static std::mutex mu;
  static std::map<std::pair<std::pair<int, const void*>, std::pair<int, size_t>>, int> cache;
  int dev = 0;
  launch_check(cudaGetDevice(&dev), "cudaGetDevice");
  const auto key = std::make_pair(std::make_pair(dev, (const void*)kernel),
                                  std::make_pair(threads, smem));
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per = 0;
  launch_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem),
               "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  cache[key] = per < 1 ? 1 : per;
  return cache[key];
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (e != cudaSuccess) {  // name the kernel (with CUDA_LAUNCH_BLOCKING=1: the faulting one)
    const char* name = nullptr;
    if (cudaFuncGetName(&name, (const void*)kernel) != cudaSuccess || !name) name = "?";
    launch_check(e, (std::string("kernel launch ") + name).c_str());
  }
}

enum : int {
  kStatusRunning = 0,
  kStatusConverged = 1,
  kStatusMaxIt = 2,
  kStatusZeroRhs = 3,
  kStatusIndefinite = 4,
  kStatusNonFinite = 5,
  kStatusFloor = 6,  // TMG_SOLVE_TRUE_RESIDUAL: true residual stuck above rtol
};

// Per-brick exact fine blocks (smoother.cuh): brick b's plane inverses are
// at G + map[b].slot * PER_BRICK (scale 1). Interior bricks whose cells and
// face halo carry one conductivity k have A_II = face_t(k, k) A_hat with
// A_hat = sum over axes of (area/h) times the 1-D Dirichlet Laplacian: they
// store no factor (slot -1) and are solved by fast diagonalisation with
// scale 1 / face_t(k, k) (smoother.cuh, brick_inverse).
struct GSlot {
  int64_t slot;
  double scale;
};
struct FineFactors {
  const double* G;
  const GSlot* map;  // virtual global (indexed by brick)
};

// Device-resident CG scalars (one per solve context).
struct PcgState {
  double bnorm, rnorm, rho, alpha, beta, pq, rtol;
  int it, maxit, done, status, first, hist_cap;
  unsigned int ticket[8];
  // partitioned solves (GridParams::dist): each reduction kernel leaves its
  // local total here; the cross-slab sum (in-process or NCCL all-reduce)
  // overwrites it and k_finalize applies the same scalar logic.
  double loc[8];
};

// PcgState::loc slots and k_finalize selectors
enum : int { kRedInit = 0, kRedSearch = 2, kRedUpdate = 3, kRedPost = 4, kRedJacobi = 5 };
constexpr int kMaxSlabs = 64;
struct FinArgs {
  PcgState* st[kMaxSlabs];
  double* hist[kMaxSlabs];
  int ns;
};

// operator.cu
void launch_to_brick(const GridParams& g, int cb, const double* src, double* dst, cudaStream_t s);
void launch_from_brick(const GridParams& g, int cb, const double* src, double* dst, cudaStream_t s);
// interpolate_design (grid.cpp:220-241) into the own cells of dst
void launch_interpolate(const GridParams& g, int cb, const double* lo, const int64_t* nlo,
                        double* dst, cudaStream_t s);
void launch_conductivity(const GridParams& g, int cb, const double* x, double* kappa, double lo,
                         double hi, int p, cudaStream_t s);
void launch_boundary(const GridParams& g, int cb, const Patch* patches, int npatch, double lx,
                     double ly, double lz, const double* kappa, const double* source,
                     uint8_t* dmask, double* rhs, unsigned long long* count, cudaStream_t s);
// sensitivity (optim.cpp:21-84) into grad (own cells; t and u ghosts filled)
void launch_sensitivity(const GridParams& g, int cb, const Patch* patches, int npatch, double lx,
                        double ly, double lz, const double* rho, const double* kappa,
                        const double* t, const double* u, double kappa_lo, double kappa_hi,
                        double f0, int p, double* grad, cudaStream_t s);
// y = |A| |x| (entrywise absolute values; the FP64 residual floor)
void launch_apply_abs(const GridParams& g, int cb, const double* coef, const double* x, double* y,
                      cudaStream_t s);
void launch_apply(const GridParams& g, int cb, const double* coef, const double* x, double* y,
                  double* dinv, cudaStream_t s);

// setup_fine.cu
// factor slot i of G <- brick list[i] (list: nslots bricks)
void launch_thomas_factor(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                          const int64_t* list, int64_t nslots, double* G, int* status,
                          cudaStream_t s);
int64_t thomas_doubles_per_brick(int cb);
// shared factors of uniform bricks: flag[b - b0] = 1 for an interior brick
// whose cells and face halo have bitwise one conductivity
void launch_uniform_bricks(const GridParams& g, int cb, const double* kappa, int* flag,
                           cudaStream_t s);
// map[b].scale = 1 / face_t(k_b, k_b) for the flagged (shared) bricks, 1
// otherwise (slots already set)
void launch_factor_scales(const GridParams& g, int cb, const double* kappa, const int* flag,
                          GSlot* map, cudaStream_t s);

// spectral.cu
// phi0: previous bases as the initial block (warm start) or nullptr
// list: the bricks to solve (nlist of them), nullptr = every owned brick
void launch_local_basis(const GridParams& g, int cb, const double* kappa, const double* phi0,
                        double* phi, double* evals, int* iters, double tol, int degree,
                        int max_outer, const int64_t* list, int64_t nlist, cudaStream_t s);
// bricks of one uniform conductivity inside: flag[b - b0] = 1
void launch_uniform_inside(const GridParams& g, int cb, const double* kappa, int* flag,
                           cudaStream_t s);
// bases of the flagged bricks in closed form (separable DCT-II modes)
void launch_local_basis_uniform(const GridParams& g, int cb, const double* kappa, const int* flag,
                                double* phi, double* evals, int* iters, cudaStream_t s);

// coarse.cu
int max_lc();  // largest supported L_c (num_local_basis)
void launch_coarse_blocks(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                          const double* phi, double* Ac, double* Bc, cudaStream_t s);
void launch_cc_basis(const GridParams& g, const double* Ac, const double* Bc, double* Rcc,
                     double* cc_evals, cudaStream_t s);
void launch_coarse_smoother(const GridParams& g, const double* Ac, double* Winv, int* status,
                            cudaStream_t s);
void launch_cc_identity(const GridParams& g, double* Rcc, double* cc_evals, cudaStream_t s);
// A_cc as a block Thomas over the cc-element z-planes (acc_planes.cu)
struct AccRowBlock {  // rows [r0, r0 + nr) of every plane inverse: R[k][nr][P]
  const double* R;
  int64_t r0, nr;
};
void launch_acc_rows_solve(const GridParams& g, const int* done, const double* C,
                           const double* rcc, double* ecc, double* wv,
                           const std::vector<AccRowBlock>& blocks,
                           const std::function<void(double* plane)>& gather, cudaStream_t s);
int acc_rows_solve_kernels(const GridParams& g, int nblocks);
// y[0..nrows) = A x for a dense nrows x ncols block (one warp per row)
void launch_gemv_block(const int* done, const double* A, int64_t nrows, int64_t ncols,
                       const double* x, double* y, cudaStream_t s);
struct AccPlanesRef {
  const double* T;  // ncz packed symmetric plane inverses
  const double* C;  // z-lo coupling blocks [element][L_cc][L_cc]
  double* wv;       // 2 P work doubles
};
int64_t acc_planes_doubles(const GridParams& g);
void launch_acc_assemble_planes(const GridParams& g, const double* Ac, const double* Rcc,
                                double* Gd, double* C, cudaStream_t s, bool zero = true);
void acc_planes_factor(const GridParams& g, double* Gd, const double* C, double* T, double* work,
                       int* status, cudaStream_t s);
void launch_acc_planes_solve(const GridParams& g, const int* done, const double* T,
                             const double* C, const double* rcc, double* ecc, double* wv,
                             double* partials, cudaStream_t s);
int acc_planes_solve_kernels(const GridParams& g);
// large cc elements (q = sd^3 L_c > 64, coarse_large.cu)
bool coarse_large_supported(int q, int lcc);
int64_t coarse_large_work_doubles(int q, int64_t neo, int lcc);
void launch_coarse_smoother_large(const GridParams& g, const double* Ac, double* Winv,
                                  double* work, int* status, cudaStream_t s);
void launch_cc_basis_large(const GridParams& g, const double* Ac, const double* Bc,
                           double* scratch, double* work, double* Rcc, double* cc_evals,
                           int* scratch_status, int* iters, double tol, int maxit,
                           cudaStream_t s);
void launch_acc_assemble(const GridParams& g, const double* Ac, const double* Rcc, double* Acc,
                         cudaStream_t s);
void launch_coarse_cycle(const GridParams& g, const int* done, const double* Ac,
                         const double* Winv, const double* Rcc, const double* Acc_tiles,
                         double* symv_partials, int64_t n_cc, const double* rc, double* rc0,
                         double* rcc, double* ecc, double* rc1, double* tc, double* ec,
                         const AccPlanesRef* planes, cudaStream_t s);

// the same cycle as one cooperative kernel (single slab; q = 32, L_cc = 8)
bool coarse_fused_supported(const GridParams& g, int64_t n_cc);
void launch_coarse_fused(const GridParams& g, const int* done, const double* Ac,
                         const double* Winv, const double* Rcc, const double* Acc_tiles,
                         double* symv_partials, int64_t n_cc, const double* rc, double* rc0,
                         double* rcc, double* rc1, double* ec, unsigned int* bar,
                         cudaStream_t s);
void launch_coarse_smooth(const GridParams& g, const int* done, const double* Winv,
                          const double* in, const double* add, double* out, cudaStream_t s);
void launch_coarse_restrict(const GridParams& g, const int* done, const double* Ac,
                            const double* Rcc, const double* rc, const double* rc0, double* rcc,
                            cudaStream_t s);
void launch_coarse_prolong(const GridParams& g, const int* done, const double* Rcc,
                           const double* rc0, const double* ecc, double* rc1, cudaStream_t s);
void launch_coarse_resid(const GridParams& g, const int* done, const double* Ac, const double* rc,
                         const double* x, double* out, cudaStream_t s);

// dense.cu
void dense_spd_inverse(double* A, int64_t n, double* work, int* status, cudaStream_t s);
int64_t dense_inverse_work_doubles(int64_t n);
const double* dense_inverse_pivots(const double* work, int64_t n, int64_t z);
void dense_spd_inverse_batched(double* A, int64_t n, int64_t batch, double* work, int* status,
                               cudaStream_t s);
void launch_gemv(const int* done, const double* A, int64_t n, const double* x, double* y,
                 cudaStream_t s);
// rows [row0, row0 + nrows) of y = A x (A n x n, row-major)
void launch_gemv_rows(const int* done, const double* A, int64_t n, int64_t row0, int64_t nrows,
                      const double* x, double* y, cudaStream_t s);
int64_t sym_tiles_doubles(int64_t n);
int64_t sym_partials_doubles(int64_t n);
void pack_sym_tiles(const double* A, int64_t n, double* T, cudaStream_t s);
void launch_symv(const int* done, const double* T, int64_t n, const double* x, double* P, double* y,
                 cudaStream_t s);

// simp.cu (x-fastest design arrays)
void launch_density_filter(int64_t nx, int64_t ny, int64_t nz, double r, const double* in,
                           const double* W, double* out, int mode, cudaStream_t s);
void launch_oc_candidate(const double* x, const double* dc, const double* dv, double lam,
                         double mv, double xmin, int64_t m, double* xnew, cudaStream_t s);
void launch_sum(const double* v, int64_t m, double* part, double* out, cudaStream_t s);
void launch_maxdiff(const double* a, const double* b, int64_t m, double* part, double* out,
                    cudaStream_t s);
int64_t sum_partials_doubles();
void launch_fill(double* p, int64_t n, double v, cudaStream_t s);

// pcg.cu
void init_kernel_attributes();
void launch_coefficients(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                         double* coef, cudaStream_t s);
// face-major T of every owned brick's 6 CB^2 face slots (k_face_t)
void launch_face_t(const GridParams& g, int cb, const double* coef, double* tf, cudaStream_t s);
void launch_init(const GridParams& g, int cb, const double* coef, const double* b, double* x,
                 int has_x0, double* r, PcgState* st, double* partials, cudaStream_t s);
void launch_search(const GridParams& g, int cb, const double* coef, const double* z,
                   const double* p_old, double* p, double* q, PcgState* st, double* partials,
                   cudaStream_t s);
// kernels launch_search enqueues (k_search + k_search_reduce on the brick kernels)
int search_kernels(int cb);
// launch_search with the coefficients recomputed from kappa (tuned bricks)
void launch_search_kappa(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                         const double* z, const double* p_old, double* p, double* q, PcgState* st,
                         double* partials, cudaStream_t s);
// out = add + A_II^{-1} in per brick (per-coarse-cell fine blocks); rdot: also
// rdot . out -> fin_post (the generic nu-sweep V-cycle)
void launch_brick_solve(const GridParams& g, int cb, const double* coef, const FineFactors& Gf,
                        const double* in, const double* add, double* out, const double* rdot,
                        PcgState* st, double* partials, int init, cudaStream_t s);
// out = add + y over the owned bricks (add nullable); rdot: rdot . out -> fin_post
void launch_add_finish(const GridParams& g, int cb, const double* y, const double* add,
                       double* out, const double* rdot, PcgState* st, double* partials, int init,
                       cudaStream_t s);
// returns the kernels enqueued (the solve kernel, plus k_reduce_fin when its grid sum is deferred)
int launch_update(const GridParams& g, int cb, const double* coef, const FineFactors& Gf, double* x,
                   const double* p, const double* q, double* r, double* r1, double* r1f, PcgState* st,
                   double* partials, double* history, int init, cudaStream_t s);
void launch_restrict(const GridParams& g, int cb, const double* coef, const double* phi,
                     const double* r, const double* r1, double* rc, const PcgState* st,
                     cudaStream_t s);
// boundary form of launch_restrict, valid when the fine blocks are the bricks
// tf: the face-major T of launch_face_t
void launch_restrict_bnd(const GridParams& g, int cb, const double* tf, const double* phif,
                         const double* r1f, double* rc, const PcgState* st, cudaStream_t s);
int launch_post(const GridParams& g, int cb, const double* coef, const double* tf, const double* phi,
                 const double* phif, const FineFactors& Gf, const double* r, const double* r1,
                 const double* r1f, const double* ec, double* z, PcgState* st, double* partials,
                 int init, cudaStream_t s);
// face-major copy of Phi on each stored brick's 6 face layers:
// phif[((b * 6 + f) * L_c + a) * CB^2 + q], q the in-face index of halo_slot
void launch_phi_faces(const GridParams& g, int cb, const double* phi, double* phif, int64_t b0,
                      int64_t nb, cudaStream_t s);
// sum PcgState::loc[which..] over the slabs in a fixed order and finish the
// reduction on every slab (partitioned solves)
void launch_finalize(const FinArgs& a, int which, int init, cudaStream_t s);
void launch_jacobi_step(const GridParams& g, int cb, const double* dinv, double* x, const double* p,
                        const double* q, double* r, double* z, PcgState* st, double* partials,
                        double* history, int init, int defer, cudaStream_t s);
// seeded designs on the device (gen.cu)
size_t gen_scratch_bytes(int64_t m);
void launch_box_filter_design(int64_t nx, int64_t ny, int64_t nz, double vf, uint64_t seed,
                              int passes, int radius, double* rho, double* f, void* scratch,
                              cudaStream_t s);
void launch_frozen_design(int64_t nx, int64_t ny, int64_t nz, double vstar, uint64_t seed,
                          int passes, double* rho, double* f, void* scratch, cudaStream_t s);
void launch_tree_design(int64_t nx, int64_t ny, int64_t nz, double lx, double ly, double lz,
                        double vf, uint64_t seed, int passes, int radius, const double* seg,
                        int nseg, double amp, double* rho, double* f, void* scratch,
                        cudaStream_t s);
// design loop with MMA (optim.cu; MmaOptions, optim.hpp:27-32)
struct MmaParams {
  double move, asy_init, asy_incr, asy_decr, xmin, xmax;
  double cgrad;  // constraint gradient (the reference's vol_grad = 1/M)
};
int mma_partials_doubles();
void launch_heat_source(const GridParams& g, int cb, const double* x, double* f, double f0, int p,
                        cudaStream_t s);
void launch_mma_asymptotes(const double* x, const double* xp, const double* xp2, double* low,
                           double* upp, int64_t n, int iteration, const MmaParams& o,
                           cudaStream_t s);
void launch_mma_dual(const double* x, const double* grad, const double* low, const double* upp,
                     int64_t n, double constraint, const MmaParams& o, double* partials,
                     unsigned int* bar, double* out, cudaStream_t s);
void launch_mma_primal(const double* x, const double* grad, const double* low, const double* upp,
                       int64_t n, const double* lam, const MmaParams& o, double* xnew,
                       double* partials, double* dx_out, cudaStream_t s);
// block-Jacobi with one block per cc element (block_jacobi.cu)
bool bj_supported(int cb, int sd);
int64_t bj_doubles_per_element(int cb, int sd);
// kernels one launch_bj_apply enqueues (1, or 2E for the per-plane E = 32 path)
int bj_apply_kernels(int cb, int sd);
// doubles of scratch the E = 32 factor (inverse work + pivot extrema) and apply
// (one value per owned cell) need; 0 for E <= 16
int64_t bj_factor_work_doubles(int cb, int sd, int64_t neo);
// work: bj_factor_work_doubles (E = 32 only, else unused)
void launch_bj_factor(const GridParams& g, int cb, const double* coef, double* G, int* status,
                      double* work, cudaStream_t s);
// ybuf: one value per owned cell, brick layout (virtual global; E = 32 only)
void launch_bj_apply(const GridParams& g, int cb, const double* coef, const double* G,
                     const double* in, const double* add, double* out, const double* rdot,
                     PcgState* st, double* partials, int init, double* ybuf, cudaStream_t s);
void launch_prolong_add(const GridParams& g, int cb, const double* phi, const double* r1,
                        const double* ec, double* r2, const PcgState* st, cudaStream_t s);
void launch_resid(const GridParams& g, int cb, const double* coef, const double* r,
                  const double* x, double* t, const PcgState* st, cudaStream_t s);

// generic.cu: any brick shape (cb = 0 at the launchers above; GridParams
// bx, by, bz give the shape). Fine-block boxes: kind 0 = bricks (one exact
// block per coarse cell), kind 1 = cc elements (fine_blocks_by_cc).
void launch_g_coefficients(const GridParams& g, const double* kappa, const uint8_t* dmask,
                           double* coef, cudaStream_t s);
// y = A x (absval: |A||x|; x, y nullable), dinv = 1/diag (nullable)
void launch_g_apply(const GridParams& g, const double* coef, const double* x, double* y,
                    double* dinv, int absval, cudaStream_t s);
void launch_g_init(const GridParams& g, const double* coef, const double* b, double* x,
                   int has_x0, double* r, PcgState* st, double* partials, cudaStream_t s);
void launch_g_search(const GridParams& g, const double* coef, const double* z, const double* p_old,
                     double* p, double* q, PcgState* st, double* partials, cudaStream_t s);
void launch_g_jacobi_step(const GridParams& g, const double* dinv, double* x, const double* p,
                          const double* q, double* r, double* z, PcgState* st, double* partials,
                          double* history, int init, int defer, cudaStream_t s);
void launch_g_resid(const GridParams& g, const double* coef, const double* r, const double* x,
                    double* t, const PcgState* st, cudaStream_t s);
void launch_g_prolong_add(const GridParams& g, const double* phi, const double* r1,
                          const double* ec, double* r2, const PcgState* st, cudaStream_t s);
void launch_g_add_finish(const GridParams& g, const double* y, const double* add, double* out,
                         const double* rdot, PcgState* st, double* partials, int init,
                         cudaStream_t s);
void launch_g_restrict(const GridParams& g, const double* coef, const double* phi, const double* r,
                       const double* r1, double* rc, const PcgState* st, cudaStream_t s);
void launch_g_coarse_blocks(const GridParams& g, const double* kappa, const uint8_t* dmask,
                            const double* coef, const double* phi, double* Ac, double* Bc,
                            cudaStream_t s);
int64_t g_local_basis_scratch_doubles(const GridParams& g);
void launch_g_local_basis(const GridParams& g, const double* kappa, const double* phi0,
                          double* phi, double* evals, int* iters, double tol, int degree,
                          int max_outer, double* scratch, cudaStream_t s);
// exact block solves on boxes: G plane-major [z][box][P][P] over the owned boxes
int64_t box_doubles(const GridParams& g, int kind);
int box_plane_cells(const GridParams& g, int kind);
int box_apply_kernels(const GridParams& g, int kind);  // plane-step launches (+1 finish)
int64_t box_factor_work_doubles(const GridParams& g, int kind);
void launch_box_factor(const GridParams& g, int kind, const double* coef, double* G, int* status,
                       double* work, cudaStream_t s);
// out = add + A_box^-1 in (add nullable); rdot: rdot . out -> fin_post;
// ybuf: one value per owned cell (brick layout, virtual global)
void launch_box_apply(const GridParams& g, int kind, const double* coef, const double* G,
                      const double* in, const double* add, double* out, const double* rdot,
                      PcgState* st, double* partials, int init, double* ybuf, cudaStream_t s);

}  // namespace tmg
