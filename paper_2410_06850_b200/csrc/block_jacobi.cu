// Block-Jacobi with one block per cc element (fine_blocks_by_cc,
// solver.cpp:353-361): the reference's block_jacobi preconditioner
// (BlockJacobiPreconditioner, solver.cpp:444-458 -- one BlockJacobiSmoother
// sweep from zero, z = A_BB^-1 r per block, solver.cpp:221-243).
//
// A block is the E^3 cells of a cc element (E = c sd), x-fastest like
// HierarchicalGrid::cells_of_coarse_coarse. In that order A_BB is block
// tridiagonal over its E z-planes of P = E^2 cells: A_kk is the plane's 2-D
// 5-point part with the full diagonal, A_k,k+1 = -D_{k+1} with D_{k+1} the
// z transmissibilities between planes k and k+1. It is factorised by block
// Thomas with explicit Schur-complement inverses
//   G_0 = A_00^-1,  G_k = (A_kk - D_k G_{k-1} D_k)^-1
// (gj_inverse_global, pivots checked with the reference's rule) and applied as
//   y_k = G_k (r_k + D_k y_{k-1}),  x_k = y_k + G_k D_{k+1} x_{k+1}.
// Storage G[e][k][P][P] (symmetric, full): 4.3 GB at 128^3 / c = 8 / sd = 2.
// Each apply streams it once (two GEMVs per plane): an HBM-bound baseline.
//
// E = 32 (32^3-cell elements: c = 8 with sd = 4, the configs[3] hierarchy;
// c = 4 with sd = 8): P = 1024, 8 MB per plane, 256 MB per element. The
// planes are stored plane-major G[k][e][P][P] so the E Schur complements of
// one plane index form one batch for the tensor-core Gauss-Jordan
// (dense_spd_inverse_batched); the LDL^T pivots of all E planes of an element
// are folded into one min / max so the reference's rule (pivot <= 1e-14 max
// over the block) applies per block. The apply runs one launch per plane
// step, each CTA computing a 128-column slice of one element's GEMV.
#include "gj_global.cuh"
#include "kernels.h"
#include "pcg_fin.cuh"
#include "stencil.cuh"

namespace tmg {

namespace {
// brick-layout offset of element cell (i, j, k)
__device__ __forceinline__ size_t elem_cell(const GridParams& g, int cb, int64_t e, int i, int j,
                                            int k) {
  const int64_t ei = e % g.ncx, ej = (e / g.ncx) % g.ncy, ek = e / (g.ncx * g.ncy);
  const int64_t b = (ei * g.sd + i / cb) + g.nbx * ((ej * g.sd + j / cb) + g.nby * (ek * g.sd + k / cb));
  return (size_t)b * (size_t)(cb * cb * cb) + (size_t)((i % cb) + cb * ((j % cb) + cb * (k % cb)));
}
}  // namespace

// One CTA (256 threads) per owned cc element; planes in sequence.
__global__ void __launch_bounds__(kGjThreads, 1) k_bj_factor(GridParams g, int cb, int E,
                                                             const double* __restrict__ coef,
                                                             double* G, int* status) {
  extern __shared__ __align__(16) double smg[];
  __shared__ GjSmem<kGjBlock> gjs;
  __shared__ double red[2][kGjThreads / 32];
  const int P = E * E, t = threadIdx.x, lane = t & 31;
  const int64_t e = blockIdx.x + g.e0, M = g.mst;
  double* Ge = G + (size_t)blockIdx.x * E * P * P;
  const GjGlobalSmem gsm = gj_global_smem(smg, P);
  double pmin = 1e300, pmax = 0.0;
  for (int k = 0; k < E; ++k) {
    double* Gk = Ge + (size_t)k * P * P;
    const double* Gp = Gk - (size_t)P * P;
    for (int idx = t; idx < P * P; idx += blockDim.x) {
      const int a = idx / P, b = idx % P;
      const int ia = a % E, ja = a / E, ib = b % E, jb = b / E;
      double v = 0.0;
      if (a == b) {
        v = coef[3 * M + elem_cell(g, cb, e, ia, ja, k)];
      } else if (ja == jb && (ib == ia + 1 || ia == ib + 1)) {
        v = -coef[elem_cell(g, cb, e, min(ia, ib), ja, k)];
      } else if (ia == ib && (jb == ja + 1 || ja == jb + 1)) {
        v = -coef[M + elem_cell(g, cb, e, ia, min(ja, jb), k)];
      }
      if (k > 0) {
        const double da = coef[2 * M + elem_cell(g, cb, e, ia, ja, k - 1)];
        const double db = coef[2 * M + elem_cell(g, cb, e, ib, jb, k - 1)];
        v -= da * Gp[idx] * db;
      }
      Gk[idx] = v;
    }
    __syncthreads();
    gj_inverse_global(Gk, P, gsm, gjs, pmin, pmax);
  }
  double mx = pmax, mn = pmin;
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if (lane == 0) {
    red[0][t >> 5] = mx;
    red[1][t >> 5] = mn;
  }
  __syncthreads();
  if (t == 0) {
    double m = 0.0, n = 1e300;
    for (int w = 0; w < kGjThreads / 32; ++w) {
      m = fmax(m, red[0][w]);
      n = fmin(n, red[1][w]);
    }
    if (!(n > 1e-14 * m)) atomicExch(status, 1);  // solver.cpp:86-92 via the smoother
  }
}

// out = add + A_BB^-1 in on every owned cc element (add nullable). With rdot
// (the PCG residual) the product rdot . out is reduced and finishes the
// iteration like the V-cycle's post kernel (fin_post: rho, beta).
// One CTA of P threads per element, thread p = plane cell (i, j).
template <int E>
__global__ void __launch_bounds__(E * E) k_bj_apply(GridParams g, int cb,
                                                   const double* __restrict__ coef,
                                                   const double* __restrict__ G,
                                                   const double* __restrict__ in,
                                                   const double* __restrict__ add, double* out,
                                                   const double* __restrict__ rdot, PcgState* st,
                                                   double* partials, int init) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  constexpr int P = E * E;
  __shared__ double y[E][P];
  __shared__ double v[P];
  __shared__ double red[80];
  __shared__ int flag;
  const int p = threadIdx.x, i = p % E, j = p / E;
  const int64_t e = blockIdx.x + g.e0, M = g.mst;
  const double* Ge = G + (size_t)blockIdx.x * E * P * P;
  auto gemv = [&](const double* Gk) {  // sum_q Gk[q][p] v[q] (Gk symmetric: coalesced)
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll 4
    for (int q = 0; q < P; q += 4) {
      s0 = fma(Gk[(size_t)q * P + p], v[q], s0);
      s1 = fma(Gk[(size_t)(q + 1) * P + p], v[q + 1], s1);
      s2 = fma(Gk[(size_t)(q + 2) * P + p], v[q + 2], s2);
      s3 = fma(Gk[(size_t)(q + 3) * P + p], v[q + 3], s3);
    }
    return (s0 + s1) + (s2 + s3);
  };
  double prev = 0.0, rz = 0.0;
  for (int k = 0; k < E; ++k) {
    const double dz = k > 0 ? coef[2 * M + elem_cell(g, cb, e, i, j, k - 1)] : 0.0;
    v[p] = in[elem_cell(g, cb, e, i, j, k)] + dz * prev;
    __syncthreads();
    prev = gemv(Ge + (size_t)k * P * P);
    y[k][p] = prev;
    __syncthreads();
  }
  double xn = y[E - 1][p];
  auto store = [&](size_t s, double xv) {
    const double o = add ? add[s] + xv : xv;
    out[s] = o;
    if (rdot) rz = fma(rdot[s], o, rz);
  };
  store(elem_cell(g, cb, e, i, j, E - 1), xn);
  for (int k = E - 2; k >= 0; --k) {
    const size_t s = elem_cell(g, cb, e, i, j, k);
    v[p] = coef[2 * M + s] * xn;
    __syncthreads();
    xn = y[k][p] + gemv(Ge + (size_t)k * P * P);
    store(s, xn);
    __syncthreads();
  }
  if (!rdot) return;
  double vv[1] = {rz};
  block_sum_k<P, 1>(vv, red);
  double tot[1];
  if (grid_reduce_last_k<1>(vv, partials, &st->ticket[5], tot, &flag, red) && p == 0) {
    if (g.dist) st->loc[kRedPost] = tot[0];
    else fin_post(st, tot[0], init);
  }
}

// r2 = r1 + R_c^T ec (solver.cpp:307-309 prolongation, per coarse cell)
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_prolong_add(GridParams g,
                                                             const double* __restrict__ phi,
                                                             const double* __restrict__ r1,
                                                             const double* __restrict__ ec,
                                                             double* r2, const PcgState* st) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  constexpr int C = CB * CB * CB;
  const int lc = g.lc;
  const int64_t b = blockIdx.x + g.b0;
  const size_t s = (size_t)b * C + threadIdx.x;
  double v = r1[s];
  for (int a = 0; a < lc; ++a) v = fma(phi[((size_t)b * lc + a) * C + threadIdx.x], ec[b * lc + a], v);
  r2[s] = v;
}

// t = r - A x (the residual before post-smoothing, solver.cpp:327)
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_resid(GridParams g, const double* __restrict__ coef,
                                                       const double* __restrict__ r,
                                                       const double* __restrict__ x, double* t,
                                                       const PcgState* st) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  __shared__ CoefSmem<CB> cs;
  __shared__ double xt[Tile<CB>::N];
  constexpr int C = CB * CB * CB;
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  load_coefs<CB>(coef, g.mst, cs, g, bc);
  load_tile<CB, true>(x, xt, g, bc);
  __syncthreads();
  const int u = threadIdx.x, li = u % CB, lj = (u / CB) % CB, lk = u / (CB * CB);
  const size_t s = bofs(bc.b, C) + u;
  t[s] = r[s] - apply_coef<CB>(cs, xt, li, lj, lk);
}

// ------------------------------------------------------ E = 32 (P = 1024)
constexpr int kE32 = 32, kP32 = kE32 * kE32, kSlice = 128, kSlices = kP32 / kSlice;

// Plane k's matrix for every owned element: A_kk - D_k G_{k-1} D_k
// (G_{k-1} already inverted in place). grid (P / 4, neo), 256 threads.
__global__ void __launch_bounds__(256) k_bj32_assemble(GridParams g, int cb,
                                                       const double* __restrict__ coef,
                                                       const double* __restrict__ Gp, double* Gk,
                                                       int k) {
  constexpr int E = kE32, P = kP32;
  const int64_t el = blockIdx.y, e = el + g.e0, M = g.mst;
  const int row0 = blockIdx.x * 4;  // 4 rows per CTA
  for (int idx = row0 * P + threadIdx.x; idx < (row0 + 4) * P; idx += 256) {
    const int a = idx / P, b = idx % P;
    const int ia = a % E, ja = a / E, ib = b % E, jb = b / E;
    double v = 0.0;
    if (a == b) {
      v = coef[3 * M + elem_cell(g, cb, e, ia, ja, k)];
    } else if (ja == jb && (ib == ia + 1 || ia == ib + 1)) {
      v = -coef[elem_cell(g, cb, e, min(ia, ib), ja, k)];
    } else if (ia == ib && (jb == ja + 1 || ja == jb + 1)) {
      v = -coef[M + elem_cell(g, cb, e, ia, min(ja, jb), k)];
    }
    if (k > 0) {
      const double da = coef[2 * M + elem_cell(g, cb, e, ia, ja, k - 1)];
      const double db = coef[2 * M + elem_cell(g, cb, e, ib, jb, k - 1)];
      v -= da * Gp[(size_t)el * P * P + idx] * db;
    }
    Gk[(size_t)el * P * P + idx] = v;
  }
}

// fold plane k's pivots into the element's extrema (ext[2 e] = min, +1 = max)
__global__ void k_bj32_fold(const double* __restrict__ work, int64_t stride, int64_t off,
                            double* ext, int k) {
  const int64_t el = blockIdx.x;
  const double* piv = work + el * stride + off;
  __shared__ double rmn[32], rmx[32];
  double mn = 1e300, mx = 0.0;
  for (int i = threadIdx.x; i < kP32; i += blockDim.x) {
    mn = fmin(mn, piv[i]);
    mx = fmax(mx, fabs(piv[i]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    rmn[threadIdx.x >> 5] = mn;
    rmx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = fmin(mn, rmn[w]);
      mx = fmax(mx, rmx[w]);
    }
    mn = fmin(mn, rmn[0]);
    mx = fmax(mx, rmx[0]);
    if (k == 0) {
      ext[2 * el] = mn;
      ext[2 * el + 1] = mx;
    } else {
      ext[2 * el] = fmin(ext[2 * el], mn);
      ext[2 * el + 1] = fmax(ext[2 * el + 1], mx);
    }
  }
}

// the reference's singular-pivot rule over the whole block (solver.cpp:86-92)
__global__ void k_bj32_check(const double* __restrict__ ext, int64_t neo, int* status) {
  for (int64_t el = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; el < neo;
       el += (int64_t)gridDim.x * blockDim.x)
    if (!(ext[2 * el] > 1e-14 * ext[2 * el + 1])) atomicExch(status, 1);
}

// One plane step of the block Thomas apply, grid (kSlices, neo), 1024
// threads: thread (qg, col) sums G_k[q][col] v[q] over 128 q of group qg.
//   fwd (bwd = 0): y_k = G_k (in_k + D_k y_{k-1})      -> ybuf plane k
//   bwd (bwd = 1): x_k = y_k + G_k (D_{k+1} x_{k+1})   -> ybuf plane k
__global__ void __launch_bounds__(1024) k_bj32_step(GridParams g, int cb,
                                                    const double* __restrict__ coef,
                                                    const double* __restrict__ G,
                                                    const double* __restrict__ in, double* ybuf,
                                                    const PcgState* st, int k, int bwd) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  constexpr int E = kE32, P = kP32;
  __shared__ double v[P];
  __shared__ double part[kSlices][kSlice];
  const int t = threadIdx.x;
  const int64_t el = blockIdx.y, e = el + g.e0, M = g.mst;
  for (int q = t; q < P; q += 1024) {
    const int i = q % E, j = q / E;
    double val;
    if (!bwd) {
      val = in[elem_cell(g, cb, e, i, j, k)];
      if (k > 0) {
        const size_t sp = elem_cell(g, cb, e, i, j, k - 1);
        val += coef[2 * M + sp] * ybuf[sp];
      }
    } else {
      val = coef[2 * M + elem_cell(g, cb, e, i, j, k)] * ybuf[elem_cell(g, cb, e, i, j, k + 1)];
    }
    v[q] = val;
  }
  __syncthreads();
  const int col = blockIdx.x * kSlice + (t % kSlice), qg = t / kSlice;
  const double* Gk = G + ((size_t)k * g.neo + el) * P * P + col;
  const int q0 = qg * (P / kSlices);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll 2
  for (int q = q0; q < q0 + P / kSlices; q += 4) {
    s0 = fma(Gk[(size_t)q * P], v[q], s0);
    s1 = fma(Gk[(size_t)(q + 1) * P], v[q + 1], s1);
    s2 = fma(Gk[(size_t)(q + 2) * P], v[q + 2], s2);
    s3 = fma(Gk[(size_t)(q + 3) * P], v[q + 3], s3);
  }
  part[qg][t % kSlice] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (t < kSlice) {
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < kSlices; ++w) tot += part[w][t];
    const size_t so = elem_cell(g, cb, e, col % E, col / E, k);
    ybuf[so] = bwd ? ybuf[so] + tot : tot;
  }
}

// out = add + x (x in ybuf) over the owned bricks; with rdot, rdot . out
// finishes the iteration (fin_post) like k_bj_apply
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_add_finish(GridParams g,
                                                             const double* __restrict__ ybuf,
                                                             const double* __restrict__ add,
                                                             double* out,
                                                             const double* __restrict__ rdot,
                                                             PcgState* st, double* partials,
                                                             int init) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  constexpr int C = CB * CB * CB;
  __shared__ double red[80];
  __shared__ int flag;
  const size_t s = (size_t)(blockIdx.x + g.b0) * C + threadIdx.x;
  const double o = add ? add[s] + ybuf[s] : ybuf[s];
  out[s] = o;
  if (!rdot) return;
  double vv[1] = {rdot[s] * o};
  block_sum_k<C, 1>(vv, red);
  double tot[1];
  if (grid_reduce_last_k<1>(vv, partials, &st->ticket[5], tot, &flag, red) && threadIdx.x == 0) {
    if (g.dist) st->loc[kRedPost] = tot[0];
    else fin_post(st, tot[0], init);
  }
}

bool bj_supported(int cb, int sd) {
  const int E = cb * sd;
  return E == 8 || E == 16 || E == kE32;
}

int bj_apply_kernels(int cb, int sd) { return cb * sd == kE32 ? 2 * kE32 : 1; }

int64_t bj_factor_work_doubles(int cb, int sd, int64_t neo) {
  if (cb * sd != kE32) return 0;
  return neo * (dense_inverse_work_doubles(kP32) + 2);
}

int64_t bj_doubles_per_element(int cb, int sd) {
  const int64_t E = cb * sd;
  return E * E * E * E * E;
}

void launch_bj_factor(const GridParams& g, int cb, const double* coef, double* G, int* status,
                      double* work, cudaStream_t s) {
  const int E = cb * g.sd, P = E * E;
  if (E == kE32) {
    const int64_t plane = g.neo * (int64_t)P * P;
    double* ext = work + g.neo * dense_inverse_work_doubles(P);
    for (int k = 0; k < E; ++k) {
      double* Gk = G + k * plane;
      k_bj32_assemble<<<dim3(P / 4, (unsigned)g.neo), 256, 0, s>>>(g, cb, coef,
                                                                  k ? Gk - plane : nullptr, Gk, k);
      dense_spd_inverse_batched(Gk, P, g.neo, work, status, s);
      k_bj32_fold<<<(unsigned)g.neo, 256, 0, s>>>(work, dense_inverse_work_doubles(P),
                                                  dense_inverse_pivots(work, P, 0) - work, ext, k);
    }
    k_bj32_check<<<(unsigned)((g.neo + 255) / 256), 256, 0, s>>>(ext, g.neo, status);
    return;
  }
  const size_t smem = gj_global_smem_bytes(P);
  cudaFuncSetAttribute(k_bj_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_bj_factor<<<(unsigned)g.neo, kGjThreads, smem, s>>>(g, cb, E, coef, G, status);
}

void launch_bj_apply(const GridParams& g, int cb, const double* coef, const double* G,
                     const double* in, const double* add, double* out, const double* rdot,
                     PcgState* st, double* partials, int init, double* ybuf, cudaStream_t s) {
  const int E = cb * g.sd;
  if (E == kE32) {
    const dim3 grid(kSlices, (unsigned)g.neo);
    for (int k = 0; k < E; ++k)
      launch_pdl(k_bj32_step, grid, dim3(1024), 0, s, g, cb, coef, G, in, ybuf,
                 (const PcgState*)st, k, 0);
    for (int k = E - 2; k >= 0; --k)
      launch_pdl(k_bj32_step, grid, dim3(1024), 0, s, g, cb, coef, G, in, ybuf,
                 (const PcgState*)st, k, 1);
    if (cb == 8)
      launch_pdl(k_add_finish<8>, dim3((unsigned)g.nbo), dim3(512), 0, s, g, (const double*)ybuf,
                 add, out, rdot, st, partials, init);
    else
      launch_pdl(k_add_finish<4>, dim3((unsigned)g.nbo), dim3(64), 0, s, g, (const double*)ybuf,
                 add, out, rdot, st, partials, init);
    return;
  }
  if (E == 16)
    launch_pdl(k_bj_apply<16>, dim3((unsigned)g.neo), dim3(256), 0, s, g, cb, coef, G, in, add,
               out, rdot, st, partials, init);
  else
    launch_pdl(k_bj_apply<8>, dim3((unsigned)g.neo), dim3(64), 0, s, g, cb, coef, G, in, add, out,
               rdot, st, partials, init);
}

void launch_add_finish(const GridParams& g, int cb, const double* y, const double* add,
                       double* out, const double* rdot, PcgState* st, double* partials, int init,
                       cudaStream_t s) {
  if (cb == 0) return launch_g_add_finish(g, y, add, out, rdot, st, partials, init, s);
  if (cb == 8)
    launch_pdl(k_add_finish<8>, dim3((unsigned)g.nbo), dim3(512), 0, s, g, y, add, out, rdot, st,
               partials, init);
  else
    launch_pdl(k_add_finish<4>, dim3((unsigned)g.nbo), dim3(64), 0, s, g, y, add, out, rdot, st,
               partials, init);
}

void launch_prolong_add(const GridParams& g, int cb, const double* phi, const double* r1,
                        const double* ec, double* r2, const PcgState* st, cudaStream_t s) {
  if (cb == 0) return launch_g_prolong_add(g, phi, r1, ec, r2, st, s);
  if (cb == 8)
    launch_pdl(k_prolong_add<8>, dim3((unsigned)g.nbo), dim3(512), 0, s, g, phi, r1, ec, r2, st);
  else
    launch_pdl(k_prolong_add<4>, dim3((unsigned)g.nbo), dim3(64), 0, s, g, phi, r1, ec, r2, st);
}

void launch_resid(const GridParams& g, int cb, const double* coef, const double* r,
                  const double* x, double* t, const PcgState* st, cudaStream_t s) {
  if (cb == 0) return launch_g_resid(g, coef, r, x, t, st, s);
  if (cb == 8)
    launch_pdl(k_resid<8>, dim3((unsigned)g.nbo), dim3(512), 0, s, g, coef, r, x, t, st);
  else
    launch_pdl(k_resid<4>, dim3((unsigned)g.nbo), dim3(64), 0, s, g, coef, r, x, t, st);
}

}  // namespace tmg
