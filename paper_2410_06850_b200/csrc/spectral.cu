// Batched local spectral bases, one coarse cell per CTA (north_star item 4).
//
// Reference: local_spectral_basis (proj/core/src/coarse_space.cpp:279-304):
// per coarse cell, the L_c smallest eigenpairs of S_loc phi = lambda M_loc phi
// with S_loc the TPFA stiffness over faces strictly inside the cell
// (box_interior_stiffness, :238-277) and M_loc = diag(kappa * vol), solved via
// B = M^-1/2 S M^-1/2 (generalized_smallest, :203-234) and returned
// M-orthonormal (phi = M^-1/2 v). The reference uses a dense symmetric
// eigensolver (:38-56). Here the problem never leaves shared memory: B is
// applied matrix-free from the cell's face transmissibilities and the lowest
// eigenvectors are found by Chebyshev-filtered subspace iteration with a block
// of K = 2 L_c vectors (Rayleigh-Ritz + CholQR each outer step), stopping when
// every wanted Ritz pair has ||B x - theta x|| <= tol * ||B||. The constant
// mode (B M^{1/2} 1 = 0) seeds the block.
#include "kernels.h"
#include "stencil.cuh"
#include "eig_small.cuh"

namespace tmg {

template <int CB, int K>
struct ChfsiCtx {
  static constexpr int C = CB * CB * CB;
  static constexpr int NW = C / 32;
};

// y = B x for K vectors held in registers; u smem [K][C].
template <int CB, int K>
__device__ __forceinline__ void bmatvec(const double (&x)[K], double (&y)[K], double* u,
                                        const double* tf, double sl, double sll, int nb[6]) {
  constexpr int C = CB * CB * CB;
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < K; ++k) u[k * C + t] = sl * x[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = sll * u[k * C + t];
#pragma unroll
    for (int f = 0; f < 6; ++f)
      if (nb[f] >= 0) s -= tf[f] * u[k * C + nb[f]];
    y[k] = sl * s;
  }
  __syncthreads();
}

// FP64 tensor-core Gram: G = (X^T Y + Y^T X) / 2 for K = 8 vectors over the
// C cells (thread t owns cell t). X and Y are staged in smem as [K][C + 4]
// (the pad puts the 8 vectors' 4-cell runs in distinct bank quarters), each
// warp accumulates its 32 cells with 8 mma.m8n8k4 (A fragment X^T[v][c] =
// B fragment layout), and the 16 (or 2) warp partials are summed in a fixed
// order, symmetrising on the way. Ends with g in smem after a barrier.
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int CB, int K>
__device__ __forceinline__ void gram_mma(const double (&x)[K], const double (&y)[K], bool same,
                                         double* xs, double* ys, double* red, double* g) {
  static_assert(K == 8, "mma.m8n8k4 Gram is built for K = 8");
  constexpr int C = CB * CB * CB, CS = C + 4, NW = C / 32;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    xs[k * CS + t] = x[k];
    if (!same) ys[k * CS + t] = y[k];
  }
  __syncthreads();
  const double* yb = same ? xs : ys;
  double acc[2] = {0.0, 0.0};
  const int off = (lane >> 2) * CS + 32 * w + (lane & 3);
#pragma unroll
  for (int s = 0; s < 8; ++s) dmma_8x8x4(acc, xs[off + 4 * s], yb[off + 4 * s]);
  // acc = rows lane/4, cols 2*(lane%4) + {0, 1} of this warp's X^T Y
  red[w * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = acc[0];
  red[w * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = acc[1];
  __syncthreads();
  if (t < 64) {
    const int i = t >> 3, j = t & 7;
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int v = 0; v < NW; ++v) {
      a += red[v * 64 + i * 8 + j];
      b += red[v * 64 + j * 8 + i];
    }
    g[t] = 0.5 * (a + b);
  }
  __syncthreads();
}

// X <- X R^{-1} where G = R^T R (Cholesky of the Gram matrix, kept in smem).
// Warp 0 factorises (lane j owns column j, right-looking updates through
// shuffles); every thread then applies R^{-1} to its row of X. Returns false
// if G is not numerically positive definite.
template <int K>
__device__ __forceinline__ bool cholqr_apply(double (&x)[K], const double* g, double* rsm,
                                             int* okflag) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double a[K];
#pragma unroll
    for (int i = 0; i < K; ++i) a[i] = lane < K ? g[i * K + lane] : 0.0;
    double gmax = lane < K ? g[lane * K + lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    bool ok = true;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double d = __shfl_sync(0xffffffffu, a[k], k);  // A_kk (column k, row k)
      ok = ok && (d > 1e-28 * gmax);
      const double rkk = ok ? sqrt(d) : 1.0;
      const double rkj = lane >= k && lane < K ? a[k] / rkk : 0.0;  // R_kj
      if (lane < K) rsm[k * K + lane] = lane >= k ? rkj : 0.0;
#pragma unroll
      for (int i = k + 1; i < K; ++i) {
        const double rki = __shfl_sync(0xffffffffu, rkj, i);
        if (lane > k) a[i] -= rki * rkj;
      }
    }
    if (lane == 0) *okflag = ok;
  }
  __syncthreads();
  const bool ok = *okflag;
  if (ok) {
    // row vector x (1 x K) times R^{-1}: solve y R = x, in place
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double s = x[j];
#pragma unroll
      for (int k = 0; k < j; ++k) s -= x[k] * rsm[k * K + j];
      x[j] = s / rsm[j * K + j];
    }
  }
  __syncthreads();
  return ok;
}

// TMG_EIG_MINB CTAs per SM (register cap) and TMG_EIG_GROUP vectors per
// Chebyshev pass (the filter is independent per vector, so smaller groups
// keep fewer vectors live); the Gram staging buffer aliases the mat-vec
// buffer so two CTAs fit one SM's shared memory.
#ifndef TMG_EIG_MINB
#define TMG_EIG_MINB 1
#endif
#ifndef TMG_EIG_GROUP
#define TMG_EIG_GROUP 8
#endif
template <int CB, int K>
__global__ void __launch_bounds__(CB * CB * CB, (CB == 8 ? TMG_EIG_MINB : 1)) k_local_basis(GridParams g,
                                                             const double* __restrict__ kappa,
                                                             const double* __restrict__ phi0,
                                                             double* phi, double* evals,
                                                             int* iters_out, double tol,
                                                             int degree, int max_outer,
                                                             const int64_t* __restrict__ list) {
  constexpr int C = CB * CB * CB;
  constexpr int NW = C / 32;
  constexpr int NP = K * (K + 1) / 2;
  extern __shared__ double sm[];
  double* u = sm;                     // K*(C+4): mat-vec exchange, aliased by the Gram staging xs
  double* kt = u + K * (C + 4);       // C
  double* red = kt + C;               // max(NP*NW + NP + 8, 64*NW)
  double* gs = red + (NP * NW + NP + 8 > 64 * NW ? NP * NW + NP + 8 : 64 * NW);  // K*K
  double* qv = gs + K * K;            // K*K
  double* rsm = qv + K * K;           // K*K
  double* scal = rsm + K * K;         // K + 8 scalars
  double* xs = u;                     // K*(C+4) Gram staging (u is idle during Gram)
  double* ys = scal + K + 8;          // K*(C+4)
  __shared__ int okflag;
  const int t = threadIdx.x, li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
  const int64_t b = list ? list[blockIdx.x] : blockIdx.x + g.b0;
  kt[t] = kappa[b * C + t];
  __syncthreads();
  // interior-face transmissibilities (coarse_space.cpp:264-274)
  const double cp[3] = {g.cpl[0], g.cpl[1], g.cpl[2]};
  int nb[6];
  double tf[6];
  double sll = 0.0;
  {
    const int co[3] = {li, lj, lk};
    const int st[3] = {1, CB, CB * CB};
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int ax = f >> 1;
      const bool hi = f & 1;
      const bool exists = hi ? co[ax] + 1 < CB : co[ax] > 0;
      nb[f] = exists ? (hi ? t + st[ax] : t - st[ax]) : -1;
      tf[f] = exists ? face_t(kt[t], kt[nb[f]]) * cp[ax] : 0.0;
      sll += tf[f];
    }
  }
  const double mass = kt[t] * g.vol;
  const double sl = 1.0 / sqrt(mass);
  // Gershgorin bound of B
  double gr = sl * sll * sl;
#pragma unroll
  for (int f = 0; f < 6; ++f)
    if (nb[f] >= 0) gr += sl * tf[f] / sqrt(kt[nb[f]] * g.vol);
  for (int o = 16; o > 0; o >>= 1) gr = fmax(gr, __shfl_xor_sync(0xffffffffu, gr, o));
  if ((t & 31) == 0) red[t >> 5] = gr;
  __syncthreads();
  if (t == 0) {
    double m = 0.0;
    for (int w = 0; w < NW; ++w) m = fmax(m, red[w]);
    scal[0] = m;
  }
  __syncthreads();
  const double bmax = scal[0];
  __syncthreads();
  // initial block: constant mode in B-space (sqrt(mass)) + pseudo-random, or
  // (warm start) the previous set-up's M-orthonormal bases mapped to the
  // B metric, x = M^{1/2} phi, completed by pseudo-random vectors
  // A warm start that has not converged after kWarmOuter rounds restarts once
  // from the cold block (a stagnating seed costs at most kWarmOuter rounds).
  constexpr int kWarmOuter = 20;
  double x[K], y[K];
  double theta[K];
  double a_cut = 0.0;
  int outer = 0, outer_total = 0;
  bool converged = false;
  for (int attempt = 0; attempt < (phi0 ? 2 : 1) && !converged; ++attempt) {
  const bool warm = phi0 && attempt == 0;
  x[0] = sqrt(mass);
#pragma unroll
  for (int k = 1; k < K; ++k) x[k] = hash_uniform(b, t, k);
  if (warm) {
    const double sm_ = sqrt(mass);
    for (int k = 0; k < g.lc && k < K; ++k) x[k] = sm_ * phi0[(b * g.lc + k) * C + t];
  }
  a_cut = 0.5 * bmax;
  const int outer_cap = warm && kWarmOuter < max_outer ? kWarmOuter : max_outer;
  for (outer = 0; outer <= outer_cap; ++outer) {
    // --- orthonormalise (CholQR twice) ---
    for (int pass = 0; pass < 2; ++pass) {
      gram_mma<CB, K>(x, x, true, xs, ys, red, gs);
      if (!cholqr_apply<K>(x, gs, rsm, &okflag)) {
        // rank loss: re-seed the trailing vectors and retry next pass
#pragma unroll
        for (int k = 1; k < K; ++k) x[k] += 1e-3 * hash_uniform(b + 7777, t, k + 31 * outer);
      }
    }
    // --- Rayleigh-Ritz ---
    bmatvec<CB, K>(x, y, u, tf, sl, sll, nb);
    gram_mma<CB, K>(x, y, false, xs, ys, red, gs);
    if (t < 32) {
      warp_jacobi_small<K>(gs, rsm);  // gs -> eigenvalues on its diagonal, rsm = vectors
      if (t == 0) {
        int ord[K];  // ascending
        for (int i = 0; i < K; ++i) ord[i] = i;
        for (int i = 0; i < K; ++i)
          for (int j = i + 1; j < K; ++j)
            if (gs[ord[j] * K + ord[j]] < gs[ord[i] * K + ord[i]]) {
              const int tmp = ord[i]; ord[i] = ord[j]; ord[j] = tmp;
            }
        for (int c = 0; c < K; ++c) {
          scal[c] = gs[ord[c] * K + ord[c]];
          for (int r = 0; r < K; ++r) qv[r * K + c] = rsm[r * K + ord[c]];
        }
      }
    }
    __syncthreads();
    double xn[K], yn[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      theta[c] = scal[c];
      double s = 0.0, s2 = 0.0;
#pragma unroll
      for (int r = 0; r < K; ++r) {
        s += x[r] * qv[r * K + c];
        s2 += y[r] * qv[r * K + c];
      }
      xn[c] = s;
      yn[c] = s2;
    }
    __syncthreads();
    // residual norms of the wanted pairs
    double rv[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      rv[c] = yn[c] - theta[c] * xn[c];
      x[c] = xn[c];
    }
    gram_mma<CB, K>(rv, rv, true, xs, ys, red, rsm);  // diagonal = squared residual norms
    double worst = 0.0;
    for (int c = 0; c < g.lc; ++c) worst = fmax(worst, sqrt(fmax(rsm[c * K + c], 0.0)));
    if (worst <= tol * bmax) { converged = true; break; }
    if (outer == outer_cap) break;
    // --- Chebyshev filter damping [a_cut, bmax], normalised at 0 ---
    a_cut = fmin(fmax(theta[K - 1], 1e-6 * bmax), 0.95 * bmax);
    const double e = 0.5 * (bmax - a_cut), c0 = 0.5 * (bmax + a_cut);
    const double sigma1 = e / (0.0 - c0);
    const double gam = 2.0 / sigma1;
    constexpr int KG = TMG_EIG_GROUP < K ? TMG_EIG_GROUP : K;
#pragma unroll
    for (int g0 = 0; g0 < K; g0 += KG) {  // vector groups, each filtered on its own
      double xg[KG], yg[KG], x0[KG];
#pragma unroll
      for (int k = 0; k < KG; ++k) xg[k] = x[g0 + k];
      double sigma = sigma1;
      bmatvec<CB, KG>(xg, yg, u, tf, sl, sll, nb);
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        x0[k] = xg[k];
        yg[k] = (yg[k] - c0 * xg[k]) * (sigma1 / e);
      }
      for (int d = 2; d <= degree; ++d) {
        const double sig2 = 1.0 / (gam - sigma);
        double by[KG];
        bmatvec<CB, KG>(yg, by, u, tf, sl, sll, nb);
#pragma unroll
        for (int k = 0; k < KG; ++k) {
          const double ynew = (by[k] - c0 * yg[k]) * (2.0 * sig2 / e) - (sigma * sig2) * x0[k];
          x0[k] = yg[k];
          yg[k] = ynew;
        }
        sigma = sig2;
      }
#pragma unroll
      for (int k = 0; k < KG; ++k) x[g0 + k] = yg[k];
    }
  }
  outer_total += outer;
  }  // attempt
  // sign convention: sum of each vector >= 0
  double sg[K];
#pragma unroll
  for (int k = 0; k < K; ++k) sg[k] = x[k] * sl;
  block_sum_k<C, K>(sg, red);
  for (int a = 0; a < g.lc; ++a) {
    const double sgn = sg[a] < 0.0 ? -1.0 : 1.0;
    phi[(b * g.lc + a) * C + t] = sgn * sl * x[a];
  }
  if (t == 0) {
    for (int a = 0; a < g.lc; ++a) evals[b * g.lc + a] = theta[a];
    iters_out[b] = converged ? outer_total : -outer_total - 1;
  }
}

size_t local_basis_smem(int cb, int K) {
  const int C = cb * cb * cb, NW = C / 32, NP = K * (K + 1) / 2;
  const int red = NP * NW + NP + 8 > 64 * NW ? NP * NW + NP + 8 : 64 * NW;
  return sizeof(double) * (size_t)(K * (C + 4) + C + red + 3 * K * K + K + 8 + K * (C + 4));
}

void launch_local_basis(const GridParams& g, int cb, const double* kappa, const double* phi0,
                        double* phi, double* evals, int* iters, double tol, int degree,
                        int max_outer, const int64_t* list, int64_t nlist, cudaStream_t s) {
  const size_t smem = local_basis_smem(cb, 8);
  const unsigned grid = (unsigned)(list ? nlist : g.nbo);
  if (grid == 0) return;
  if (cb == 8) {
    ensure_dyn_smem(k_local_basis<8, 8>, smem);
    k_local_basis<8, 8><<<grid, 512, smem, s>>>(g, kappa, phi0, phi, evals, iters, tol, degree,
                                                max_outer, list);
  } else {
    ensure_dyn_smem(k_local_basis<4, 8>, smem);
    k_local_basis<4, 8><<<grid, 64, smem, s>>>(g, kappa, phi0, phi, evals, iters, tol, degree,
                                               max_outer, list);
  }
}

// flag[i] = 1: every cell of brick b0 + i has bitwise the same conductivity.
template <int CB>
__global__ void __launch_bounds__(256) k_uniform_inside(GridParams g, const double* __restrict__ kappa,
                                                       int* flag) {
  constexpr int C = CB * CB * CB;
  const int64_t b = g.b0 + blockIdx.x;
  __shared__ int same;
  if (threadIdx.x == 0) same = 1;
  __syncthreads();
  const double k0 = kappa[b * C];
  bool ok = true;
  for (int t = threadIdx.x; t < C; t += blockDim.x) ok = ok && kappa[b * C + t] == k0;
  if (!ok) same = 0;  // every writer stores 0
  __syncthreads();
  if (threadIdx.x == 0) flag[blockIdx.x] = same;
}

// Local bases of the flagged bricks in closed form. With one conductivity k
// inside, the local problem (box_interior_stiffness + mass,
// coarse_space.cpp:238-304) is t S_hat, t = face_t(k, k), and k vol I, where
// S_hat = sum over axes of area/h times the 1-D Neumann Laplacian (unit
// coupling). Its eigenvectors are the separable DCT-II products
//   v_pqr(i, j, l) = cos(pi p (i + 1/2) / CB) cos(pi q (j + 1/2) / CB) cos(pi r (l + 1/2) / CB)
// with B-eigenvalues t / (k vol) sum_ax (area/h)_ax (2 - 2 cos(pi p_ax / CB)).
// The L_c smallest (ties by mode index p + CB (q + CB r): a fixed choice
// inside a degenerate cluster cut by L_c, as any eigensolver makes one) are
// written M-orthonormal, phi = v / ||v|| / sqrt(k vol). Exact, and the same
// bits in every partition of the grid.
template <int CB>
__global__ void __launch_bounds__(256) k_local_basis_uniform(GridParams g,
                                                            const double* __restrict__ kappa,
                                                            const int* __restrict__ flag,
                                                            double* phi, double* evals, int* iters) {
  constexpr int C = CB * CB * CB;
  constexpr int LMAX = 8;
  const int64_t b = g.b0 + blockIdx.x;
  if (!flag[blockIdx.x]) return;
  const int lc = g.lc;
  __shared__ int mode[LMAX];
  __shared__ double mu[LMAX];
  if (threadIdx.x == 0) {
    int n = 0;
    for (int m = 0; m < C; ++m) {
      const int pm[3] = {m % CB, (m / CB) % CB, m / (CB * CB)};
      double v = 0.0;
      for (int ax = 0; ax < 3; ++ax) v += g.cpl[ax] * (2.0 - 2.0 * cospi((double)pm[ax] / CB));
      // insertion into the sorted (mu, mode) list of the lc smallest
      int pos = n < lc ? n : lc;
      while (pos > 0 && v < mu[pos - 1]) --pos;
      if (pos >= lc) continue;
      for (int k = (n < lc ? n : lc - 1); k > pos; --k) {
        mu[k] = mu[k - 1];
        mode[k] = mode[k - 1];
      }
      mu[pos] = v;
      mode[pos] = m;
      if (n < lc) ++n;
    }
  }
  __syncthreads();
  const double kb = kappa[b * C];
  const double sc = 1.0 / sqrt(kb * g.vol);
  for (int e = threadIdx.x; e < lc * C; e += blockDim.x) {
    const int a = e / C, l = e % C;
    const int m = mode[a];
    const int pm[3] = {m % CB, (m / CB) % CB, m / (CB * CB)};
    const int co[3] = {l % CB, (l / CB) % CB, l / (CB * CB)};
    double v = 1.0, nrm2 = 1.0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      v *= cospi((double)pm[ax] * (co[ax] + 0.5) / CB);
      nrm2 *= pm[ax] == 0 ? (double)CB : 0.5 * CB;
    }
    phi[(b * lc + a) * C + l] = sc * v / sqrt(nrm2);
  }
  if ((int)threadIdx.x < lc) evals[b * lc + threadIdx.x] = face_t(kb, kb) / (kb * g.vol) * mu[threadIdx.x];
  if (threadIdx.x == 0) iters[b] = 0;
}

void launch_uniform_inside(const GridParams& g, int cb, const double* kappa, int* flag,
                           cudaStream_t s) {
  if (cb == 8) k_uniform_inside<8><<<(unsigned)g.nbo, 256, 0, s>>>(g, kappa, flag);
  else k_uniform_inside<4><<<(unsigned)g.nbo, 64, 0, s>>>(g, kappa, flag);
}

void launch_local_basis_uniform(const GridParams& g, int cb, const double* kappa, const int* flag,
                                double* phi, double* evals, int* iters, cudaStream_t s) {
  if (cb == 8)
    k_local_basis_uniform<8><<<(unsigned)g.nbo, 256, 0, s>>>(g, kappa, flag, phi, evals, iters);
  else
    k_local_basis_uniform<4><<<(unsigned)g.nbo, 64, 0, s>>>(g, kappa, flag, phi, evals, iters);
}

}  // namespace tmg
