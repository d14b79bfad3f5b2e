// Coarse level for large cc elements (q = sd^3 L_c > 64, e.g. sd = 4: q = 256;
// the 512^3 / 1024^3 hierarchies of SURVEY.md §8). The element matrices no
// longer fit in shared memory, so they live in global memory (L2-resident per
// CTA) and are inverted by a batched blocked Gauss-Jordan with 64 x 64 pivot
// blocks (register-resident pivot inversion, gj.cuh); the cc eigenproblem is
// solved by subspace iteration on a shifted inverse with Rayleigh-Ritz on the
// projected stiffness (coarse_coarse_basis, coarse_space.cpp:343-406).
#include "coarse_elem.cuh"
#include "gj_global.cuh"

namespace tmg {

namespace {
constexpr int GB = kGjBlock;
constexpr int GJT = kGjThreads;

__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double m = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
  return m;
}
}  // namespace

// Element matrix of A_c restricted to the cc element (couplings between its
// children only), optionally minus the boundary terms Bc (the projected
// stiffness of the cc eigenproblem) plus shift_rel * max_i M_ii * I;
// symmetrised. One CTA per element, out[e - e0][q][q].
__global__ void k_elem_matrix(GridParams g, const double* __restrict__ Ac,
                              const double* __restrict__ Bc, double shift_rel, double* out) {
  __shared__ double red[32];
  const int q = g.sd * g.sd * g.sd * g.lc, nch = g.sd * g.sd * g.sd;
  const ElemCoord ec = elem_coord(g, blockIdx.x + g.e0);
  double* M = out + (int64_t)blockIdx.x * q * q;
  for (int e = threadIdx.x; e < q * q; e += blockDim.x) M[e] = 0.0;
  __syncthreads();
  for (int e = threadIdx.x; e < nch * 7 * g.lc * g.lc; e += blockDim.x) {
    const int ci = e / (7 * g.lc * g.lc), rem = e % (7 * g.lc * g.lc);
    const int dir = rem / (g.lc * g.lc), ab = rem % (g.lc * g.lc), a = ab / g.lc, b = ab % g.lc;
    const int64_t I = child_brick(g, ec, ci);
    int cj;
    if (dir == 0) cj = ci;
    else {
      const int64_t J = brick_nbr(g, I, dir - 1);
      cj = J >= 0 ? child_index(g, ec, J) : -1;
    }
    if (cj < 0) continue;
    double v = Ac[(I * 7 + dir) * g.lc * g.lc + ab];
    if (dir == 0 && Bc) v -= Bc[I * g.lc * g.lc + ab];
    M[(ci * g.lc + a) * q + cj * g.lc + b] += v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < q * q; e += blockDim.x) {
    const int i = e / q, j = e % q;
    if (i < j) {
      const double s = 0.5 * (M[i * q + j] + M[j * q + i]);
      M[i * q + j] = s;
      M[j * q + i] = s;
    }
  }
  if (shift_rel == 0.0) return;
  double mx = 0.0;
  for (int i = threadIdx.x; i < q; i += blockDim.x) mx = fmax(mx, M[i * q + i]);
  mx = block_max(mx, red);
  for (int i = threadIdx.x; i < q; i += blockDim.x) M[i * q + i] += shift_rel * mx;
}

// In-place inverse of each SPD q x q matrix (gj_global.cuh), one CTA per
// matrix; the reference singular-pivot rule (solver.cpp:86-92) over each
// matrix's pivots, status = 2 on failure.
__global__ void __launch_bounds__(GJT, 1) k_batched_gj(double* A, int q, int* status) {
  extern __shared__ __align__(16) double smg[];
  __shared__ GjSmem<GB> gjs;
  __shared__ double red[2][GJT / 32];
  const int t = threadIdx.x, lane = t & 31;
  double pmin = 1e300, pmax = 0.0;
  gj_inverse_global(A + (int64_t)blockIdx.x * q * q, q, gj_global_smem(smg, q), gjs, pmin, pmax);
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
    for (int w = 0; w < GJT / 32; ++w) {
      m = fmax(m, red[0][w]);
      n = fmin(n, red[1][w]);
    }
    if (!(n > 1e-14 * m)) atomicExch(status, 2);
  }
}

// ---------------------------------------------- cc eigensolver for large q
//
// Lowest L_cc eigenpairs of the projected stiffness H = P S_E P^T of each cc
// element (coarse_coarse_basis, coarse_space.cpp:343-406) by subspace
// iteration on the shifted inverse Hs = (H + sigma I)^-1 (k_elem_matrix +
// k_batched_gj): KS columns, two SVQB orthonormalisation passes per step and
// Rayleigh-Ritz on H, applied sparsely from Ac / Bc. Stops when every wanted
// Ritz pair has ||H x - theta x|| <= tol * max_i H_ii. Output as k_cc_basis:
// ascending eigenvalues, each vector signed so that its entries sum to >= 0.
// sigma = 1e-5 max_i H_ii: H is singular (Neumann), and a smaller shift makes
// the rounding of Hs X the residual floor (1e-10 at sigma = 1e-10); measured
// on the oracle's projected matrices at contrast 1e3..1e6, 1e-5 reaches
// 1e-13 in <= 24 steps (tests/cc_subspace_sim.py).
namespace {
__device__ __forceinline__ double hash_unit(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return (double)x * (1.0 / 4294967296.0) - 0.5;
}

// sum over the block of one value per thread (every thread gets the total)
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  __syncthreads();
  return s;
}

// Block-wide cyclic Jacobi on the K x K symmetric M (smem): round-robin
// ordering, K/2 disjoint rotations per round, the (row, pair) updates spread
// over the block; V (K x K) collects the eigenvectors in its columns.
template <int K>
__device__ void block_jacobi(double* M, double* V, double* red) {
  constexpr int NP = K / 2;
  __shared__ double rc[NP], rs[NP];
  __shared__ int rp[NP], rq[NP];
  const int t = threadIdx.x, nt = blockDim.x;
  for (int e = t; e < K * K; e += nt) V[e] = (e / K == e % K) ? 1.0 : 0.0;
  __syncthreads();
  for (int sweep = 0; sweep < 30; ++sweep) {
    double tot = 0.0, off = 0.0;
    for (int e = t; e < K * K; e += nt) {
      const double v = M[e] * M[e];
      tot += v;
      if (e / K != e % K) off += v;
    }
    tot = block_sum(tot, red);
    off = block_sum(off, red);
    if (off <= 1e-26 * tot || off == 0.0) break;
    for (int round = 0; round < K - 1; ++round) {
      if (t < NP) {  // circle method, player K-1 fixed
        int p = t == 0 ? round : (round + t) % (K - 1);
        int qq = t == 0 ? K - 1 : (round - t + (K - 1)) % (K - 1);
        if (p > qq) {
          const int tmp = p;
          p = qq;
          qq = tmp;
        }
        const double apq = M[p * K + qq], app = M[p * K + p], aqq = M[qq * K + qq];
        double c = 1.0, sn = 0.0;
        if (!(fabs(apq) <= 1e-300 || fabs(apq) <= 1e-18 * sqrt(fabs(app * aqq)))) {
          const double theta = (aqq - app) / (2.0 * apq);
          const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(tt * tt + 1.0);
          sn = tt * c;
        }
        rc[t] = c;
        rs[t] = sn;
        rp[t] = p;
        rq[t] = qq;
      }
      __syncthreads();
      for (int e = t; e < K * NP; e += nt) {  // columns p, q of row r
        const int r = e / NP, gq = e % NP, p = rp[gq], qq = rq[gq];
        const double c = rc[gq], sn = rs[gq];
        const double akp = M[r * K + p], akq = M[r * K + qq];
        M[r * K + p] = c * akp - sn * akq;
        M[r * K + qq] = sn * akp + c * akq;
        const double vkp = V[r * K + p], vkq = V[r * K + qq];
        V[r * K + p] = c * vkp - sn * vkq;
        V[r * K + qq] = sn * vkp + c * vkq;
      }
      __syncthreads();
      for (int e = t; e < K * NP; e += nt) {  // rows p, q at column col
        const int gq = e / K, col = e % K, p = rp[gq], qq = rq[gq];
        const double c = rc[gq], sn = rs[gq];
        const double apk = M[p * K + col], aqk = M[qq * K + col];
        M[p * K + col] = c * apk - sn * aqk;
        M[qq * K + col] = sn * apk + c * aqk;
      }
      __syncthreads();
    }
  }
}

// Gram entries T[i][j] = sum_r A[r][i] B[r][j] (q x KS row-major A, B),
// (i, j) pairs spread over the block; sym: 0.5 (A^T B + B^T A)
template <int KS>
__device__ void gram(const double* A, const double* B, int q, double* T, bool sym) {
  for (int e = threadIdx.x; e < KS * KS; e += blockDim.x) {
    const int i = e / KS, j = e % KS;
    double s = 0.0, s2 = 0.0;
    for (int r = 0; r < q; ++r) {
      s = fma(A[r * KS + i], B[r * KS + j], s);
      if (sym) s2 = fma(A[r * KS + j], B[r * KS + i], s2);
    }
    T[e] = sym ? 0.5 * (s + s2) : s;
  }
  __syncthreads();
}

// X = orthonormal basis of span(Y) (q x KS, row-major): scaled Gram matrix,
// its eigendecomposition, X = Y D W Lambda^-1/2.
template <int KS>
__device__ void svqb_pass(const double* Y, double* X, int q, double* T, double* V, double* F,
                          double* dsc, double* red) {
  const int t = threadIdx.x;
  gram<KS>(Y, Y, q, T, false);
  for (int k = t; k < KS; k += blockDim.x) dsc[k] = rsqrt(fmax(T[k * KS + k], 1e-300));
  __syncthreads();
  for (int e = t; e < KS * KS; e += blockDim.x) T[e] *= dsc[e / KS] * dsc[e % KS];
  __syncthreads();
  block_jacobi<KS>(T, V, red);
  for (int e = t; e < KS * KS; e += blockDim.x) {
    const int i = e / KS, j = e % KS;
    F[e] = dsc[i] * V[i * KS + j] * rsqrt(fmax(T[j * KS + j], 1e-24));
  }
  __syncthreads();
  for (int r = t; r < q; r += blockDim.x) {
    double y[KS];
#pragma unroll
    for (int i = 0; i < KS; ++i) y[i] = Y[r * KS + i];
#pragma unroll
    for (int j = 0; j < KS; ++j) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < KS; ++i) s = fma(y[i], F[i * KS + j], s);
      X[r * KS + j] = s;
    }
  }
  __syncthreads();
}

// X = Y R^-1 with Y^T Y = R^T R (CholQR; Y == X allowed): one warp factors
// the KS x KS Gram matrix with shuffles, every thread back-substitutes its
// rows. Returns false (X untouched) when the Gram matrix is not numerically
// positive definite, for the caller's SVQB fallback.
template <int KS>
__device__ bool cholqr_pass(const double* Y, double* X, int q, double* T, double* R,
                            int* okflag) {
  const int t = threadIdx.x;
  gram<KS>(Y, Y, q, T, false);
  if (t < 32) {
    const int lane = t;
    double a[KS];
#pragma unroll
    for (int i = 0; i < KS; ++i) a[i] = lane < KS ? T[i * KS + lane] : 0.0;
    double gmax = lane < KS ? T[lane * KS + lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    bool ok = true;
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const double d = __shfl_sync(0xffffffffu, a[k], k);
      ok = ok && (d > 1e-24 * gmax);
      const double rkk = ok ? sqrt(d) : 1.0;
      const double rkj = lane >= k && lane < KS ? a[k] / rkk : 0.0;
      if (lane < KS) R[k * KS + lane] = lane >= k ? rkj : 0.0;
#pragma unroll
      for (int i = k + 1; i < KS; ++i) {
        const double rki = __shfl_sync(0xffffffffu, rkj, i);
        if (lane > k) a[i] -= rki * rkj;
      }
    }
    if (lane == 0) *okflag = ok;
  }
  __syncthreads();
  if (!*okflag) return false;
  for (int r = t; r < q; r += blockDim.x) {
    double x[KS];
#pragma unroll
    for (int i = 0; i < KS; ++i) x[i] = Y[r * KS + i];
#pragma unroll
    for (int j = 0; j < KS; ++j) {
      double v = x[j];
#pragma unroll
      for (int k = 0; k < j; ++k) v = fma(-x[k], R[k * KS + j], v);
      x[j] = v / R[j * KS + j];
    }
#pragma unroll
    for (int i = 0; i < KS; ++i) X[r * KS + i] = x[i];
  }
  __syncthreads();
  return true;
}

// Z = H X with H = (A_c - Bc on the diagonal blocks) restricted to E's children.
template <int KS>
__device__ void apply_projected(const GridParams& g, const ElemCoord& ec, const double* Ac,
                                const double* Bc, const double* X, double* Z, int q) {
  for (int r = threadIdx.x; r < q; r += blockDim.x) {
    const int ci = r / g.lc, a = r % g.lc;
    const int64_t I = child_brick(g, ec, ci);
    double z[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) z[k] = 0.0;
    for (int dir = 0; dir < 7; ++dir) {
      int cj = ci;
      if (dir > 0) {
        const int64_t J = brick_nbr(g, I, dir - 1);
        cj = J >= 0 ? child_index(g, ec, J) : -1;
      }
      if (cj < 0) continue;
#pragma unroll
      for (int b = 0; b < g.lc; ++b) {
        double h = Ac[(I * 7 + dir) * g.lc * g.lc + a * g.lc + b];
        if (dir == 0) h -= Bc[I * g.lc * g.lc + a * g.lc + b];
        const double* xr = X + (cj * g.lc + b) * KS;
#pragma unroll
        for (int k = 0; k < KS; ++k) z[k] = fma(h, xr[k], z[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < KS; ++k) Z[r * KS + k] = z[k];
  }
}
}  // namespace

constexpr int kRREvery = 4;

// One CTA (256 threads) per element. X, Y, Z (q x KS each) in shared memory,
// or in gscr (3 q KS doubles per element) when they do not fit (q > 256).
template <int KS>
__global__ void __launch_bounds__(256) k_cc_subspace(GridParams g, const double* __restrict__ Ac,
                                                     const double* __restrict__ Bc,
                                                     const double* __restrict__ Hs, double tol,
                                                     int maxit, double* Rcc, double* cc_evals,
                                                     int* iters, double* gscr) {
  extern __shared__ __align__(16) double sms[];
  const int q = g.sd * g.sd * g.sd * g.lc, t = threadIdx.x, nt = blockDim.x;
  double* T = sms;
  double* V = T + KS * KS;
  double* F = V + KS * KS;
  double* dsc = F + KS * KS;
  double* th = dsc + KS;
  double* res = th + KS;
  double* vec = gscr ? gscr + (size_t)blockIdx.x * 3 * q * KS : res + KS;
  double* X = vec;
  double* Y = X + q * KS;
  double* Z = Y + q * KS;
  __shared__ int perm[KS];
  __shared__ int flag;
  __shared__ double red[32];
  const ElemCoord ec = elem_coord(g, blockIdx.x + g.e0);
  const double* H = Hs + (int64_t)blockIdx.x * q * q;
  double hd = 0.0;
  for (int r = t; r < q; r += nt) {
    const int64_t I = child_brick(g, ec, r / g.lc);
    const int a = r % g.lc;
    hd = fmax(hd, Ac[I * 7 * g.lc * g.lc + a * (g.lc + 1)] - Bc[I * g.lc * g.lc + a * (g.lc + 1)]);
  }
  const double thr = tol * block_max(hd, red);
  // start: the constant vector and hashed columns
  for (int e = t; e < q * KS; e += nt) {
    const int r = e / KS, k = e % KS;
    Y[e] = k == 0 ? 1.0 : hash_unit((uint32_t)(r * KS + k + 1));
  }
  __syncthreads();
  int it = 0;
  for (;; ++it) {
    // orthonormalise Y -> X: CholQR twice (one warp, no block-wide Jacobi
    // sweeps); SVQB for a pass whose Gram matrix is not numerically PD
    if (!cholqr_pass<KS>(Y, X, q, T, F, &flag)) svqb_pass<KS>(Y, X, q, T, V, F, dsc, red);
    if (!cholqr_pass<KS>(X, X, q, T, F, &flag)) svqb_pass<KS>(X, X, q, T, V, F, dsc, red);
    // Rayleigh-Ritz on H and the convergence test every kRREvery steps (the
    // iteration itself only needs the orthonormalised block; the Ritz pairs
    // are read out at the end)
    if ((it % kRREvery == kRREvery - 1) || it + 1 >= maxit) {
      apply_projected<KS>(g, ec, Ac, Bc, X, Z, q);
      __syncthreads();
      gram<KS>(X, Z, q, T, true);
      block_jacobi<KS>(T, V, red);
      if (t == 0) {  // ascending, ties by index
        unsigned used = 0;
        for (int k = 0; k < KS; ++k) {
          int best = -1;
          for (int i = 0; i < KS; ++i)
            if (!(used >> i & 1u) && (best < 0 || T[i * (KS + 1)] < T[best * (KS + 1)])) best = i;
          used |= 1u << best;
          perm[k] = best;
          th[k] = T[best * (KS + 1)];
        }
      }
      __syncthreads();
      for (int r = t; r < q; r += nt) {
        double xr[KS], zr[KS];
  #pragma unroll
        for (int i = 0; i < KS; ++i) {
          xr[i] = X[r * KS + i];
          zr[i] = Z[r * KS + i];
        }
  #pragma unroll
        for (int k = 0; k < KS; ++k) {
          const int pk = perm[k];
          double xs = 0.0, zs = 0.0;
  #pragma unroll
          for (int i = 0; i < KS; ++i) {
            xs = fma(xr[i], V[i * KS + pk], xs);
            zs = fma(zr[i], V[i * KS + pk], zs);
          }
          X[r * KS + k] = xs;
          Z[r * KS + k] = zs;
        }
      }
      __syncthreads();
      // residual norms of the wanted pairs: 16 lanes per column
      for (int k0 = 0; k0 < KS; k0 += nt >> 4) {
        const int k = k0 + (t >> 4), part = t & 15;
        double s = 0.0;
        if (k < KS)
          for (int r = part; r < q; r += 16) {
            const double d = Z[r * KS + k] - th[k] * X[r * KS + k];
            s = fma(d, d, s);
          }
        for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (k < KS && part == 0) res[k] = sqrt(s);
      }
      __syncthreads();
      if (t == 0) {
        int ok = 1;
        for (int k = 0; k < g.lcc; ++k) ok &= res[k] <= thr;
        flag = ok;
      }
      __syncthreads();
      if (flag || it + 1 >= maxit) break;
    }
    // Y = Hs X (Hs symmetric: column r read coalesced)
    for (int r = t; r < q; r += nt) {
      double acc[KS];
#pragma unroll
      for (int k = 0; k < KS; ++k) acc[k] = 0.0;
      for (int c = 0; c < q; ++c) {
        const double h = H[(int64_t)c * q + r];
        const double2* xc = reinterpret_cast<const double2*>(X + c * KS);
#pragma unroll
        for (int k = 0; k < KS / 2; ++k) {
          const double2 xv = xc[k];
          acc[2 * k] = fma(h, xv.x, acc[2 * k]);
          acc[2 * k + 1] = fma(h, xv.y, acc[2 * k + 1]);
        }
      }
#pragma unroll
      for (int k = 0; k < KS; ++k) Y[r * KS + k] = acc[k];
    }
    __syncthreads();
  }
  for (int k = t; k < g.lcc; k += nt) {
    double s = 0.0;
    for (int r = 0; r < q; ++r) s += X[r * KS + k];
    dsc[k] = s < 0.0 ? -1.0 : 1.0;
    cc_evals[ec.e * g.lcc + k] = th[k];
  }
  __syncthreads();
  for (int e = t; e < g.lcc * q; e += nt) {
    const int k = e / q, r = e % q;
    Rcc[(ec.e * g.lcc + k) * q + r] = dsc[k] * X[r * KS + k];
  }
  if (t == 0 && iters) atomicMax(iters, it + 1);
}

// q <= 256: one CTA per element (k_batched_gj); larger q (sd = 8: 2048) with
// the tensor-core blocked Gauss-Jordan batched over the elements (dense.cu).
// L_cc <= 12: 16 subspace columns, <= 20: 24.
bool coarse_large_supported(int q, int lcc) { return q > 64 && q <= 4096 && lcc <= 20; }

// element inverses: one CTA per element (register/shared Gauss-Jordan,
// gj_global.cuh) for q = 128, 192, 256; the tensor-core blocked Gauss-Jordan
// batched over the elements (dense.cu) for every other q
static bool gj_per_cta(int q) { return q % GB == 0 && q <= GJT; }

// TMG_CC_KS=16/24 overrides (diagnostics)
static int subspace_width(int lcc) {
  const char* e = getenv("TMG_CC_KS");
  if (e && atoi(e) == 24) return 24;
  if (e && atoi(e) == 16 && lcc <= 12) return 16;
  return lcc <= 12 ? 16 : 24;
}

static bool subspace_in_smem(int q, int ks) { return q <= 256 && 3 * q * ks * 8 <= 160 * 1024; }

// scratch doubles the large-q set-up needs besides Winv's storage
int64_t coarse_large_work_doubles(int q, int64_t neo, int lcc) {
  if (gj_per_cta(q) && subspace_in_smem(q, subspace_width(lcc))) return 0;
  const int64_t inv = gj_per_cta(q) ? 0 : neo * dense_inverse_work_doubles(q);
  const int64_t sub = neo * 3 * (int64_t)q * subspace_width(lcc);
  return inv > sub ? inv : sub;
}

size_t batched_gj_smem(int q) { return gj_global_smem_bytes(q); }

static void invert_elements(double* A, int q, int64_t neo, double* work, int* status,
                            cudaStream_t s) {
  if (gj_per_cta(q)) {
    const size_t smem = batched_gj_smem(q);
    cudaFuncSetAttribute(k_batched_gj, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_batched_gj<<<(unsigned)neo, GJT, smem, s>>>(A, q, status);
  } else {
    dense_spd_inverse_batched(A, q, neo, work, status, s);
  }
}

// Winv of every owned cc element (coarse_blocks_by_cc smoother) for large q.
void launch_coarse_smoother_large(const GridParams& g, const double* Ac, double* Winv,
                                  double* work, int* status, cudaStream_t s) {
  const int q = g.sd * g.sd * g.sd * g.lc;
  k_elem_matrix<<<(unsigned)g.neo, 256, 0, s>>>(g, Ac, nullptr, 0.0, Winv + g.e0 * q * q);
  invert_elements(Winv + g.e0 * q * q, q, g.neo, work, status, s);
}

template <int KS>
static void launch_subspace(const GridParams& g, const double* Ac, const double* Bc,
                            const double* Hs, double tol, int maxit, double* Rcc, double* cc_evals,
                            int* iters, double* work, cudaStream_t s) {
  const int q = g.sd * g.sd * g.sd * g.lc;
  const bool in_smem = subspace_in_smem(q, KS);
  const size_t sm2 = sizeof(double) * (size_t)((in_smem ? 3 * q * KS : 0) + 3 * KS * KS + 3 * KS);
  cudaFuncSetAttribute(k_cc_subspace<KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  k_cc_subspace<KS><<<(unsigned)g.neo, 256, sm2, s>>>(g, Ac, Bc, Hs, tol, maxit, Rcc, cc_evals,
                                                      iters, in_smem ? nullptr : work);
}

// R_cc rows and cc eigenvalues of every owned cc element for large q; scratch
// holds the shifted inverses (neo q^2 doubles, virtual-global like Winv),
// work coarse_large_work_doubles().
void launch_cc_basis_large(const GridParams& g, const double* Ac, const double* Bc,
                           double* scratch, double* work, double* Rcc, double* cc_evals,
                           int* scratch_status, int* iters, double tol, int maxit,
                           cudaStream_t s) {
  const int q = g.sd * g.sd * g.sd * g.lc;
  if (const char* e = getenv("TMG_CC_TOL")) tol = atof(e);  // diagnostics
  if (const char* e = getenv("TMG_CC_MAXIT")) maxit = atoi(e);
  double* Hs = scratch + g.e0 * q * q;
  k_elem_matrix<<<(unsigned)g.neo, 256, 0, s>>>(g, Ac, Bc, 1e-5, Hs);
  invert_elements(Hs, q, g.neo, work, scratch_status, s);
  if (subspace_width(g.lcc) == 16)
    launch_subspace<16>(g, Ac, Bc, Hs, tol, maxit, Rcc, cc_evals, iters, work, s);
  else
    launch_subspace<24>(g, Ac, Bc, Hs, tol, maxit, Rcc, cc_evals, iters, work, s);
}

}  // namespace tmg
