// Coarsest-level direct solve (north_star item 6).
//
// Reference: DirectSolver (proj/core/src/solver.cpp:60-126) factorises A_cc
// with LDL^T once per set-up and solves once per V-cycle (:304). Here the SPD
// A_cc (n_cc = L_cc * m_cc) is inverted once per set-up by blocked in-place
// Gauss-Jordan sweeps (pivot block NB; the scalar pivots are the LDL^T pivots
// and the reference's singular-pivot rule d > 1e-14 max|d| is applied to
// them), symmetrised, and every V-cycle applies it as one bandwidth-bound
// GEMV — a single wide kernel instead of two latency-bound triangular solves.
#include "kernels.h"

namespace tmg {

constexpr int NB = 32;

// Invert the pivot block A[K,K] (nbk x nbk) into Dinv (NB x NB), record pivots.
__global__ void k_gj_diag(const double* __restrict__ A, int64_t n, int64_t k0, int nbk,
                          double* Dinv, double* pivots) {
  __shared__ double M[NB * NB];
  __shared__ double col[NB], rowp[NB];
  for (int e = threadIdx.x; e < nbk * nbk; e += blockDim.x) {
    const int i = e / nbk, j = e % nbk;
    M[e] = A[(k0 + i) * n + k0 + j];
  }
  __syncthreads();
  for (int p = 0; p < nbk; ++p) {
    const double pv = M[p * nbk + p];
    if (threadIdx.x < nbk) {
      col[threadIdx.x] = M[threadIdx.x * nbk + p];
      rowp[threadIdx.x] = M[p * nbk + threadIdx.x];
    }
    if (threadIdx.x == 0) pivots[k0 + p] = pv;
    __syncthreads();
    const double inv = 1.0 / pv;
    for (int e = threadIdx.x; e < nbk * nbk; e += blockDim.x) {
      const int i = e / nbk, j = e % nbk;
      double v;
      if (i == p && j == p) v = inv;
      else if (i == p) v = rowp[j] * inv;
      else if (j == p) v = -col[i] * inv;
      else v = M[e] - col[i] * (rowp[j] * inv);
      M[e] = v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nbk * nbk; e += blockDim.x) Dinv[e] = M[e];
}

// Pn[r][j] = sum_c Dinv[r][c] A[k0+c][j]  (row panel, new);  Cold[i][c] = A[i][k0+c]
__global__ void k_gj_panels(const double* __restrict__ A, int64_t n, int64_t k0, int nbk,
                            const double* __restrict__ Dinv, double* Pn, double* Cold) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  double a[NB];
  for (int c = 0; c < nbk; ++c) a[c] = A[(k0 + c) * n + j];
  for (int r = 0; r < nbk; ++r) {
    double s = 0.0;
    for (int c = 0; c < nbk; ++c) s += Dinv[r * nbk + c] * a[c];
    Pn[r * n + j] = s;
  }
  // by symmetry of the current iterate's structure we still copy the column explicitly
  for (int c = 0; c < nbk; ++c) Cold[j * NB + c] = A[j * n + k0 + c];
}

// A <- swept(A) given Dinv, Pn (new row panel), Cold (old column panel).
// 64 x 64 tiles, 256 threads, 4 x 4 per thread.
__global__ void __launch_bounds__(256) k_gj_update(double* A, int64_t n, int64_t k0, int nbk,
                                                   const double* __restrict__ Dinv,
                                                   const double* __restrict__ Pn,
                                                   const double* __restrict__ Cold) {
  __shared__ double Cs[64][NB + 1];
  __shared__ double Ps[NB][64 + 1];
  __shared__ double Ds[NB][NB + 1];
  const int64_t i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  for (int e = threadIdx.x; e < 64 * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    const int64_t i = i0 + r;
    Cs[r][c] = (i < n && c < nbk) ? Cold[i * NB + c] : 0.0;
  }
  for (int e = threadIdx.x; e < NB * 64; e += 256) {
    const int r = e / 64, c = e % 64;
    const int64_t j = j0 + c;
    Ps[r][c] = (j < n && r < nbk) ? Pn[r * n + j] : 0.0;
  }
  for (int e = threadIdx.x; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    Ds[r][c] = (r < nbk && c < nbk) ? Dinv[r * nbk + c] : 0.0;
  }
  __syncthreads();
  for (int a = 0; a < 4; ++a) {
    const int r = ty + 16 * a;
    const int64_t i = i0 + r;
    if (i >= n) continue;
    const bool iK = i >= k0 && i < k0 + nbk;
    for (int b = 0; b < 4; ++b) {
      const int c = tx + 16 * b;
      const int64_t j = j0 + c;
      if (j >= n) continue;
      const bool jK = j >= k0 && j < k0 + nbk;
      double v;
      if (iK && jK) {
        v = Ds[i - k0][j - k0];
      } else if (iK) {
        v = Ps[i - k0][c];
      } else if (jK) {
        // -A_iK Dinv
        double s = 0.0;
        for (int q = 0; q < nbk; ++q) s += Cs[r][q] * Ds[q][j - k0];
        v = -s;
      } else {
        double s = 0.0;
        for (int q = 0; q < nbk; ++q) s += Cs[r][q] * Ps[q][c];
        v = A[i * n + j] - s;
      }
      A[i * n + j] = v;
    }
  }
}

__global__ void k_symmetrize(double* A, int64_t n) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * n) return;
  const int64_t i = e / n, j = e % n;
  if (i < j) {
    const double s = 0.5 * (A[i * n + j] + A[j * n + i]);
    A[i * n + j] = s;
    A[j * n + i] = s;
  }
}

__global__ void k_pivot_check(const double* pivots, int64_t n, int* status) {
  __shared__ double red[32];
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, fabs(pivots[i]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    red[0] = m;
  }
  __syncthreads();
  const double m = red[0];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    if (!(pivots[i] > 1e-14 * m)) atomicExch(status, 3);
}

// y = A x, one warp per row, fixed-order lane-strided sums (deterministic).
__global__ void __launch_bounds__(256) k_gemv(const int* __restrict__ done,
                                              const double* __restrict__ A, int64_t n,
                                              const double* __restrict__ x, double* y) {
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  const double* a = A + row * n;
  double s = 0.0;
  if ((n & 1) == 0) {
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const double2* x2 = reinterpret_cast<const double2*>(x);
    for (int64_t j = lane; j < n / 2; j += 32) {
      const double2 av = __ldg(a2 + j), xv = __ldg(x2 + j);
      s = fma(av.x, xv.x, s);
      s = fma(av.y, xv.y, s);
    }
  } else {
    for (int64_t j = lane; j < n; j += 32) s = fma(__ldg(a + j), __ldg(x + j), s);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = s;
}

void dense_spd_inverse(double* A, int64_t n, double* work, int* status, cudaStream_t s) {
  // work: NB*NB (Dinv) + NB*n (Pn) + n*NB (Cold) + n (pivots)
  double* Dinv = work;
  double* Pn = Dinv + NB * NB;
  double* Cold = Pn + (int64_t)NB * n;
  double* piv = Cold + n * NB;
  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    const int nbk = (int)((n - k0) < NB ? (n - k0) : NB);
    k_gj_diag<<<1, 256, 0, s>>>(A, n, k0, nbk, Dinv, piv);
    k_gj_panels<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(A, n, k0, nbk, Dinv, Pn, Cold);
    dim3 grid((unsigned)((n + 63) / 64), (unsigned)((n + 63) / 64));
    k_gj_update<<<grid, 256, 0, s>>>(A, n, k0, nbk, Dinv, Pn, Cold);
  }
  k_symmetrize<<<(unsigned)((n * n + 255) / 256), 256, 0, s>>>(A, n);
  k_pivot_check<<<1, 1024, 0, s>>>(piv, n, status);
}

int64_t dense_inverse_work_doubles(int64_t n) { return NB * NB + 2 * (int64_t)NB * n + n; }

void launch_gemv(const int* done, const double* A, int64_t n, const double* x, double* y,
                 cudaStream_t s) {
  k_gemv<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(done, A, n, x, y);
}

}  // namespace tmg
