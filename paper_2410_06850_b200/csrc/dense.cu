// Coarsest-level direct solve (north_star item 6).
// The Gauss-Jordan sweeps keep only the lower triangle: for SPD A every sweep
// preserves A_ij = s_i s_j A_ji with s = -1 on processed pivot blocks, so the
// pivot row/column panels are rebuilt from lower entries, the trailing
// update skips tiles above the diagonal (half the DMMA work), and the final
// pass mirrors the symmetric inverse.
//
// Reference: DirectSolver (proj/core/src/solver.cpp:60-126) factorises A_cc
// with LDL^T once per set-up and solves once per V-cycle (:304). Here the SPD
// A_cc (n_cc = L_cc * m_cc) is inverted once per set-up by blocked in-place
// Gauss-Jordan sweeps (pivot block NB; the scalar pivots are the LDL^T pivots
// and the reference's singular-pivot rule d > 1e-14 max|d| is applied to
// them), symmetrised, and every V-cycle applies it as one bandwidth-bound
// GEMV — a single wide kernel instead of two latency-bound triangular solves.
#include "kernels.h"
#include "tma.cuh"
#include "symv.cuh"
#include "gj.cuh"

namespace tmg {

constexpr int NB = 64;  // Gauss-Jordan pivot block
// leading dimension of the Pn panel: rows start 16-byte aligned for the TMA
// bulk copies whatever the parity of n
__host__ __device__ __forceinline__ int64_t pn_ld(int64_t n) { return (n + 1) & ~(int64_t)1; }

// Invert the pivot block A[K,K] (nbk x nbk, nbk <= NB, identity-padded to NB)
// into Dinv and record the pivots: one CTA, register-resident Gauss-Jordan
// (gj.cuh).
constexpr int kDiagThreads = 256;
// Batched calls (dense_spd_inverse_batched): matrix blockIdx.z at A + z sA,
// its work (Dinv, Pn, Cold, pivots) at + z sW; single calls pass 0 strides.
__global__ void __launch_bounds__(kDiagThreads) k_gj_diag(const double* __restrict__ A, int64_t n,
                                                          int64_t k0, int nbk, double* Dinv,
                                                          double* pivots, int64_t sA,
                                                          int64_t sW) {
  A += blockIdx.z * sA;
  Dinv += blockIdx.z * sW;
  pivots += blockIdx.z * sW;
  using L = GjLayout<NB, kDiagThreads>;
  constexpr int CW = L::CW, RH = L::RH;
  __shared__ GjSmem<NB> gjs;
  const int lane = threadIdx.x & 31, c0 = CW * (threadIdx.x >> 5);
  double v[RH][CW];
#pragma unroll
  for (int h = 0; h < RH; ++h) {
    const int i = lane + 32 * h;
#pragma unroll
    for (int q = 0; q < CW; ++q) {
      const int j = c0 + q;
      v[h][q] = (i < nbk && j < nbk) ? (j <= i ? A[(k0 + i) * n + k0 + j] : A[(k0 + j) * n + k0 + i])
                                     : (i == j ? 1.0 : 0.0);
    }
  }
  double pmin = 1e300, pmax = 0.0;
  gj_invert<NB, kDiagThreads>(v, gjs, pmin, pmax, pivots + k0);
#pragma unroll
  for (int h = 0; h < RH; ++h) {
    const int i = lane + 32 * h;
#pragma unroll
    for (int q = 0; q < CW; ++q) {
      const int j = c0 + q;
      if (i < nbk && j < nbk) Dinv[i * nbk + j] = v[h][q];
    }
  }
}

// Pn[r][j] = sum_c Dinv[r][c] A[k0+c][j] (new pivot rows); Cold[i][c] = A[i][k0+c]
// (old pivot columns, ld NB, zero padded past nbk). CTA = 32 columns x 8 row
// groups of NB/8 rows.
__global__ void __launch_bounds__(256) k_gj_panels(const double* __restrict__ A, int64_t n,
                                                   int64_t k0, int nbk,
                                                   const double* __restrict__ Dinv, double* Pn,
                                                   double* Cold, int64_t sA, int64_t sW) {
  A += blockIdx.z * sA;
  Dinv += blockIdx.z * sW;
  Pn += blockIdx.z * sW;
  Cold += blockIdx.z * sW;
  __shared__ double Ds[NB][NB];  // read as warp broadcasts
  __shared__ double As[NB][32];
  const int t = threadIdx.x, jx = t & 31, ry = t >> 5;
  const int64_t j = blockIdx.x * 32LL + jx;
  for (int e = t; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    Ds[r][c] = (r < nbk && c < nbk) ? Dinv[r * nbk + c] : 0.0;
  }
  // A_{K,j} from the lower triangle: below the diagonal directly, above it
  // (j > row, both unprocessed: symmetric) from the mirror entry
  for (int c = ry; c < NB; c += 8) {
    const int64_t r = k0 + c;
    As[c][jx] = (c < nbk && j < n) ? (j <= r ? A[r * n + j] : A[j * n + r]) : 0.0;
  }
  __syncthreads();
  const int64_t ldp = pn_ld(n);
  if (j == n && j < ldp)  // odd n: the padding column (read by the even-width TMA rows)
    for (int q = 0; q < NB / 8; ++q) Pn[(ry * (NB / 8) + q) * ldp + j] = 0.0;
  if (j < n) {
    constexpr int RG = NB / 8;
    double acc[RG];
#pragma unroll
    for (int q = 0; q < RG; ++q) acc[q] = 0.0;
#pragma unroll 8
    for (int c = 0; c < NB; ++c) {
      const double a = As[c][jx];
#pragma unroll
      for (int q = 0; q < RG; ++q) acc[q] = fma(Ds[ry * RG + q][c], a, acc[q]);
    }
#pragma unroll
    for (int q = 0; q < RG; ++q) Pn[(ry * RG + q) * ldp + j] = acc[q];
  }
  // Cold: this CTA's 32 rows i = j-range, NB columns each; A_{i,K} from the
  // lower triangle (processed rows i < k0 carry the sign of the sweep:
  // A_iK = -A_Ki^T)
  for (int e = t; e < 32 * NB; e += 256) {
    const int64_t i = blockIdx.x * 32LL + e / NB;
    const int c = e % NB;
    const int64_t col = k0 + c;
    double v = 0.0;
    if (i < n && c < nbk) v = i >= col ? A[i * n + col] : (i >= k0 ? A[col * n + i] : -A[col * n + i]);
    if (i < n) Cold[i * NB + c] = v;
  }
}

__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Trailing update A -= Cold * Pn on FP64 tensor cores (mma.m8n8k4, DMMA).
// 128 x 64 output tile per CTA (2 CTAs per SM), 8 warps of 32 x 32; both panels are
// staged whole in shared memory (padded so each fragment load is 2
// wavefronts) while the C tile is prefetched into L2 by bulk prefetches. The
// pivot rows/columns get overwritten by k_gj_fix afterwards.
constexpr int GT = 128;              // output tile rows
constexpr int GN = 64;               // output tile columns
constexpr int AS_LD = NB + 4;        // smem row stride of the Cold panel
constexpr int BS_LD = GN + 8;        // smem row stride of the Pn panel
constexpr size_t kGemmSmem = sizeof(double) * (size_t)(GT * AS_LD + NB * BS_LD);

__global__ void __launch_bounds__(256, 2) k_gj_gemm(double* A, int64_t n,
                                                    const double* __restrict__ Cold,
                                                    const double* __restrict__ Pn, int64_t sA,
                                                    int64_t sW) {
  A += blockIdx.z * sA;
  Cold += blockIdx.z * sW;
  Pn += blockIdx.z * sW;
  extern __shared__ __align__(16) double smg[];
  double* As = smg;
  double* Bs = smg + GT * AS_LD;
  const int64_t i0 = (int64_t)blockIdx.y * GT, j0 = (int64_t)blockIdx.x * GN;
  if (i0 + GT - 1 < j0) return;  // strictly above the diagonal: not maintained
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t < GT && i0 + t < n && !(n & 1)) {  // (16-byte aligned rows only)
    const int64_t cols = (n - j0) < GN ? (n - j0) : GN;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A + (i0 + t) * n + j0),
                 "r"((unsigned)(cols * sizeof(double)))
                 : "memory");
  }
  // both operand panels arrive by TMA bulk copies (one per panel row) on one
  // mbarrier; rows past n are zero-filled by the threads instead
  __shared__ uint64_t bar;
  const int rows_a = (int)((n - i0) < GT ? (n - i0) : GT);
  const int64_t ldp = pn_ld(n);
  // even width: the copy size stays a multiple of 16 bytes (odd n: one
  // padding column of Pn, zero, rides along)
  const int cols_b = (int)((ldp - j0) < GN ? (ldp - j0) : GN);
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (t == 0)
    mbar_arrive_expect_tx(&bar, (uint32_t)(sizeof(double) * (rows_a * NB + NB * cols_b)));
  __syncwarp();
  if (w == 0) {
    for (int r = lane; r < rows_a; r += 32)
      bulk_g2s(As + r * AS_LD, Cold + (i0 + r) * NB, NB * sizeof(double), &bar);
    for (int r = lane; r < NB; r += 32)
      bulk_g2s(Bs + r * BS_LD, Pn + r * ldp + j0, (uint32_t)(cols_b * sizeof(double)), &bar);
  }
  for (int e = rows_a * AS_LD + t; e < GT * AS_LD; e += 256) As[e] = 0.0;
  if (cols_b < GN)
    for (int e = t; e < NB * GN; e += 256)
      if (e % GN >= cols_b) Bs[(e / GN) * BS_LD + e % GN] = 0.0;
  mbar_wait(&bar, 0);
  __syncthreads();
  const int wm = w & 3, wn = w >> 2;  // warp tile rows 32 wm.., cols 32 wn..
  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  const double* ap = As + (32 * wm + (lane >> 2)) * AS_LD + (lane & 3);
  const double* bp = Bs + (lane & 3) * BS_LD + 32 * wn + (lane >> 2);
#pragma unroll 2
  for (int k = 0; k < NB; k += 4) {
    double a[4], b[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = ap[mi * 8 * AS_LD + k];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = bp[k * BS_LD + 8 * ni];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma_m8n8k4(acc[mi][ni], a[mi], b[ni]);
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int64_t i = i0 + 32 * wm + 8 * mi + (lane >> 2);
    if (i >= n) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int64_t j = j0 + 32 * wn + 8 * ni + 2 * (lane & 3);
      if (j >= n) continue;
      if (!(n & 1)) {
        double2* cp = reinterpret_cast<double2*>(A + i * n + j);
        double2 c = *cp;
        c.x -= acc[mi][ni][0];
        c.y -= acc[mi][ni][1];
        *cp = c;
      } else {  // odd n: rows are not 16-byte aligned; column n is padding
        A[i * n + j] -= acc[mi][ni][0];
        if (j + 1 < n) A[i * n + j + 1] -= acc[mi][ni][1];
      }
    }
  }
}

// Pivot rows <- Pn, pivot block <- Dinv, pivot columns <- -Cold Dinv.
__global__ void __launch_bounds__(256) k_gj_fix(double* A, int64_t n, int64_t k0, int nbk,
                                                const double* __restrict__ Dinv,
                                                const double* __restrict__ Pn,
                                                const double* __restrict__ Cold, int64_t sA,
                                                int64_t sW) {
  A += blockIdx.z * sA;
  Dinv += blockIdx.z * sW;
  Pn += blockIdx.z * sW;
  Cold += blockIdx.z * sW;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * nbk) return;
  // rows: e -> (r, j); the lower triangle only (j < k0 + nbk)
  {
    const int r = (int)(e / n);
    const int64_t j = e % n;
    const bool jK = j >= k0 && j < k0 + nbk;
    if (j < k0 + nbk) A[(k0 + r) * n + j] = jK ? Dinv[r * nbk + (j - k0)] : Pn[r * pn_ld(n) + j];
  }
  // columns: e -> (i, c); below the pivot block only
  {
    const int64_t i = e / nbk;
    const int c = (int)(e % nbk);
    if (i >= k0 + nbk) {
      double s = 0.0;
      for (int q = 0; q < nbk; ++q) s = fma(Cold[i * NB + q], Dinv[q * nbk + c], s);
      A[i * n + k0 + c] = -s;
    }
  }
}

__global__ void k_symmetrize(double* A, int64_t n, int64_t sA) {
  A += blockIdx.z * sA;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * n) return;
  const int64_t i = e / n, j = e % n;
  if (i < j) A[i * n + j] = A[j * n + i];  // the sweeps kept the lower triangle
}

__global__ void k_pivot_check(const double* pivots, int64_t n, int* status, int64_t sW) {
  pivots += blockIdx.z * sW;
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
                                              const double* __restrict__ A, int64_t nrows,
                                              int64_t ncols, const double* __restrict__ x,
                                              double* y) {
  pdl_trigger();
  pdl_wait();
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= nrows) return;
  const double* a = A + row * ncols;
  double s = 0.0;
  if ((ncols & 1) == 0) {
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const double2* x2 = reinterpret_cast<const double2*>(x);
    for (int64_t j = lane; j < ncols / 2; j += 32) {
      const double2 av = __ldg(a2 + j), xv = __ldg(x2 + j);
      s = fma(av.x, xv.x, s);
      s = fma(av.y, xv.y, s);
    }
  } else {
    for (int64_t j = lane; j < ncols; j += 32) s = fma(__ldg(a + j), __ldg(x + j), s);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = s;
}

// ------------------------------------------------ symmetric tiled GEMV
// (symv.cuh). Persistent: one or two CTAs per SM.
__global__ void __launch_bounds__(256) k_symv_tiles(const int* __restrict__ done,
                                                    const double* __restrict__ T, int64_t n,
                                                    const double* __restrict__ x, double* P) {
  pdl_trigger();
  extern __shared__ __align__(128) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>(smraw);  // kSymvSlots x TS*TS
  double* xs = ring + kSymvSlots * TS * TS;         // all of x, zero padded to nt*TS
  __shared__ SymvSmem ss;
  symv_begin(ss, ring, T, n);  // constant tiles: before the dependency wait
  pdl_wait();
  if (done && *done) {
    symv_drain(ss, n);
    return;
  }
  symv_run(ss, ring, xs, T, n, x, P);
}

__global__ void k_pack_sym_tiles(const double* __restrict__ A, int64_t n, double* T) {
  const int64_t tile = blockIdx.x;
  int64_t I, J;
  symv_tile_ij(tile, I, J);
  for (int e = threadIdx.x; e < TS * TS; e += blockDim.x) {
    const int64_t r = I * TS + e / TS, c = J * TS + e % TS;
    T[tile * TS * TS + e] = (r < n && c < n) ? A[r * n + c] : 0.0;
  }
}

__global__ void k_symv_reduce(const int* __restrict__ done, const double* __restrict__ P,
                              int64_t n, double* y) {
  pdl_trigger();
  pdl_wait();
  if (done && *done) return;
  const int64_t nt = (n + TS - 1) / TS;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t I = k / TS, r = k % TS;
  double s = 0.0;
  for (int64_t J = 0; J < nt; ++J) s += P[(I * nt + J) * TS + r];
  y[k] = s;
}

int64_t sym_tiles_doubles(int64_t n) {
  const int64_t nt = (n + TS - 1) / TS;
  return nt * (nt + 1) / 2 * TS * TS;
}
int64_t sym_partials_doubles(int64_t n) {
  const int64_t nt = (n + TS - 1) / TS;
  return nt * nt * TS;
}

void pack_sym_tiles(const double* A, int64_t n, double* T, cudaStream_t s) {
  const int64_t nt = (n + TS - 1) / TS;
  k_pack_sym_tiles<<<(unsigned)(nt * (nt + 1) / 2), 256, 0, s>>>(A, n, T);
}

void launch_symv(const int* done, const double* T, int64_t n, const double* x, double* P, double* y,
                 cudaStream_t s) {
  const int64_t nt = (n + TS - 1) / TS;
  const size_t smem = symv_dyn_smem(n);
  const int64_t ntiles = nt * (nt + 1) / 2;
  const int64_t slots = (int64_t)device_occupancy(k_symv_tiles, 256, smem) * device_sm_count();
  const unsigned grid = (unsigned)(ntiles < slots ? ntiles : slots);
  launch_pdl(k_symv_tiles, dim3(grid), dim3(256), smem, s, done, T, n, x, P);
  launch_pdl(k_symv_reduce, dim3((unsigned)((n + 127) / 128)), dim3(128), 0, s, done, P, n, y);
}

// work per matrix: NB*NB (Dinv) + NB*ldp (Pn) + ldp*NB (Cold) + ldp + NB
// (pivots), ldp = n rounded up to even: every panel starts 16-byte aligned
static void gj_inverse_impl(double* A, int64_t n, int64_t batch, int64_t sA, double* work,
                            int64_t sW, int* status, cudaStream_t s) {
  const int64_t ldp = pn_ld(n);
  double* Dinv = work;
  double* Pn = Dinv + NB * NB;
  double* Cold = Pn + (int64_t)NB * ldp;
  double* piv = Cold + ldp * NB;
  const unsigned B = (unsigned)batch;
  cudaFuncSetAttribute(k_gj_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem);
  const dim3 grid((unsigned)((n + GN - 1) / GN), (unsigned)((n + GT - 1) / GT), B);
  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    const int nbk = (int)((n - k0) < NB ? (n - k0) : NB);
    k_gj_diag<<<dim3(1, 1, B), kDiagThreads, 0, s>>>(A, n, k0, nbk, Dinv, piv, sA, sW);
    k_gj_panels<<<dim3((unsigned)((n + 31) / 32), 1, B), 256, 0, s>>>(A, n, k0, nbk, Dinv, Pn,
                                                                      Cold, sA, sW);
    k_gj_gemm<<<grid, 256, kGemmSmem, s>>>(A, n, Cold, Pn, sA, sW);
    k_gj_fix<<<dim3((unsigned)((n * nbk + 255) / 256), 1, B), 256, 0, s>>>(A, n, k0, nbk, Dinv,
                                                                            Pn, Cold, sA, sW);
  }
  k_symmetrize<<<dim3((unsigned)((n * n + 255) / 256), 1, B), 256, 0, s>>>(A, n, sA);
  k_pivot_check<<<dim3(1, 1, B), 1024, 0, s>>>(piv, n, status, sW);
}

void dense_spd_inverse(double* A, int64_t n, double* work, int* status, cudaStream_t s) {
  gj_inverse_impl(A, n, 1, 0, work, 0, status, s);
}

// batch SPD matrices of order n at A + b n^2, each inverted in place (same
// blocked Gauss-Jordan, the batch on gridDim.z); work: batch *
// dense_inverse_work_doubles(n). A singular pivot sets *status = 3.
void dense_spd_inverse_batched(double* A, int64_t n, int64_t batch, double* work, int* status,
                               cudaStream_t s) {
  gj_inverse_impl(A, n, batch, n * n, work, dense_inverse_work_doubles(n), status, s);
}

// (+ NB: the identity-padded last pivot block writes NB pivots)
int64_t dense_inverse_work_doubles(int64_t n) {
  return NB * NB + 2 * (int64_t)NB * pn_ld(n) + pn_ld(n) + NB;
}

// the n LDL^T pivots of batch matrix z after dense_spd_inverse_batched
const double* dense_inverse_pivots(const double* work, int64_t n, int64_t z) {
  return work + z * dense_inverse_work_doubles(n) + NB * NB + 2 * (int64_t)NB * pn_ld(n);
}

void launch_gemv(const int* done, const double* A, int64_t n, const double* x, double* y,
                 cudaStream_t s) {
  k_gemv<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(done, A, n, n, x, y);
}

void launch_gemv_block(const int* done, const double* A, int64_t nrows, int64_t ncols,
                       const double* x, double* y, cudaStream_t s) {
  launch_pdl(k_gemv, dim3((unsigned)((nrows + 7) / 8)), dim3(256), 0, s, done, A, nrows, ncols, x,
             y);
}

void launch_gemv_rows(const int* done, const double* A, int64_t n, int64_t row0, int64_t nrows,
                      const double* x, double* y, cudaStream_t s) {
  // rows of A and y shifted so the kernel's row r is global row row0 + r
  launch_pdl(k_gemv, dim3((unsigned)((nrows + 7) / 8)), dim3(256), 0, s, done, A + row0 * n, nrows,
             n, x, y + row0);
}

}  // namespace tmg
