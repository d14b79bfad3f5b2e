// The coarse-coarse direct solve (DirectSolver on A_cc, solver.cpp:60-126) as
// a block Thomas over the z-planes of cc elements. In the cc dof order
// (element-major, elements x-fastest) A_cc = R_cc A_c R_cc^T is block
// tridiagonal over the ncz planes of P = ncx ncy L_cc unknowns: A_kk couples
// the elements of plane k (self, x and y faces); A_{k,k-1} = C_k is block
// diagonal, one L_cc x L_cc block per element (its z-lo face).
//   set-up: G_0 = A_00^-1, G_k = (A_kk - C_k G_{k-1} C_k^T)^-1 (blocked
//           Gauss-Jordan on the tensor cores, the reference's pivot rule),
//           each packed into symmetric 64 x 64 tiles;
//   solve:  y_k = G_k (r_k - C_k y_{k-1}), x_k = y_k - G_k C_{k+1}^T x_{k+1}.
// At 512^3 (n_cc = 49152, P = 3072) this replaces a 49152^2 inverse (7.5 s,
// 29 GB with its tiles) by 16 inverses of 3072^2 (0.6 GB of tiles).
#include "coarse_elem.cuh"
#include "kernels.h"

namespace tmg {

// Schur update of plane k: S[a,b] -= C_a G[a,b] C_b^T per pair of elements
// (a, b) of the plane (L x L blocks), G = G_{k-1} (full symmetric, ld P).
__global__ void k_acc_schur(double* S, const double* __restrict__ G,
                            const double* __restrict__ C, int64_t P, int L) {
  extern __shared__ double sm[];
  double* Gab = sm;
  double* Ca = Gab + L * L;
  double* Cb = Ca + L * L;
  double* T1 = Cb + L * L;
  const int64_t a = blockIdx.y, b = blockIdx.x;
  for (int e = threadIdx.x; e < L * L; e += blockDim.x) {
    const int i = e / L, j = e % L;
    Gab[e] = G[(a * L + i) * P + b * L + j];
    Ca[e] = C[a * L * L + e];
    Cb[e] = C[b * L * L + e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < L * L; e += blockDim.x) {  // T1 = C_a G_ab
    const int i = e / L, j = e % L;
    double s = 0.0;
    for (int m = 0; m < L; ++m) s = fma(Ca[i * L + m], Gab[m * L + j], s);
    T1[e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < L * L; e += blockDim.x) {  // S_ab -= T1 C_b^T
    const int i = e / L, j = e % L;
    double s = 0.0;
    for (int m = 0; m < L; ++m) s = fma(T1[i * L + m], Cb[j * L + m], s);
    S[(a * L + i) * P + b * L + j] -= s;
  }
}

// w = r - C y (forward, with y = y_{k-1}) or w = C^T x (backward, x = x_{k+1});
// C block diagonal (one L x L block per element of the plane)
__global__ void k_acc_couple(const int* __restrict__ done, const double* __restrict__ C,
                             const double* __restrict__ v, const double* __restrict__ r,
                             double* w, int64_t P, int L, int transpose) {
  pdl_trigger();
  pdl_wait();
  if (*done) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int64_t e = i / L;
  const int a = (int)(i % L);
  const double* Ce = C + e * L * L;
  const double* ve = v + e * L;
  double s = 0.0;
  for (int m = 0; m < L; ++m) s = fma(transpose ? Ce[m * L + a] : Ce[a * L + m], ve[m], s);
  w[i] = transpose ? s : r[i] - s;
}

// x -= t
__global__ void k_acc_sub(const int* __restrict__ done, double* x, const double* __restrict__ t,
                          int64_t P) {
  pdl_trigger();
  pdl_wait();
  if (*done) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < P) x[i] -= t[i];
}

int64_t acc_planes_doubles(const GridParams& g) {
  const int64_t P = g.ncx * g.ncy * g.lcc;
  // tiles per plane + coupling blocks + 2 work vectors
  return g.ncz * sym_tiles_doubles(P) + g.ncz * g.ncx * g.ncy * g.lcc * g.lcc + 2 * P;
}

// Factor from the plane blocks (Gd: ncz dense P x P diagonal blocks, C: the
// z-lo coupling blocks, both written by launch_acc_assemble_planes); Gd is
// consumed (inverted in place). Output tiles T (ncz * sym_tiles_doubles(P)).
void acc_planes_factor(const GridParams& g, double* Gd, const double* C, double* T, double* work,
                       int* status, cudaStream_t s) {
  const int64_t P = g.ncx * g.ncy * g.lcc, nxy = g.ncx * g.ncy;
  const int L = g.lcc;
  const size_t sm = sizeof(double) * 4 * L * L;
  for (int64_t k = 0; k < g.ncz; ++k) {
    double* Sk = Gd + k * P * P;
    if (k > 0)
      k_acc_schur<<<dim3((unsigned)nxy, (unsigned)nxy), 128, sm, s>>>(
          Sk, Sk - P * P, C + k * nxy * L * L, P, L);
    dense_spd_inverse(Sk, P, work, status, s);
    if (T) pack_sym_tiles(Sk, P, T + k * sym_tiles_doubles(P), s);  // T null: keep Gd only
  }
}

// ecc = A_cc^-1 rcc through the plane factors. wv: 2P doubles of work,
// partials: sym_partials_doubles(P).
void launch_acc_planes_solve(const GridParams& g, const int* done, const double* T,
                             const double* C, const double* rcc, double* ecc, double* wv,
                             double* partials, cudaStream_t s) {
  const int64_t P = g.ncx * g.ncy * g.lcc, nxy = g.ncx * g.ncy, K = g.ncz;
  const int L = g.lcc;
  const int64_t ts = sym_tiles_doubles(P);
  double* w = wv;
  double* t = wv + P;
  const unsigned nb = (unsigned)((P + 255) / 256);
  for (int64_t k = 0; k < K; ++k) {
    const double* rk = rcc + k * P;
    if (k == 0) {
      launch_symv(done, T, P, rk, partials, ecc, s);
    } else {
      launch_pdl(k_acc_couple, dim3(nb), dim3(256), 0, s, done, C + k * nxy * L * L,
                 (const double*)(ecc + (k - 1) * P), rk, w, P, L, 0);
      launch_symv(done, T + k * ts, P, w, partials, ecc + k * P, s);
    }
  }
  for (int64_t k = K - 2; k >= 0; --k) {
    launch_pdl(k_acc_couple, dim3(nb), dim3(256), 0, s, done, C + (k + 1) * nxy * L * L,
               (const double*)(ecc + (k + 1) * P), (const double*)nullptr, w, P, L, 1);
    launch_symv(done, T + k * ts, P, w, partials, t, s);
    launch_pdl(k_acc_sub, dim3(nb), dim3(256), 0, s, done, ecc + k * P, (const double*)t, P);
  }
}

// Row-distributed plane solve (partitioned contexts): slab j
// keeps rows [r0, r0 + nr) of every dense plane inverse, R[k][nr][P]; every
// plane step forms the coupled right-hand side (replicated, P values), each
// slab multiplies its row block, and the caller all-gathers the plane's
// rows between steps (`gather`, an in-place NCCL all-gather; nothing for the
// slabs of one process, which share x).
void launch_acc_rows_solve(const GridParams& g, const int* done, const double* C,
                           const double* rcc, double* ecc, double* wv,
                           const std::vector<AccRowBlock>& blocks,
                           const std::function<void(double* plane)>& gather, cudaStream_t s) {
  const int64_t P = g.ncx * g.ncy * g.lcc, nxy = g.ncx * g.ncy, K = g.ncz;
  const int L = g.lcc;
  double* w = wv;
  double* t = wv + P;
  const unsigned nb = (unsigned)((P + 255) / 256);
  for (int64_t k = 0; k < K; ++k) {
    const double* rk = rcc + k * P;
    const double* in = rk;
    if (k > 0) {
      launch_pdl(k_acc_couple, dim3(nb), dim3(256), 0, s, done, C + k * nxy * L * L,
                 (const double*)(ecc + (k - 1) * P), rk, w, P, L, 0);
      in = w;
    }
    for (const AccRowBlock& b : blocks)
      launch_gemv_block(done, b.R + k * b.nr * P, b.nr, P, in, ecc + k * P + b.r0, s);
    gather(ecc + k * P);
  }
  for (int64_t k = K - 2; k >= 0; --k) {
    launch_pdl(k_acc_couple, dim3(nb), dim3(256), 0, s, done, C + (k + 1) * nxy * L * L,
               (const double*)(ecc + (k + 1) * P), (const double*)nullptr, w, P, L, 1);
    for (const AccRowBlock& b : blocks) {
      launch_gemv_block(done, b.R + k * b.nr * P, b.nr, P, w, t + b.r0, s);
      launch_pdl(k_acc_sub, dim3((unsigned)((b.nr + 255) / 256)), dim3(256), 0, s, done,
                 ecc + k * P + b.r0, (const double*)(t + b.r0), b.nr);
    }
    gather(ecc + k * P);
  }
}

int acc_rows_solve_kernels(const GridParams& g, int nblocks) {
  return (int)((g.ncz - 1) + g.ncz * nblocks + (g.ncz - 1) * (1 + 2 * nblocks));
}

// kernels launched per solve (for the launch count)
int acc_planes_solve_kernels(const GridParams& g) { return (int)(2 + 7 * (g.ncz - 1)); }

}  // namespace tmg
