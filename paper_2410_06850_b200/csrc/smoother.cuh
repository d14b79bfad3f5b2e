// Fine-level smoother: exact block-Jacobi with one block per coarse cell
// (north_star item 2).
//
// Reference semantics: BlockJacobiSmoother (proj/core/src/solver.cpp:128-251)
// with the partition {cells_of_coarse(I)} — one sweep from z = 0 gives
// z_I = A_II^{-1} r_I, the exact solve of the coarse cell's diagonal block of A.
// The reference factorises each block with Eigen LDL^T (solver.cpp:69-109); here
// each brick's block is factorised as a block-tridiagonal matrix over its CB
// z-planes (CB^2 cells each): S_0 = A_0, S_k = A_k - B_k S_{k-1}^{-1} B_k with
// B_k = diag(-T_z) the plane coupling, and the Schur inverses G_k = S_k^{-1}
// are stored densely (packed symmetric). One solve is then 2*CB-1 dense
// CB^2 x CB^2 mat-vecs — the same arithmetic as the LDL^T solve, reorganised
// into wide parallel steps. The pivots of the in-place Gauss-Jordan sweeps are
// the LDL^T pivots of A_II in natural order; the reference's singular-pivot
// rule (d_i > 1e-14 max|d|, solver.cpp:86-92) is applied to them.
#pragma once
#include "stencil.cuh"

namespace tmg {

template <int CB>
struct Thomas {
  static constexpr int P = CB * CB;              // cells per plane
  static constexpr int PP = P * (P + 1) / 2;     // packed symmetric plane
  static constexpr int PER_BRICK = CB * PP;      // doubles per brick
  static constexpr int TPR = CB;                 // threads per mat-vec row
  __device__ static __forceinline__ int pidx(int i, int j) {
    return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i;
  }
};

// y_i = sum_j G(i,j) w_j over one plane; G packed in smem, w in smem.
// Thread layout: row i = tid / TPR, lane-group sum over j = s, s+TPR, ...
// Returns the row value in the TPR threads of row i (all lanes of the group).
template <int CB>
__device__ __forceinline__ double plane_matvec(const double* Gp, const double* w) {
  constexpr int P = Thomas<CB>::P, TPR = Thomas<CB>::TPR;
  const int i = threadIdx.x / TPR, s = threadIdx.x % TPR;
  double acc = 0.0;
#pragma unroll
  for (int j = s; j < P; j += TPR) acc = fma(Gp[Thomas<CB>::pidx(i, j)], w[j], acc);
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// Exact block solve x = A_II^{-1} t for one brick.
//  t   : smem, C values (brick order, plane k = t[k*P .. k*P+P))
//  tz  : smem, C values; tz[l] = T_z between cell l and the cell one plane below
//        (0 for lk = 0)
//  u   : smem scratch, C values;  x : smem output, C values (may alias t)
//  gbuf: smem, PP values
//  G   : global, this brick's CB planes of packed inverses
template <int CB>
__device__ __forceinline__ void thomas_solve(const double* __restrict__ G, const double* t,
                                             const double* tz, double* u, double* x, double* gbuf,
                                             double* w) {
  constexpr int P = Thomas<CB>::P, PP = Thomas<CB>::PP, C = CB * CB * CB, TPR = Thomas<CB>::TPR;
  const int tid = threadIdx.x;
  const int row = tid / TPR, sub = tid % TPR;
  // forward: w_k = t_k + Tz_k * u_{k-1};  u_k = G_k w_k
  for (int k = 0; k < CB; ++k) {
    for (int e = tid; e < PP; e += C) gbuf[e] = __ldg(G + (size_t)k * PP + e);
    if (tid < P) {
      const int l = k * P + tid;
      w[tid] = k == 0 ? t[l] : fma(tz[l], u[l - P], t[l]);
    }
    __syncthreads();
    const double y = plane_matvec<CB>(gbuf, w);
    if (sub == 0) u[k * P + row] = y;
    __syncthreads();
  }
  // backward: x_{K-1} = u_{K-1};  x_k = u_k - G_k (B_{k+1} x_{k+1}),  B = -Tz
  if (tid < P) x[(CB - 1) * P + tid] = u[(CB - 1) * P + tid];
  for (int k = CB - 2; k >= 0; --k) {
    for (int e = tid; e < PP; e += C) gbuf[e] = __ldg(G + (size_t)k * PP + e);
    if (tid < P) {
      const int l = (k + 1) * P + tid;
      w[tid] = -tz[l] * x[l];
    }
    __syncthreads();
    const double y = plane_matvec<CB>(gbuf, w);
    if (sub == 0) x[k * P + row] = u[k * P + row] - y;
    __syncthreads();
  }
}

}  // namespace tmg
