// In-place inverse of an SPD q x q matrix in global memory by one CTA of 256
// threads (q a multiple of 64, q <= 256): blocked Gauss-Jordan sweeps with
// 64 x 64 pivot blocks. Thread j owns column j: the trailing update
// A_ij -= Cold_i . Pn_j reads the old pivot columns Cold (q x 64, shared
// memory) and keeps its own new pivot-row entries Pn_j (64 values) in
// registers; the pivot blocks are inverted register-resident (gj.cuh). pmin /
// pmax collect the LDL^T pivots (natural order) this thread saw. Symmetrised
// on exit. Used by the large-element coarse level (coarse_large.cu) and the
// cc-element block-Jacobi factors (block_jacobi.cu).
#pragma once
#include "gj.cuh"

namespace tmg {

constexpr int kGjBlock = 64;     // pivot block
constexpr int kGjThreads = 256;  // one column per thread (q <= 256)

struct GjGlobalSmem {
  double* Cold;  // q x 64
  double* Ds;    // 64 x 64
  double* Dt;    // its transpose
};
__host__ __device__ inline size_t gj_global_smem_bytes(int q) {
  return sizeof(double) * (size_t)(q * kGjBlock + 2 * kGjBlock * kGjBlock);
}
__device__ inline GjGlobalSmem gj_global_smem(double* base, int q) {
  return {base, base + q * kGjBlock, base + q * kGjBlock + kGjBlock * kGjBlock};
}

__device__ inline void gj_inverse_global(double* M, int q, const GjGlobalSmem& sm,
                                         GjSmem<kGjBlock>& gjs, double& pmin, double& pmax) {
  constexpr int GB = kGjBlock, GJT = kGjThreads;
  double* Cold = sm.Cold;
  double* Ds = sm.Ds;
  double* Dt = sm.Dt;
  const int t = threadIdx.x, lane = t & 31;
  using L = GjLayout<GB, GJT>;
  constexpr int CW = L::CW, RH = L::RH;
  const int c0 = CW * (t >> 5);
  for (int K = 0; K < q / GB; ++K) {
    const int k0 = K * GB;
    // (a) pivot block inverse (register-resident)
    double v[RH][CW];
#pragma unroll
    for (int h = 0; h < RH; ++h)
#pragma unroll
      for (int qq = 0; qq < CW; ++qq) v[h][qq] = M[(k0 + lane + 32 * h) * q + k0 + c0 + qq];
    gj_invert<GB, GJT>(v, gjs, pmin, pmax);
#pragma unroll
    for (int h = 0; h < RH; ++h)
#pragma unroll
      for (int qq = 0; qq < CW; ++qq) Ds[(lane + 32 * h) * GB + c0 + qq] = v[h][qq];
    // (b) old pivot columns; D^-1 transposed for the pivot-row product
    for (int e = t; e < q * GB; e += GJT) Cold[e] = M[(e / GB) * q + k0 + e % GB];
    for (int e = t; e < GB * GB; e += GJT) Dt[e] = Ds[(e % GB) * GB + e / GB];
    __syncthreads();
    // (c) new pivot row entries of column j: Pn_j = D^-1 A_{K, j}
    const int j = t;
    const bool jcol = j < q;
    double pn[GB];
#pragma unroll
    for (int r = 0; r < GB; ++r) pn[r] = 0.0;
    if (jcol) {
      for (int k = 0; k < GB; ++k) {
        const double a = M[(int64_t)(k0 + k) * q + j];
        const double2* dk = reinterpret_cast<const double2*>(Dt + k * GB);
#pragma unroll
        for (int r = 0; r < GB / 2; ++r) {
          const double2 d = dk[r];
          pn[2 * r] = fma(d.x, a, pn[2 * r]);
          pn[2 * r + 1] = fma(d.y, a, pn[2 * r + 1]);
        }
      }
    }
    __syncthreads();  // every column read its pivot-row entries
    if (jcol) {
      const bool jK = j >= k0 && j < k0 + GB;
      for (int i = 0; i < q; ++i) {
        if (i == k0) {  // pivot rows last
          i += GB - 1;
          continue;
        }
        const double2* ci = reinterpret_cast<const double2*>(Cold + i * GB);
        double x;
        if (jK) {  // pivot columns: -Cold_i D^-1
          double s = 0.0;
          for (int k = 0; k < GB; ++k) s = fma(Cold[i * GB + k], Ds[k * GB + (j - k0)], s);
          x = -s;
        } else {  // trailing update
          double s0 = M[(int64_t)i * q + j], s1 = 0.0;
#pragma unroll
          for (int k = 0; k < GB / 2; ++k) {
            const double2 c2 = ci[k];
            s0 = fma(-c2.x, pn[2 * k], s0);
            s1 = fma(-c2.y, pn[2 * k + 1], s1);
          }
          x = s0 + s1;
        }
        M[(int64_t)i * q + j] = x;
      }
      // pivot rows: D^-1 on the pivot block, Pn elsewhere
#pragma unroll
      for (int k = 0; k < GB; ++k)
        M[(int64_t)(k0 + k) * q + j] = jK ? Ds[k * GB + (j - k0)] : pn[k];
    }
    __syncthreads();
  }
  for (int e = t; e < q * q; e += GJT) {
    const int i = e / q, jj = e % q;
    if (i < jj) {
      const double s = 0.5 * (M[i * q + jj] + M[jj * q + i]);
      M[i * q + jj] = s;
      M[jj * q + i] = s;
    }
  }
  __syncthreads();
}

}  // namespace tmg
