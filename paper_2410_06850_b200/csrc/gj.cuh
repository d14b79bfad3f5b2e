// Register-resident Gauss-Jordan sweep inversion of a P x P SPD matrix by one
// CTA of NTF threads (set-up kernels: smoother factors, A_cc pivot blocks).
// Warp w owns columns [CW*w, CW*w + CW) of all P rows, lane l the rows
// l + 32 h (h < RH): per pivot the generic update is one multiply and one FMA
// per entry, and the pivot column's special case is warp-uniform (one warp).
// Pivot row, pivot column and 1/pivot go through shared memory
// (double-buffered, one barrier per pivot). No pivoting: the pivots are the
// LDL^T pivots in natural order; pmin / pmax collect the ones this thread saw.
#pragma once
#include "common.cuh"

namespace tmg {

template <int P, int NTF>
struct GjLayout {
  static constexpr int NW = NTF / 32;
  static constexpr int CW = P / NW;                 // columns per warp
  static constexpr int RH = P > 32 ? P / 32 : 1;    // rows per lane
  static_assert(CW % 2 == 0 && CW * NW == P && (P >= 32 ? RH * 32 == P : true), "layout");
};

template <int P>
struct GjSmem {
  alignas(16) double rowbuf[2][P];
  double colbuf[2][P];
  double invbuf[2];
};

template <int P, int NTF>
__device__ __forceinline__ void gj_invert(double (&v)[GjLayout<P, NTF>::RH][GjLayout<P, NTF>::CW],
                                          GjSmem<P>& sm, double& pmin, double& pmax,
                                          double* piv_out = nullptr) {
  constexpr int CW = GjLayout<P, NTF>::CW, RH = GjLayout<P, NTF>::RH, NW = GjLayout<P, NTF>::NW;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, c0 = CW * wid;
  const bool lane_active = lane < P;
  // Pivots in groups of CW: group wp lies in warp wp's columns, so inside a
  // group the pivot's column index j is a compile-time constant (no selects
  // over the register row; the pivot row's h = p / 32 is the only runtime
  // index).
#pragma unroll 1
  for (int wp = 0; wp < NW; ++wp) {
    const bool colw = wid == wp;  // this warp owns the group's columns
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const int p = wp * CW + j, b = p & 1, pr = p & 31, ph = p >> 5;
      if (lane_active) {
        if (lane == pr) {
#pragma unroll
          for (int h = 0; h < RH; ++h)
            if (h == ph) {
#pragma unroll
              for (int q = 0; q < CW; q += 2)
                *reinterpret_cast<double2*>(&sm.rowbuf[b][c0 + q]) =
                    make_double2(v[h][q], v[h][q + 1]);
            }
        }
        if (colw) {
#pragma unroll
          for (int h = 0; h < RH; ++h) {
            const double cv = v[h][j];
            sm.colbuf[b][lane + 32 * h] = cv;
            if (lane == pr && h == ph) {
              sm.invbuf[b] = 1.0 / cv;
              pmin = fmin(pmin, cv);
              pmax = fmax(pmax, fabs(cv));
              if (piv_out) piv_out[p] = cv;
            }
          }
        }
      }
      __syncthreads();
      if (lane_active) {
        const double inv = sm.invbuf[b];
        double rji[CW];
#pragma unroll
        for (int q = 0; q < CW; q += 2) {
          const double2 r2 = *reinterpret_cast<const double2*>(&sm.rowbuf[b][c0 + q]);
          rji[q] = r2.x * inv;
          rji[q + 1] = r2.y * inv;
        }
#pragma unroll
        for (int h = 0; h < RH; ++h) {
          const double cvi = sm.colbuf[b][lane + 32 * h];
#pragma unroll
          for (int q = 0; q < CW; ++q) v[h][q] = fma(-cvi, rji[q], v[h][q]);
          if (colw) v[h][j] = -cvi * inv;  // pivot column: -c_i / pivot
          if (lane == pr && h == ph) {     // pivot row: r_j / pivot, pivot: 1 / pivot
#pragma unroll
            for (int q = 0; q < CW; ++q) v[h][q] = rji[q];
            if (colw) v[h][j] = inv;
          }
        }
      }
    }
  }
}

}  // namespace tmg
