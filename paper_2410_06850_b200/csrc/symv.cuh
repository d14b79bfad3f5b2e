// Symmetric tiled GEMV of A_cc^-1 (north_star item 6), shared by the
// stand-alone kernel (dense.cu) and the fused coarse-level kernel (coarse.cu).
//
// A_cc^-1 is symmetric: only its lower block-triangle of 64 x 64 tiles is kept
// (tile (I, J <= I) at I(I+1)/2 + J, row-major, zero padded), halving the
// bytes streamed per V-cycle. Each CTA walks tiles blockIdx.x, +gridDim.x, ...;
// a tile's row products (contribution to y_I) and, off the diagonal, its
// column products (contribution to y_J) go to a partial buffer P[I][J][64];
// the nt partials of every output are summed afterwards in a fixed order
// (deterministic). Tiles arrive by TMA bulk copy into a kSymvSlots-deep ring.
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace tmg {

constexpr int TS = 64;
#ifndef TMG_SYMV_SLOTS
#define TMG_SYMV_SLOTS 2
#endif
constexpr int kSymvSlots = TMG_SYMV_SLOTS;
constexpr uint32_t kTileBytes = TS * TS * sizeof(double);

struct SymvSmem {
  uint64_t bars[kSymvSlots];
  double colp[4][TS];
};

// x is staged in shared memory up to this many unknowns; larger systems read
// it from global memory (L2-resident) tile by tile
constexpr int64_t kSymvStageMax = 12288;
__host__ __device__ inline bool symv_staged(int64_t n) { return n <= kSymvStageMax; }

// dynamic shared memory of a CTA that runs the GEMV: ring (+ all of x)
inline size_t symv_dyn_smem(int64_t n) {
  const int64_t nt = (n + TS - 1) / TS;
  return sizeof(double) * (size_t)(kSymvSlots * TS * TS + (symv_staged(n) ? nt * TS : 0));
}

// lower-triangle tile index -> (I, J <= I): closed-form triangular root,
// corrected by one step either way against rounding
__device__ __forceinline__ void symv_tile_ij(int64_t tile, int64_t& I, int64_t& J) {
  I = (int64_t)((sqrt(8.0 * (double)tile + 1.0) - 1.0) * 0.5);
  if (I * (I + 1) / 2 > tile) --I;
  if ((I + 1) * (I + 2) / 2 <= tile) ++I;
  J = tile - I * (I + 1) / 2;
}

// Barrier init and the first kSymvSlots tile loads (the tiles are constant,
// so this may run before the CTA waits for its input vector). Ends with a
// __syncthreads.
__device__ __forceinline__ void symv_begin(SymvSmem& ss, double* ring, const double* __restrict__ T,
                                           int64_t n) {
  const int64_t nt = (n + TS - 1) / TS, ntiles = nt * (nt + 1) / 2;
  if (threadIdx.x == 0) {
    for (int k = 0; k < kSymvSlots; ++k) mbar_init(&ss.bars[k], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < kSymvSlots; ++k) {
      const int64_t tile = blockIdx.x + k * (int64_t)gridDim.x;
      if (tile < ntiles) {
        mbar_arrive_expect_tx(&ss.bars[k], kTileBytes);
        bulk_g2s(ring + k * TS * TS, T + tile * TS * TS, kTileBytes, &ss.bars[k]);
      }
    }
}

// Wait for the loads symv_begin issued (CTA exiting without running the loop).
__device__ __forceinline__ void symv_drain(SymvSmem& ss, int64_t n) {
  const int64_t nt = (n + TS - 1) / TS, ntiles = nt * (nt + 1) / 2;
  if (threadIdx.x == 0)
    for (int k = 0; k < kSymvSlots; ++k)
      if (blockIdx.x + k * (int64_t)gridDim.x < ntiles) mbar_wait(&ss.bars[k], 0);
}

// Stage x (zero padded) and run this CTA's tiles. 256 threads.
__device__ __forceinline__ void symv_run(SymvSmem& ss, double* ring, double* xs,
                                         const double* __restrict__ T, int64_t n,
                                         const double* __restrict__ x, double* P) {
  const int64_t nt = (n + TS - 1) / TS, ntiles = nt * (nt + 1) / 2;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool staged = symv_staged(n);
  if (staged)
    for (int64_t k = t; k < nt * TS; k += blockDim.x) xs[k] = k < n ? __ldcg(x + k) : 0.0;
  // large systems: a per-tile copy of the two x segments (the last tile row
  // is zero padded past n)
  __shared__ double xseg[2][TS];
  __syncthreads();
  int64_t tile = blockIdx.x;
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int slot = it % kSymvSlots;
    int64_t I, J;
    symv_tile_ij(tile, I, J);
    const double* xi;
    const double* xj;
    if (staged) {
      xi = xs + I * TS;
      xj = xs + J * TS;
    } else {
      if (t < 2 * TS) {
        const int64_t k = (t < TS ? I : J) * TS + (t % TS);
        xseg[t / TS][t % TS] = k < n ? __ldcg(x + k) : 0.0;
      }
      xi = xseg[0];
      xj = xseg[1];
    }
    mbar_wait(&ss.bars[slot], (uint32_t)((it / kSymvSlots) & 1));
    __syncthreads();
    const double* A = ring + slot * TS * TS;
    // row products: warp w owns rows 8w..8w+7; lane l covers columns l, l+32
    {
      double pr[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double* row = A + (8 * warp + k) * TS;
        pr[k] = fma(row[lane], xj[lane], row[lane + 32] * xj[lane + 32]);
      }
      // reduce-scatter over 32 lanes: 8 -> 4 -> 2 -> 1 values, then 2 more folds
      const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
      double c4[4], c2[2];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        c4[k] = (b16 ? pr[k + 4] : pr[k]) + __shfl_xor_sync(0xffffffffu, b16 ? pr[k] : pr[k + 4], 16);
#pragma unroll
      for (int k = 0; k < 2; ++k)
        c2[k] = (b8 ? c4[k + 2] : c4[k]) + __shfl_xor_sync(0xffffffffu, b8 ? c4[k] : c4[k + 2], 8);
      double c1 = (b4 ? c2[1] : c2[0]) + __shfl_xor_sync(0xffffffffu, b4 ? c2[0] : c2[1], 4);
      c1 += __shfl_xor_sync(0xffffffffu, c1, 2);
      c1 += __shfl_xor_sync(0xffffffffu, c1, 1);
      // lane with bits (b16 b8 b4) holds row 8w + 4*b16 + 2*b8 + b4
      if ((lane & 3) == 0) {
        const int k = (b16 ? 4 : 0) + (b8 ? 2 : 0) + (b4 ? 1 : 0);
        P[(I * nt + J) * TS + 8 * warp + k] = c1;
      }
    }
    // column products (off-diagonal tiles): thread (group g, column c)
    if (I != J) {
      const int c = t & (TS - 1), gq = t >> 6;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int r = 0; r < 16; r += 2) {
        s0 = fma(A[(16 * gq + r) * TS + c], xi[16 * gq + r], s0);
        s1 = fma(A[(16 * gq + r + 1) * TS + c], xi[16 * gq + r + 1], s1);
      }
      ss.colp[gq][c] = s0 + s1;
    }
    __syncthreads();  // ring slot and xi/xj/colp consumed
    if (I != J && t < TS)
      P[(J * nt + I) * TS + t] = (ss.colp[0][t] + ss.colp[1][t]) + (ss.colp[2][t] + ss.colp[3][t]);
    if (t == 0 && tile + kSymvSlots * (int64_t)gridDim.x < ntiles) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&ss.bars[slot], kTileBytes);
      bulk_g2s(ring + slot * TS * TS, T + (tile + kSymvSlots * gridDim.x) * TS * TS, kTileBytes,
               &ss.bars[slot]);
    }
    __syncthreads();
  }
}

}  // namespace tmg
