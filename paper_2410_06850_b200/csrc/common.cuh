// Shared device-side definitions for the B200 PCG + multiscale-MG hot path.
//
// Layout in HBM ("brick" layout): every fine-grid vector is
// stored coarse-cell by coarse-cell. Brick b = bi + nbx*(bj + nby*bk) is the
// reference's coarse_index (proj/core/include/topmg/grid.hpp:107-109); inside a
// brick cells are x-fastest, li + CB*(lj + CB*lk), the order of
// HierarchicalGrid::cells_of_coarse (grid.cpp:169-173) and therefore of the
// columns of one R_c row block (coarse_space.cpp:328-337). Storage index =
// b*CB^3 + l. A brick is one CTA's tile: contiguous 4 KiB per vector at CB=8.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tmg {

constexpr int kMaxPatches = 16;

struct Patch {
  int face;
  double u0, v0, u1, v1, value;
};

// Everything a kernel needs to know about the grid, passed by value.
struct GridParams {
  int64_t nx, ny, nz;        // fine cells per axis
  int64_t nbx, nby, nbz;     // bricks (= coarse cells) per axis
  int64_t nb;                // number of bricks
  int64_t ncx, ncy, ncz;     // cc elements per axis
  int64_t ncc;               // number of cc elements
  int sd;                    // coarse cells per cc element per axis
  int lc;                    // L_c
  int lcc;                   // L_cc
  double cpl[3];             // area/h per axis (fvm.cpp:23-26)
  double vol;                // cell volume
  double hx, hy, hz;
  // Partition: this context owns bricks [b0, b0 + nbo) and
  // cc elements [e0, e0 + neo) -- whole z-layers of cc elements. Kernels index
  // global bricks/elements; device arrays are windows of the global arrays
  // (own layers plus one ghost brick layer per neighbouring slab). mst is the
  // stored cells per fine vector (component stride of coef).
  int64_t b0, nbo, e0, neo, mst;
  int dist;  // 1: reductions finish in k_finalize after the cross-slab sum
  // Brick (= coarse cell) extent in fine cells per axis: the reference's
  // HierarchicalGrid::cells_per_c (grid.hpp:100). The templated kernels are
  // built for cubic 4^3 / 8^3 bricks; any other shape runs the generic
  // kernels of generic.cu (cb = 0 at the launchers).
  int bx, by, bz;
};

// cells per brick
__host__ __device__ __forceinline__ int64_t brick_cells(const GridParams& g) {
  return (int64_t)g.bx * g.by * g.bz;
}

// ------------------------------------------ programmatic dependent launch
// Iteration kernels are launched with PDL (launch_pdl): each CTA lets the next
// kernel in the stream be scheduled as soon as it starts (pdl_trigger), so the
// next kernel's CTAs fill SMs freed by this kernel's tail and run their
// prologue (barrier init, constant-data TMA/L2 prefetch) early; pdl_wait()
// blocks until the previous kernel has completed and its writes are visible,
// and must precede the first read of anything that kernel produced.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// L2 prefetch of constant data (no shared-memory side effects)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ double face_t(double kl, double kr) {
  // fvm.cpp:9-14: 2*kl*kr/(kl+kr) — no contraction, bitwise with the reference
  return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, kl), kr), __dadd_rn(kl, kr));
}

// ---------------------------------------------------------------- reductions

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  // deterministic tree: warp xor-shuffle then fixed-order smem tree
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double s = lane < NW ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[0] = s;
  }
  __syncthreads();
  const double out = red[0];
  __syncthreads();
  return out;
}

// Sum K values per thread across the block. out[k] valid in all threads.
template <int NT, int K>
__device__ __forceinline__ void block_sum_k(double (&v)[K], double* red /* >= K*NT/32 */) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    v[k] = x;
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) red[k * NW + wid] = v[k];
  }
  __syncthreads();
  // K*NW partial sums; thread t < K reduces row t in fixed order
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += red[threadIdx.x * NW + w];
    red[K * NW + threadIdx.x] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = red[K * NW + k];
  __syncthreads();
}

// K-value variant of grid_reduce_last: partials laid out [K][gridDim.x].
template <int K>
__device__ __forceinline__ bool grid_reduce_last_k(const double (&partial)[K], double* partials,
                                                   unsigned int* ticket, double (&total)[K],
                                                   int* smem_flag, double* red) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) partials[(size_t)k * gridDim.x + blockIdx.x] = partial[k];
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    *smem_flag = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!*smem_flag) return false;
  __threadfence();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
    for (unsigned int i = threadIdx.x; i < gridDim.x; i += blockDim.x)
      s += ((volatile double*)partials)[(size_t)k * gridDim.x + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[k * 32 + wid] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += red[k * 32 + w];
      red[K * 32 + k] = t;
    }
    *ticket = 0u;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) total[k] = red[K * 32 + k];
  return true;
}

}  // namespace tmg
