// Microbenchmark (diagnostics, not part of the library): two bricks per CTA
// in lock-step (one pair of barriers per plane step for both bricks, the
// mat-vecs of the two bricks interleaved per thread: ILP 2, the tree sums of
// both bricks on 128 threads) against one brick per CTA (smoother.cuh).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        --expt-relaxed-constexpr -I paper_2410_06850_b200/csrc tools/thomas_pair_bench.cu
#include <cmath>
#include <cstdio>
#include <vector>

#include "smoother.cuh"

using namespace tmg;
constexpr int CB = 8, P = 64, C = 512;
using TH = Thomas<CB>;

struct PairSmem {
  double slots[2][kSlots][TH::PLANE];
  ThomasSmem<CB> th[2];
  double tv[2][C];
  double tz[2][C];
};

__device__ __forceinline__ void pair_solve(PairSmem& sm, const double* G0, const double* G1) {
  const int tid = threadIdx.x;
  const MvRole<CB> m = mv_role<CB>();
  const bool waiter = tid >= (int)blockDim.x - 32, issuer = tid == (int)blockDim.x - 32;
  const double* G[2] = {G0, G1};
  if (waiter) {
    mbar_wait(&sm.th[0].bars[0], 0);
    mbar_wait(&sm.th[1].bars[0], 0);
  }
  if (tid < 2 * P) sm.th[tid / P].w2[0][tid % P] = sm.tv[tid / P][tid % P];
  __syncthreads();
#pragma unroll 1
  for (int n = 0; n < TH::NL; ++n) {
    const int slot = n % kSlots;
    mv_partials<CB>(sm.th[0], sm.slots[0][slot], sm.th[0].w2[n & 1], m);
    mv_partials<CB>(sm.th[1], sm.slots[1][slot], sm.th[1].w2[n & 1], m);
    __syncthreads();
    if (issuer && n + kSlots < TH::NL) {
      fence_proxy_async_smem();
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        mbar_arrive_expect_tx(&sm.th[b].bars[slot], TH::PLANE * sizeof(double));
        bulk_g2s(sm.slots[b][slot], G[b] + (size_t)TH::plane_of(n + kSlots) * TH::PLANE,
                 TH::PLANE * sizeof(double), &sm.th[b].bars[slot]);
      }
    }
    if (tid < 2 * P) {
      const int b = tid / P, row = tid % P;
      ThomasSmem<CB>& th = sm.th[b];
      double* t = sm.tv[b];
      const double* tz = sm.tz[b];
      double pr[TH::NBK];
#pragma unroll
      for (int s = 0; s < TH::NBK; ++s) pr[s] = th.part[s][row];
#pragma unroll
      for (int w = 1; w < TH::NBK; w *= 2)
#pragma unroll
        for (int s = 0; s + w < TH::NBK; s += 2 * w) pr[s] += pr[s + w];
      const double acc = pr[0];
      double* wn = th.w2[(n + 1) & 1];
      if (n < CB) {
        const int l = n * P + row;
        t[l] = acc;
        if (n + 1 < CB) wn[row] = fma(tz[l + P], acc, t[l + P]);
        else wn[row] = -tz[l] * acc;
      } else {
        const int k = TH::plane_of(n), l = k * P + row;
        const double xv = t[l] - acc;
        t[l] = xv;
        if (k > 0) wn[row] = -tz[l] * xv;
      }
    }
    if (waiter && n + 1 < TH::NL) {
      mbar_wait(&sm.th[0].bars[(n + 1) % kSlots], (uint32_t)(((n + 1) / kSlots) & 1));
      mbar_wait(&sm.th[1].bars[(n + 1) % kSlots], (uint32_t)(((n + 1) / kSlots) & 1));
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(TH::NT, 2) k_pair(const double* __restrict__ Gf, const double* __restrict__ tin,
                                                   double* xout) {
  extern __shared__ __align__(128) unsigned char smraw[];
  PairSmem& sm = *reinterpret_cast<PairSmem*>(smraw);
  const int b0 = 2 * blockIdx.x;
  for (int b = 0; b < 2; ++b) {
    sm.th[b].slots = sm.slots[b];
    thomas_init<CB>(sm.th[b]);
  }
  __syncthreads();
  for (int b = 0; b < 2; ++b) thomas_prefetch<CB>(sm.th[b], Gf + (size_t)(b0 + b) * TH::PER_BRICK);
  for (int c = threadIdx.x; c < 2 * C; c += blockDim.x) {
    sm.tv[c / C][c % C] = tin[(size_t)b0 * C + c];
    sm.tz[c / C][c % C] = (c % C) >= P ? -0.1 : 0.0;
  }
  __syncthreads();
  pair_solve(sm, Gf + (size_t)b0 * TH::PER_BRICK, Gf + (size_t)(b0 + 1) * TH::PER_BRICK);
  for (int c = threadIdx.x; c < 2 * C; c += blockDim.x) xout[(size_t)b0 * C + c] = sm.tv[c / C][c % C];
}

__global__ void __launch_bounds__(TH::NT, 4) k_one(const double* __restrict__ Gf, const double* __restrict__ tin,
                                                  double* xout) {
  extern __shared__ __align__(128) unsigned char smraw[];
  struct Sm {
    double slots[kSlots][TH::PLANE];
    ThomasSmem<CB> th;
    double tv[C];
    double tz[C];
  };
  Sm& sm = *reinterpret_cast<Sm*>(smraw);
  const int b = blockIdx.x;
  const double* G = Gf + (size_t)b * TH::PER_BRICK;
  sm.th.slots = sm.slots;
  thomas_init<CB>(sm.th);
  __syncthreads();
  thomas_prefetch<CB>(sm.th, G);
  for (int c = threadIdx.x; c < C; c += TH::NT) {
    sm.tv[c] = tin[(size_t)b * C + c];
    sm.tz[c] = c >= P ? -0.1 : 0.0;
  }
  __syncthreads();
  thomas_solve<CB>(sm.th, G, sm.tv, sm.tz, sm.tv);
  for (int c = threadIdx.x; c < C; c += TH::NT) xout[(size_t)b * C + c] = sm.tv[c];
}

template <typename K>
float timeit(K kern, int grid, const double* G, const double* t, double* x, size_t smem) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  for (int w = 0; w < 3; ++w) kern<<<grid, TH::NT, smem>>>(G, t, x);
  cudaEventRecord(a);
  for (int r = 0; r < 20; ++r) kern<<<grid, TH::NT, smem>>>(G, t, x);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, e);
  return 1e3f * ms / 20;
}

int main() {
  const int nb = 4096;
  std::vector<double> hg(TH::PER_BRICK * (size_t)nb), ht((size_t)C * nb);
  for (size_t i = 0; i < hg.size(); ++i) hg[i] = 1e-3 * (double)((i * 2654435761u) % 1000) / 1000.0;
  for (size_t i = 0; i < ht.size(); ++i) ht[i] = 1.0 + 1e-3 * (double)(i % 97);
  double *G, *t, *x;
  cudaMalloc(&G, sizeof(double) * hg.size());
  cudaMalloc(&t, sizeof(double) * ht.size());
  cudaMalloc(&x, sizeof(double) * ht.size());
  cudaMemcpy(G, hg.data(), sizeof(double) * hg.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(t, ht.data(), sizeof(double) * ht.size(), cudaMemcpyHostToDevice);
  std::vector<double> x0(ht.size()), x1(ht.size());
  const size_t s1 = sizeof(double) * (kSlots * TH::PLANE + 2 * C) + sizeof(ThomasSmem<CB>) + 256;
  const float t1 = timeit(k_one, nb, G, t, x, s1);
  cudaMemcpy(x0.data(), x, sizeof(double) * x0.size(), cudaMemcpyDeviceToHost);
  const float t2 = timeit(k_pair, nb / 2, G, t, x, sizeof(PairSmem) + 256);
  cudaMemcpy(x1.data(), x, sizeof(double) * x1.size(), cudaMemcpyDeviceToHost);
  double md = 0.0;
  for (size_t i = 0; i < x0.size(); ++i) md = fmax(md, fabs(x0[i] - x1[i]) / (fabs(x0[i]) + 1e-30));
  printf("one brick / CTA (4 per SM): %7.1f us\npair / CTA (2 per SM):      %7.1f us   max rel diff %.2e   smem %zu KB\n%s\n",
         t1, t2, md, (sizeof(PairSmem) + 256) >> 10, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
