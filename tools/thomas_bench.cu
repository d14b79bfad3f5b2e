// Microbenchmark of the fine block solve (diagnostics, not part of the
// library): k_update's thread layout, shared memory and TMA ring over 4096
// bricks, timed in three modes to separate HBM streaming from the solve's
// own latency:
//   0  real: each brick's 8 G planes (forward + backward sweep)
//   1  L2:   every plane load reads brick 0 / plane 0 (L2-resident)
//   2  copy: ring only (loads issued and awaited, no mat-vec work)
// plus a persistent variant of mode 0 (k_bench_persist: 148 x 3 / 4 CTAs,
// bricks strided, with and without the TMA ring carried across bricks).
// argv[1] = number of bricks (default 4096 = 128^3 cells; 32768 for a
// steady-state figure). -DTMG_MV_ROWS / -DTMG_DIAG_PACK / -DTMG_L2_AHEAD /
// -DTMG_G_HINTS select the variants measured in DESIGN.md §4.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        --expt-relaxed-constexpr -I paper_2410_06850_b200/csrc tools/thomas_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "smoother.cuh"

using namespace tmg;

constexpr int CB = 8;
// -DBENCH_CTAS=5 -DBENCH_TZ_GLOBAL=1 (with -DTMG_DIAG_PACK=1): the shared-memory
// budget of five CTAs per SM -- T_z read through a global pointer instead of
// the 4 KB shared array
#ifndef BENCH_CTAS
#define BENCH_CTAS 4
#endif
#ifndef BENCH_TZ_GLOBAL
#define BENCH_TZ_GLOBAL 0
#endif
__device__ double g_tz[CB * CB * CB];

template <int MODE>
__global__ void __launch_bounds__(Thomas<CB>::NT, BENCH_CTAS) k_bench(const double* __restrict__ Gf,
                                                            const double* __restrict__ tin,
                                                            double* xout) {
  constexpr int C = CB * CB * CB, NT = Thomas<CB>::NT;
  extern __shared__ __align__(128) unsigned char smraw[];
  struct Sm {
    double slots[kSlots][Thomas<CB>::PLANE];
    ThomasSmem<CB> th;
    double tv[C];
#if !BENCH_TZ_GLOBAL
    double tz[C];
#endif
  };
  Sm& sm = *reinterpret_cast<Sm*>(smraw);
#if BENCH_TZ_GLOBAL
  const double* tzp = g_tz;
#else
  double* tzp = sm.tz;
#endif
  const int b = blockIdx.x;
  const double* G = Gf + (MODE == 1 ? 0 : (size_t)b * Thomas<CB>::PER_BRICK);
  sm.th.slots = sm.slots;
  thomas_init<CB>(sm.th);
  __syncthreads();
  thomas_prefetch<CB>(sm.th, G);
  for (int c = threadIdx.x; c < C; c += NT) {
    sm.tv[c] = tin[(size_t)b * C + c];
#if !BENCH_TZ_GLOBAL
    sm.tz[c] = c >= CB * CB ? -0.1 : 0.0;
#endif
  }
  if (MODE == 2) {
    // stream the same 15 plane loads through the ring, no compute
    const bool waiter = threadIdx.x >= (int)blockDim.x - 32;
    const bool issuer = threadIdx.x == (int)blockDim.x - 32;
    for (int n = 0; n < Thomas<CB>::NL; ++n) {
      const int slot = n % kSlots;
      if (waiter) mbar_wait(&sm.th.bars[slot], (uint32_t)((n / kSlots) & 1));
      __syncthreads();
      if (issuer && n + kSlots < Thomas<CB>::NL) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&sm.th.bars[slot], Thomas<CB>::PLANE * sizeof(double));
        bulk_g2s(sm.slots[slot], G + (size_t)Thomas<CB>::plane_of(n + kSlots) * Thomas<CB>::PLANE,
                 Thomas<CB>::PLANE * sizeof(double), &sm.th.bars[slot]);
      }
      __syncthreads();
    }
  } else {
    thomas_solve<CB>(sm.th, G, sm.tv, tzp, sm.tv);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += NT) xout[(size_t)b * C + c] = sm.tv[c];
}

// Persistent variant of mode 0: one CTA per resident slot, bricks strided over
// the grid, the TMA ring carried across bricks (the next brick's first planes
// are requested while this brick's last planes are consumed).
__global__ void __launch_bounds__(Thomas<CB>::NT, 4) k_bench_persist(const double* __restrict__ Gf,
                                                                    const double* __restrict__ tin,
                                                                    double* xout, int nb, int chain) {
  constexpr int C = CB * CB * CB, NT = Thomas<CB>::NT;
  extern __shared__ __align__(128) unsigned char smraw[];
  struct Sm {
    double slots[kSlots][Thomas<CB>::PLANE];
    ThomasSmem<CB> th;
    double tv[C];
    double tz[C];
  };
  Sm& sm = *reinterpret_cast<Sm*>(smraw);
  sm.th.slots = sm.slots;
  thomas_init<CB>(sm.th);
  __syncthreads();
  uint32_t m = 0;
  int b = blockIdx.x;
  if (b < nb) thomas_prefetch<CB>(sm.th, Gf + (size_t)b * Thomas<CB>::PER_BRICK, 0);
  for (; b < nb; b += gridDim.x) {
    const double* G = Gf + (size_t)b * Thomas<CB>::PER_BRICK;
    const int bn = b + (int)gridDim.x;
    const double* Gn = bn < nb ? Gf + (size_t)bn * Thomas<CB>::PER_BRICK : nullptr;
    if (!chain && b != (int)blockIdx.x) thomas_prefetch<CB>(sm.th, G, m);
    for (int c = threadIdx.x; c < C; c += NT) {
      sm.tv[c] = tin[(size_t)b * C + c];
      sm.tz[c] = c >= CB * CB ? -0.1 : 0.0;
    }
    thomas_solve<CB>(sm.th, G, sm.tv, sm.tz, sm.tv, 1.0, m, chain ? Gn : nullptr);
    m += Thomas<CB>::NL;
    for (int c = threadIdx.x; c < C; c += NT) xout[(size_t)b * C + c] = sm.tv[c];
    __syncthreads();
  }
}

float run_persist(const double* G, const double* t, double* x, int nb, size_t smem, int grid, int chain) {
  cudaFuncSetAttribute(k_bench_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  for (int w = 0; w < 3; ++w) k_bench_persist<<<grid, Thomas<CB>::NT, smem>>>(G, t, x, nb, chain);
  cudaEventRecord(a);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) k_bench_persist<<<grid, Thomas<CB>::NT, smem>>>(G, t, x, nb, chain);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, e);
  return 1e3f * ms / reps;
}

template <int MODE>
float run(const double* G, const double* t, double* x, int nb, size_t smem) {
  cudaFuncSetAttribute(k_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  for (int w = 0; w < 3; ++w) k_bench<MODE><<<nb, Thomas<CB>::NT, smem>>>(G, t, x);
  cudaEventRecord(a);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) k_bench<MODE><<<nb, Thomas<CB>::NT, smem>>>(G, t, x);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, e);
  return 1e3f * ms / reps;
}

__global__ void k_dirty(double* buf, size_t n, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    buf[i] = v + (double)i;
}

// time k_bench<0> right after a kernel that leaves `mb` MB of dirty lines
float run_after_dirty(const double* G, const double* t, double* x, int nb, size_t smem, double* buf,
                      size_t mb) {
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  float tot = 0.f;
  const int reps = 20;
  for (int i = 0; i < reps + 3; ++i) {
    if (mb) k_dirty<<<148 * 8, 256>>>(buf, mb << 17, (double)i);
    cudaEventRecord(a);
    k_bench<0><<<nb, Thomas<CB>::NT, smem>>>(G, t, x);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, e);
    if (i >= 3) tot += ms;
  }
  return 1e3f * tot / reps;
}

int main(int argc, char** argv) {
  const int nb = argc > 1 ? atoi(argv[1]) : 4096;  // bricks (4096 = 128^3 cells)
  const size_t per = Thomas<CB>::PER_BRICK, C = CB * CB * CB;
  std::vector<double> hg(per * nb), ht(C * nb);
  for (size_t i = 0; i < hg.size(); ++i) hg[i] = 1e-3 * (double)((i * 2654435761u) % 1000) / 1000.0;
  for (size_t i = 0; i < ht.size(); ++i) ht[i] = 1.0;
  double *G, *t, *x;
  cudaMalloc(&G, sizeof(double) * hg.size());
  cudaMalloc(&t, sizeof(double) * ht.size());
  cudaMalloc(&x, sizeof(double) * ht.size());
  cudaMemcpy(G, hg.data(), sizeof(double) * hg.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(t, ht.data(), sizeof(double) * ht.size(), cudaMemcpyHostToDevice);
  const size_t smem = sizeof(double) * (kSlots * Thomas<CB>::PLANE + (BENCH_TZ_GLOBAL ? 1 : 2) * C) + sizeof(ThomasSmem<CB>) + 256;
  {
    std::vector<double> htz(C);
    for (size_t c = 0; c < C; ++c) htz[c] = c >= CB * CB ? -0.1 : 0.0;
    cudaMemcpyToSymbol(g_tz, htz.data(), sizeof(double) * C);
  }
  const double gb = (double)sizeof(double) * per * nb / 1e9;
  const float t0 = run<0>(G, t, x, nb, smem), t1 = run<1>(G, t, x, nb, smem), t2 = run<2>(G, t, x, nb, smem);
  printf("threads %d smem %zu KB  G %.0f MB\n", Thomas<CB>::NT, smem >> 10, gb * 1e3);
  printf("real   %7.1f us  (%.0f GB/s of G)\n", t0, gb / (t0 * 1e-6));
  printf("L2     %7.1f us\n", t1);
  printf("copy   %7.1f us  (%.0f GB/s of G)\n", t2, gb / (t2 * 1e-6));
#if !BENCH_TZ_GLOBAL
  {
    // reference result of the one-CTA-per-brick kernel, then the persistent ones
    std::vector<double> x0(C * nb), x1(C * nb);
    k_bench<0><<<nb, Thomas<CB>::NT, smem>>>(G, t, x);
    cudaMemcpy(x0.data(), x, sizeof(double) * x0.size(), cudaMemcpyDeviceToHost);
    for (int chain = 0; chain < 2; ++chain)
      for (int per_sm : {3, 4}) {
        const float tp = run_persist(G, t, x, nb, smem, 148 * per_sm, chain);
        cudaMemcpy(x1.data(), x, sizeof(double) * x1.size(), cudaMemcpyDeviceToHost);
        size_t bad = 0;
        for (size_t i = 0; i < x0.size(); ++i) bad += x0[i] != x1[i];
        printf("persist chain=%d grid=148x%d  %7.1f us  (%.0f GB/s of G)  mismatches %zu\n", chain, per_sm, tp,
               gb / (tp * 1e-6), bad);
      }
  }
#endif
  double* buf;
  cudaMalloc(&buf, (size_t)512 << 20);
  for (size_t mb : {0, 32, 64, 128, 256})
    printf("after %3zu MB dirty: real %7.1f us\n", mb, run_after_dirty(G, t, x, nb, smem, buf, mb));
  cudaError_t err = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(err));
  return 0;
}
