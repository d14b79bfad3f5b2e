// Microbenchmark (diagnostics, not part of the library): fine block solve with
// one thread per plane row (P = 64 threads per brick) over a packed
// lower-triangle plane layout, against the 288-thread block-row solve of
// smoother.cuh. Thread i forms y_i = sum_{j<=i} L[i][j] w_j (its packed row,
// address tri(i) + j) + sum_{j>i} L[j][i] w_j (its column, address tri(j) + i):
// both are register base + immediate, so the mat-vec needs no shuffles, no
// partial-sum arrays and one barrier per plane step.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        --expt-relaxed-constexpr -I paper_2410_06850_b200/csrc tools/thomas_v2_bench.cu
#include <cmath>
#include <cstdio>
#include <vector>

#include "smoother.cuh"

using namespace tmg;

constexpr int CB = 8;
using TH = Thomas<CB>;
constexpr int P = CB * CB;
constexpr int PL2 = P * (P + 1) / 2;  // packed plane (2080 doubles)
constexpr int NL = 2 * CB - 1;
__host__ __device__ constexpr int tri(int i) { return i * (i + 1) / 2; }

template <int NS>
struct V2Smem {
  alignas(16) double slots[NS][PL2];
  alignas(16) double w2[2][P];
  double tv[CB * CB * CB];
  double tz[CB * CB * CB];
  uint64_t bars[NS];
};
__device__ __forceinline__ int plane_at(int n) { return n < CB ? n : 2 * CB - 2 - n; }

template <int J0, int J1>
__device__ __forceinline__ void mv_lower(const double* __restrict__ Lrow, const double* w, double (&a)[4]) {
#pragma unroll
  for (int j = J0; j < J1; j += 2) {
    const double2 wv = *reinterpret_cast<const double2*>(w + j);
    a[j & 3] = fma(Lrow[j], wv.x, a[j & 3]);
    a[(j + 1) & 3] = fma(Lrow[j + 1], wv.y, a[(j + 1) & 3]);
  }
}
template <int J0, int J1>
__device__ __forceinline__ void mv_upper(const double* __restrict__ Lcol, const double* w, double (&a)[4]) {
#pragma unroll
  for (int j = J0; j < J1; j += 2) {
    const double2 wv = *reinterpret_cast<const double2*>(w + j);
    a[j & 3] = fma(Lcol[tri(j)], wv.x, a[j & 3]);
    a[(j + 1) & 3] = fma(Lcol[tri(j + 1)], wv.y, a[(j + 1) & 3]);
  }
}
template <int J0, int J1>
__device__ __forceinline__ void mv_mixed(const double* __restrict__ Lrow, const double* __restrict__ Lcol,
                                         const double* w, int i, double (&a)[4]) {
#pragma unroll
  for (int j = J0; j < J1; j += 2) {
    const double2 wv = *reinterpret_cast<const double2*>(w + j);
    const double g0 = j <= i ? Lrow[j] : Lcol[tri(j)];
    const double g1 = j + 1 <= i ? Lrow[j + 1] : Lcol[tri(j + 1)];
    a[j & 3] = fma(g0, wv.x, a[j & 3]);
    a[(j + 1) & 3] = fma(g1, wv.y, a[(j + 1) & 3]);
  }
}

template <int NS, int PF>
__device__ __forceinline__ void solve_v2(V2Smem<NS>& sm, const double* __restrict__ G, double* t, const double* tz) {
  const int i = threadIdx.x;
#pragma unroll 1
  for (int n = 0; n < NL; ++n) {
    const int slot = n % NS;
    if (PF == 2 && i == 0 && n + NS + 1 < CB)
      prefetch_l2(G + (size_t)(n + NS + 1) * PL2, PL2 * sizeof(double));
    mbar_wait(&sm.bars[slot], (uint32_t)((n / NS) & 1));
    const double* L = sm.slots[slot];
    const double* w = sm.w2[n & 1];
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    if (i < 32) {
      mv_mixed<0, 32>(L + tri(i), L + i, w, i, a);
      mv_upper<32, 64>(L + i, w, a);
    } else {
      mv_lower<0, 32>(L + tri(i), w, a);
      mv_mixed<32, 64>(L + tri(i), L + i, w, i, a);
    }
    const double acc = (a[0] + a[1]) + (a[2] + a[3]);
    double* wn = sm.w2[(n + 1) & 1];
    if (n < CB) {
      const int l = n * P + i;
      t[l] = acc;  // u_n over the consumed t_n
      if (n + 1 < CB) wn[i] = fma(tz[l + P], acc, t[l + P]);
      else wn[i] = -tz[l] * acc;
    } else {
      const int k = 2 * CB - 2 - n;
      const int l = k * P + i;
      const double xv = t[l] - acc;
      t[l] = xv;
      if (k > 0) wn[i] = -tz[l] * xv;
    }
    __syncthreads();
    if (i == 0 && n + NS < NL) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&sm.bars[slot], PL2 * sizeof(double));
      const int pn = plane_at(n + NS);
      bulk_g2s(sm.slots[slot], G + (size_t)pn * PL2, PL2 * sizeof(double), &sm.bars[slot]);
    }
  }
}

template <int MINB, int NS, int PF>
__global__ void __launch_bounds__(P, MINB) k_v2(const double* __restrict__ Gf, const double* __restrict__ tin,
                                               double* xout) {
  constexpr int C = CB * CB * CB;
  extern __shared__ __align__(128) unsigned char smraw[];
  V2Smem<NS>& sm = *reinterpret_cast<V2Smem<NS>*>(smraw);
  const int b = blockIdx.x;
  const double* G = Gf + (size_t)b * CB * PL2;
  if (threadIdx.x == 0) {
    for (int n = 0; n < NS; ++n) mbar_init(&sm.bars[n], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && PF == 1)
    for (int n = NS; n < CB; ++n) prefetch_l2(G + (size_t)n * PL2, PL2 * sizeof(double));
  if (threadIdx.x == 0)
    for (int n = 0; n < NS; ++n) {
      mbar_arrive_expect_tx(&sm.bars[n], PL2 * sizeof(double));
      bulk_g2s(sm.slots[n], G + (size_t)n * PL2, PL2 * sizeof(double), &sm.bars[n]);
    }
  for (int c = threadIdx.x; c < C; c += P) {
    sm.tv[c] = tin[(size_t)b * C + c];
    sm.tz[c] = c >= P ? -0.1 : 0.0;
  }
  if (threadIdx.x < P) sm.w2[0][threadIdx.x] = tin[(size_t)b * C + threadIdx.x];
  __syncthreads();
  solve_v2<NS, PF>(sm, G, sm.tv, sm.tz);
  for (int c = threadIdx.x; c < C; c += P) xout[(size_t)b * C + c] = sm.tv[c];
}

// reference: smoother.cuh's solve
__global__ void __launch_bounds__(TH::NT, 4) k_old(const double* __restrict__ Gf, const double* __restrict__ tin,
                                                  double* xout) {
  constexpr int C = CB * CB * CB, NT = TH::NT;
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
  for (int c = threadIdx.x; c < C; c += NT) {
    sm.tv[c] = tin[(size_t)b * C + c];
    sm.tz[c] = c >= P ? -0.1 : 0.0;
  }
  thomas_solve<CB>(sm.th, G, sm.tv, sm.tz, sm.tv);
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += NT) xout[(size_t)b * C + c] = sm.tv[c];
}

template <typename K>
float timeit(K kern, int threads, const double* G, const double* t, double* x, int nb, size_t smem) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  for (int w = 0; w < 3; ++w) kern<<<nb, threads, smem>>>(G, t, x);
  cudaEventRecord(a);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) kern<<<nb, threads, smem>>>(G, t, x);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, e);
  return 1e3f * ms / reps;
}

int main() {
  const int nb = 4096;
  const size_t C = CB * CB * CB;
  std::vector<double> gold(TH::PER_BRICK * (size_t)nb), gnew((size_t)CB * PL2 * nb), ht(C * nb);
  std::vector<double> full(P * P);
  unsigned long long s = 12345;
  auto rnd = [&]() { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return (double)(s >> 11) * 0x1.0p-53; };
  for (int b = 0; b < nb; ++b)
    for (int k = 0; k < CB; ++k) {
      for (int i = 0; i < P; ++i)
        for (int j = 0; j <= i; ++j) full[i * P + j] = full[j * P + i] = (i == j ? 0.05 : 0.0) + 1e-3 * rnd();
      double* po = &gold[((size_t)b * CB + k) * TH::PLANE];
      for (int blk = 0; blk < TH::NBLK; ++blk) {
        int I, J;
        const int v = blk;  // storage order of smoother.cuh (kBlockOrder8)
        static const unsigned char ord[36] = {44, 33, 41, 36, 60, 51, 59, 52, 17, 18, 25, 9, 26, 50, 63, 58, 24, 27,
                                              16, 0,  57, 62, 54, 49, 45, 8,  32, 40, 61, 56, 53, 48, 34, 43, 42, 35};
        I = ord[v] >> 3;
        J = ord[v] & 7;
        for (int r = 0; r < 8; ++r)
          for (int c = 0; c < 8; ++c) po[blk * 64 + swz(r, c)] = full[(8 * I + r) * P + 8 * J + c];
      }
      double* pn = &gnew[((size_t)b * CB + k) * PL2];
      for (int i = 0; i < P; ++i)
        for (int j = 0; j <= i; ++j) pn[tri(i) + j] = full[i * P + j];
    }
  for (size_t i = 0; i < ht.size(); ++i) ht[i] = 1.0 + 1e-3 * (double)(i % 97);
  double *Go, *Gn, *t, *x;
  cudaMalloc(&Go, sizeof(double) * gold.size());
  cudaMalloc(&Gn, sizeof(double) * gnew.size());
  cudaMalloc(&t, sizeof(double) * ht.size());
  cudaMalloc(&x, sizeof(double) * ht.size());
  cudaMemcpy(Go, gold.data(), sizeof(double) * gold.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(Gn, gnew.data(), sizeof(double) * gnew.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(t, ht.data(), sizeof(double) * ht.size(), cudaMemcpyHostToDevice);
  const size_t smem_old = sizeof(double) * (kSlots * TH::PLANE + 2 * C) + sizeof(ThomasSmem<CB>) + 256;
  const size_t smem2 = sizeof(V2Smem<2>) + 128, smem3 = sizeof(V2Smem<3>) + 128;
  std::vector<double> x0(C * nb), x1(C * nb);
  const float t0 = timeit(k_old, TH::NT, Go, t, x, nb, smem_old);
  cudaMemcpy(x0.data(), x, sizeof(double) * x0.size(), cudaMemcpyDeviceToHost);
  const double gbo = sizeof(double) * gold.size() / 1e9, gbn = sizeof(double) * gnew.size() / 1e9;
  printf("old 288-thread block rows: %7.1f us (%.0f GB/s of G, %.0f MB)\n", t0, gbo / (t0 * 1e-6), gbo * 1e3);
  auto rep = [&](const char* name, float tt) {
    cudaMemcpy(x1.data(), x, sizeof(double) * x1.size(), cudaMemcpyDeviceToHost);
    double md = 0.0;
    for (size_t i = 0; i < x0.size(); ++i) md = fmax(md, fabs(x0[i] - x1[i]) / (fabs(x0[i]) + 1e-30));
    printf("%-28s %7.1f us (%.0f GB/s of G)  max rel diff %.2e\n", name, tt, gbn / (tt * 1e-6), md);
  };
  rep("v2 ring2 minb5", timeit(k_v2<5, 2, 0>, P, Gn, t, x, nb, smem2));
  rep("v2 ring2 minb5 L2 all", timeit(k_v2<5, 2, 1>, P, Gn, t, x, nb, smem2));
  rep("v2 ring2 minb5 L2 rolling", timeit(k_v2<5, 2, 2>, P, Gn, t, x, nb, smem2));
  rep("v2 ring3 minb3", timeit(k_v2<3, 3, 0>, P, Gn, t, x, nb, smem3));
  rep("v2 ring3 minb3 L2 rolling", timeit(k_v2<3, 3, 2>, P, Gn, t, x, nb, smem3));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
