// Microbenchmark (diagnostics, not part of the library): the fine block solve
// with the G planes read straight into registers (no shared-memory staging)
// against the TMA-ring solve of smoother.cuh. The plane data then crosses the
// SM's L1/shared data path once instead of twice (TMA write + LDS read).
//   tma      thomas_solve (smoother.cuh), swizzled layout
//   rd       register-direct, chunk-major layout, distance-1 register prefetch
//   rd+l2    the same plus cp.async.bulk.prefetch.L2 of the brick's planes at entry
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        --expt-relaxed-constexpr -I paper_2410_06850_b200/csrc tools/thomas_rd_bench.cu
#include <cmath>
#include <cstdio>
#include <vector>

#include "smoother.cuh"

using namespace tmg;

constexpr int CB = 8;
using TH = Thomas<CB>;

// chunk-major block layout: 16-byte chunk q of row r at chunk slot q*8 + r
__host__ __device__ constexpr int cm(int r, int c) { return ((c >> 1) * 8 + r) * 2 + (c & 1); }

__device__ __forceinline__ double2 ldg_na(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void load_row(double (&g)[8], const double* Gp, const MvRole<CB>& m) {
  const double* row = Gp + m.blk * 64 + 2 * m.r;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double2 v = ldg_na(row + 16 * q);
    g[2 * q] = v.x;
    g[2 * q + 1] = v.y;
  }
}

__device__ __forceinline__ void mv_partials_reg(ThomasSmem<CB>& sm, const double (&gv)[8], const double* w,
                                                const MvRole<CB>& m) {
  const bool off_diag = m.J < m.I;
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int c = 0; c < 8; c += 2) {
    const double2 wv = *reinterpret_cast<const double2*>(w + 8 * m.J + c);
    a0 = fma(gv[c], wv.x, a0);
    a1 = fma(gv[c + 1], wv.y, a1);
  }
  sm.part[m.J][8 * m.I + m.r] = a0 + a1;
  const double wr = off_diag ? w[8 * m.I + m.r] : 0.0;
  double b[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) b[c] = gv[c] * wr;
  const double cs = reduce_scatter8(b, m.r);
  if (off_diag) sm.part[m.I][8 * m.J + m.r] = cs;
}

__device__ __forceinline__ void thomas_solve_rd(ThomasSmem<CB>& sm, const double* __restrict__ G,
                                                const double* t, const double* tz, double* x) {
  constexpr int P = TH::P, NL = TH::NL, NBK = TH::NBK;
  const int tid = threadIdx.x;
  const MvRole<CB> m = mv_role<CB>();
  double gc[8], gn[8];
  load_row(gc, G, m);
  if (tid < P) sm.w2[0][tid] = t[tid];
  __syncthreads();
#pragma unroll 1
  for (int n = 0; n < NL; ++n) {
    if (n + 1 < NL) load_row(gn, G + (size_t)TH::plane_of(n + 1) * TH::PLANE, m);
    mv_partials_reg(sm, gc, sm.w2[n & 1], m);
    __syncthreads();
    if (tid < P) {
      double pr[NBK];
#pragma unroll
      for (int s = 0; s < NBK; ++s) pr[s] = sm.part[s][tid];
#pragma unroll
      for (int w = 1; w < NBK; w *= 2)
#pragma unroll
        for (int s = 0; s + w < NBK; s += 2 * w) pr[s] += pr[s + w];
      const double acc = pr[0];
      double* wn = sm.w2[(n + 1) & 1];
      const int row = tid;
      if (n < CB) {
        const int l = n * P + row;
        x[l] = acc;
        if (n + 1 < CB) {
          wn[row] = fma(tz[l + P], acc, t[l + P]);
        } else {
          x[l] = acc;
          wn[row] = -tz[l] * acc;
        }
      } else {
        const int k = TH::plane_of(n);
        const int l = k * P + row;
        const double xv = x[l] - acc;
        x[l] = xv;
        if (k > 0) wn[row] = -tz[l] * xv;
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) gc[c] = gn[c];
    __syncthreads();
  }
}

template <int MODE>  // 0 tma, 1 rd, 2 rd + L2 prefetch
__global__ void __launch_bounds__(TH::NT, MODE == 0 ? 4 : 3) k_bench(const double* __restrict__ Gf,
                                                                   const double* __restrict__ tin,
                                                                   double* xout) {
  constexpr int C = CB * CB * CB, NT = TH::NT;
  extern __shared__ __align__(128) unsigned char smraw[];
  struct Sm {
    ThomasSmem<CB> th;
    double tv[C];
    double tz[C];
  };
  Sm& sm = *reinterpret_cast<Sm*>(smraw + (MODE == 0 ? sizeof(double) * kSlots * TH::PLANE : 0));
  const int b = blockIdx.x;
  const double* G = Gf + (size_t)b * TH::PER_BRICK;
  if (MODE == 0) {
    sm.th.slots = reinterpret_cast<double(*)[TH::PLANE]>(smraw);
    thomas_init<CB>(sm.th);
    __syncthreads();
    thomas_prefetch<CB>(sm.th, G);
  }
  if (MODE == 2 && threadIdx.x == 0)
    for (int k = 0; k < CB; ++k) prefetch_l2(G + (size_t)k * TH::PLANE, TH::PLANE * sizeof(double));
  for (int c = threadIdx.x; c < C; c += NT) {
    sm.tv[c] = tin[(size_t)b * C + c];
    sm.tz[c] = c >= CB * CB ? -0.1 : 0.0;
  }
  if (MODE == 0) thomas_solve<CB>(sm.th, G, sm.tv, sm.tz, sm.tv);
  else {
    __syncthreads();
    thomas_solve_rd(sm.th, G, sm.tv, sm.tz, sm.tv);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += NT) xout[(size_t)b * C + c] = sm.tv[c];
}

template <int MODE>
float run(const double* G, const double* t, double* x, int nb, size_t smem, int reps = 20) {
  cudaFuncSetAttribute(k_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  for (int w = 0; w < 3; ++w) k_bench<MODE><<<nb, TH::NT, smem>>>(G, t, x);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k_bench<MODE><<<nb, TH::NT, smem>>>(G, t, x);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, e);
  return 1e3f * ms / reps;
}

int main() {
  const int nb = 4096;
  const size_t per = TH::PER_BRICK, C = CB * CB * CB;
  std::vector<double> hg(per * nb), hc(per * nb), ht(C * nb);
  // diagonally dominant symmetric planes so the solve stays bounded
  for (size_t i = 0; i < hg.size(); ++i) hg[i] = 1e-3 * (double)((i * 2654435761u) % 1000) / 1000.0;
  // swizzled -> chunk-major copy of the same matrices
  for (size_t blkbase = 0; blkbase < hg.size(); blkbase += 64)
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 8; ++c) hc[blkbase + cm(r, c)] = hg[blkbase + swz(r, c)];
  for (size_t i = 0; i < ht.size(); ++i) ht[i] = 1.0 + 1e-3 * (double)(i % 97);
  double *G, *Gc, *t, *x;
  cudaMalloc(&G, sizeof(double) * hg.size());
  cudaMalloc(&Gc, sizeof(double) * hc.size());
  cudaMalloc(&t, sizeof(double) * ht.size());
  cudaMalloc(&x, sizeof(double) * ht.size());
  cudaMemcpy(G, hg.data(), sizeof(double) * hg.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(Gc, hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(t, ht.data(), sizeof(double) * ht.size(), cudaMemcpyHostToDevice);
  const size_t smem_rd = sizeof(double) * 2 * C + sizeof(ThomasSmem<CB>) + 256;
  const size_t smem_tma = smem_rd + sizeof(double) * kSlots * TH::PLANE;
  const double gb = (double)sizeof(double) * per * nb / 1e9;
  std::vector<double> x0(C * nb), x1(C * nb);
  const float t0 = run<0>(G, t, x, nb, smem_tma);
  cudaMemcpy(x0.data(), x, sizeof(double) * x0.size(), cudaMemcpyDeviceToHost);
  const float t1 = run<1>(Gc, t, x, nb, smem_rd);
  cudaMemcpy(x1.data(), x, sizeof(double) * x1.size(), cudaMemcpyDeviceToHost);
  double md = 0.0;
  for (size_t i = 0; i < x0.size(); ++i) md = fmax(md, fabs(x0[i] - x1[i]) / (fabs(x0[i]) + 1e-300));
  const float t2 = run<2>(Gc, t, x, nb, smem_rd);
  printf("smem tma %zu KB rd %zu KB, G %.0f MB, max rel diff rd vs tma %.3e\n", smem_tma >> 10, smem_rd >> 10,
         gb * 1e3, md);
  printf("tma    %7.1f us  (%.0f GB/s of G)\n", t0, gb / (t0 * 1e-6));
  printf("rd     %7.1f us  (%.0f GB/s of G)\n", t1, gb / (t1 * 1e-6));
  printf("rd+l2  %7.1f us  (%.0f GB/s of G)\n", t2, gb / (t2 * 1e-6));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
