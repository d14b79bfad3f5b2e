// SIMP design loop on the device (BASELINE
// configs[2]): density filter, sensitivity filter (transpose), optimality-
// criteria update with a bisection on the volume multiplier. The filter and OC
// rules are builder-defined (the reference's own outer loop
// uses MMA, optim.cpp:121-345); the state/adjoint solves and the sensitivity
// are the reference's (optim.cpp:245-288, 21-84).
//
// Design vectors are x-fastest global arrays (one slab); the solver's brick
// layout is reached through the to/from-brick kernels.
#include "kernels.h"

namespace tmg {

// Linear-hat density filter of radius r (cells): w(d) = max(0, r - |d|) over
// the clipped (2R+1)^3 window, R = floor(r).
//  mode 0 (weights):   out_c = W_c = sum_n w_cn (in-domain neighbours)
//  mode 1 (filter):    out_c = sum_n w_cn in_n / W_c
//  mode 2 (transpose): out_c = sum_n w_cn in_n / W_n  (chain rule of mode 1)
__global__ void k_density_filter(int64_t nx, int64_t ny, int64_t nz, double r, int R,
                                 const double* __restrict__ in, const double* __restrict__ W,
                                 double* out, int mode) {
  const int64_t m = nx * ny * nz;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
    double acc = 0.0;
    for (int dk = -R; dk <= R; ++dk)
      for (int dj = -R; dj <= R; ++dj)
        for (int di = -R; di <= R; ++di) {
          const int64_t ii = i + di, jj = j + dj, kk = k + dk;
          if (ii < 0 || jj < 0 || kk < 0 || ii >= nx || jj >= ny || kk >= nz) continue;
          const double w = r - sqrt((double)(di * di + dj * dj + dk * dk));
          if (w <= 0.0) continue;
          const int64_t nbr = ii + nx * (jj + ny * kk);
          acc += mode == 0 ? w : (mode == 1 ? w * in[nbr] : w * in[nbr] / W[nbr]);
        }
    out[c] = mode == 1 ? acc / W[c] : acc;
  }
}

// OC candidate for multiplier lam (Sigmund's rule, move limit mv):
// x_new = clamp(x * sqrt(-dc / (lam * dv)), max(0, x - mv), min(1, x + mv)).
__global__ void k_oc_candidate(const double* __restrict__ x, const double* __restrict__ dc,
                               const double* __restrict__ dv, double lam, double mv, double xmin,
                               int64_t m, double* xnew) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m;
       c += (int64_t)gridDim.x * blockDim.x) {
    const double be = fmax(0.0, -dc[c]) / (lam * dv[c]);
    double v = x[c] * sqrt(be);
    v = fmin(fmin(v, x[c] + mv), 1.0);
    v = fmax(fmax(v, x[c] - mv), xmin);
    xnew[c] = v;
  }
}

// sum of v (deterministic: block tree + single-block final pass)
__global__ void k_sum_partial(const double* __restrict__ v, int64_t m, double* part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m;
       c += (int64_t)gridDim.x * blockDim.x)
    s += v[c];
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_sum_final(const double* __restrict__ part, int n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) *out = s;
}

// max |a - b| (||dx||_inf of an update)
__global__ void k_maxdiff_partial(const double* __restrict__ a, const double* __restrict__ b,
                                  int64_t m, double* part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m;
       c += (int64_t)gridDim.x * blockDim.x)
    s = fmax(s, fabs(a[c] - b[c]));
  for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
    part[blockIdx.x] = mx;
  }
}
__global__ void k_max_final(const double* __restrict__ part, int n, double* out) {
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int i = 0; i < n; ++i) mx = fmax(mx, part[i]);
    *out = mx;
  }
}

constexpr int kSumBlocks = 296;

void launch_maxdiff(const double* a, const double* b, int64_t m, double* part, double* out,
                    cudaStream_t s) {
  k_maxdiff_partial<<<kSumBlocks, 256, 0, s>>>(a, b, m, part);
  k_max_final<<<1, 32, 0, s>>>(part, kSumBlocks, out);
}

void launch_density_filter(int64_t nx, int64_t ny, int64_t nz, double r, const double* in,
                           const double* W, double* out, int mode, cudaStream_t s) {
  const int64_t m = nx * ny * nz;
  const int R = (int)floor(r);
  int64_t blocks = (m + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_density_filter<<<(unsigned)blocks, 256, 0, s>>>(nx, ny, nz, r, R, in, W, out, mode);
}

void launch_oc_candidate(const double* x, const double* dc, const double* dv, double lam,
                         double mv, double xmin, int64_t m, double* xnew, cudaStream_t s) {
  int64_t blocks = (m + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_oc_candidate<<<(unsigned)blocks, 256, 0, s>>>(x, dc, dv, lam, mv, xmin, m, xnew);
}

void launch_sum(const double* v, int64_t m, double* part, double* out, cudaStream_t s) {
  k_sum_partial<<<kSumBlocks, 256, 0, s>>>(v, m, part);
  k_sum_final<<<1, 256, 0, s>>>(part, kSumBlocks, out);
}

int64_t sum_partials_doubles() { return kSumBlocks; }

__global__ void k_fill(double* p, int64_t n, double v) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x)
    p[c] = v;
}
void launch_fill(double* p, int64_t n, double v, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_fill<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(p, n, v);
}

}  // namespace tmg
