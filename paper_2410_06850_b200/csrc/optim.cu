// The reference's design loop on the device (topmg::optimize, optim.cpp:240-345):
// design-dependent heat source and the single-constraint MMA update
// (mma_update, optim.cpp:121-220). Design arrays are x-fastest here.
//
// MMA per cell j (range = xmax - xmin = 1):
//   asymptotes: iteration < 2: low = x - asy_init, upp = x + asy_init; else
//     widened / shrunk by the oscillation trend and guarded (:140-156);
//   subproblem: alpha = max(xmin, low + 0.1 (x - low), x - move),
//     beta = min(xmax, upp - 0.1 (upp - x), x + move), du = upp - x,
//     dl = x - low, p0 = du^2 max(g, 0), q0 = dl^2 max(-g, 0), and the same
//     with the constraint gradient c (the reference passes c = 1/M);
//   r1 = constraint - sum_j (p1/du + q1/dl);
//   x(lambda) = clamp((low sqrt(p) + upp sqrt(q)) / (sqrt(p) + sqrt(q)),
//                     alpha, beta), p = p0 + lambda p1, q = q0 + lambda q1;
//   dual: lambda = 0 unless the constraint approximation at 0 is positive,
//     then hi doubles from 1 until it is <= 0 (at most 80 times, else
//     SolverError), 128 bisection steps, lambda = hi (:187-208).
// The dual runs as one cooperative kernel: every evaluation of the
// constraint approximation is a grid-wide sum whose per-CTA partials every
// CTA adds in the same fixed order, so all CTAs take the same branch.
#include "kernels.h"

namespace tmg {

namespace {
constexpr int kMmaThreads = 256;

struct MmaSub {
  double x, low, upp, alpha, beta, p0, q0, p1, q1;
};

__device__ __forceinline__ MmaSub mma_sub(double x, double g, double low, double upp, double c,
                                          double move, double xmin, double xmax) {
  MmaSub s;
  const double range = xmax - xmin;
  s.x = x;
  s.low = low;
  s.upp = upp;
  s.alpha = fmax(fmax(xmin, low + 0.1 * (x - low)), x - move * range);
  s.beta = fmin(fmin(xmax, upp - 0.1 * (upp - x)), x + move * range);
  const double du = upp - x, dl = x - low;
  s.p0 = du * du * fmax(g, 0.0);
  s.q0 = dl * dl * fmax(-g, 0.0);
  s.p1 = du * du * fmax(c, 0.0);
  s.q1 = dl * dl * fmax(-c, 0.0);
  return s;
}

// primal_from_multiplier (optim.cpp:95-108)
__device__ __forceinline__ double mma_primal(const MmaSub& s, double lambda) {
  const double pj = s.p0 + lambda * s.p1, qj = s.q0 + lambda * s.q1;
  double xi;
  if (pj <= 0.0 && qj <= 0.0) {
    xi = s.x;
  } else {
    const double sp = sqrt(pj), sq = sqrt(qj);
    xi = (s.low * sp + s.upp * sq) / (sp + sq);
  }
  return fmin(fmax(xi, s.alpha), s.beta);
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

__device__ __forceinline__ void coop_barrier(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = bar + 1;
    const unsigned int my = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == my) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}
}  // namespace

// f = f0 (1 - x^p) (heat_source, material.cpp:61-66), repeated multiply
__global__ void k_heat_source(const double* __restrict__ x, double* f, int64_t s0, int64_t m,
                              double f0, int p) {
  for (int64_t s = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < s0 + m;
       s += (int64_t)gridDim.x * blockDim.x) {
    double r = 1.0;
    for (int i = 0; i < p; ++i) r = __dmul_rn(r, x[s]);
    f[s] = __dmul_rn(f0, __dsub_rn(1.0, r));
  }
}

// moving asymptotes (optim.cpp:138-157)
__global__ void k_mma_asymptotes(const double* __restrict__ x, const double* __restrict__ xp,
                                 const double* __restrict__ xp2, double* low, double* upp,
                                 int64_t n, int iteration, MmaParams o) {
  const double range = o.xmax - o.xmin;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double xj = x[j];
    if (iteration < 2) {
      low[j] = xj - o.asy_init * range;
      upp[j] = xj + o.asy_init * range;
    } else {
      const double trend = (xj - xp[j]) * (xp[j] - xp2[j]);
      double factor = 1.0;
      if (trend > 0.0) factor = o.asy_incr;
      else if (trend < 0.0) factor = o.asy_decr;
      double l = xj - factor * (xp[j] - low[j]);
      double u = xj + factor * (upp[j] - xp[j]);
      l = fmax(l, xj - 10.0 * range);
      l = fmin(l, xj - 0.01 * range);
      u = fmin(u, xj + 10.0 * range);
      u = fmax(u, xj + 0.01 * range);
      low[j] = l;
      upp[j] = u;
    }
  }
}

// The multiplier: r1, then the reference's bracket expansion and bisection.
// out[0] = lambda, out[1] = status (0 ok, 1 bracket expansion failed),
// out[2] = last hi (for the error message).
__global__ void __launch_bounds__(kMmaThreads) k_mma_dual(const double* __restrict__ x,
                                                          const double* __restrict__ grad,
                                                          const double* __restrict__ low,
                                                          const double* __restrict__ upp,
                                                          int64_t n, double constraint,
                                                          MmaParams o, double* partials,
                                                          unsigned int* bar, double* out) {
  __shared__ double red[32];
  int buf = 0;
  // every CTA returns the same total: partials summed in CTA order
  auto grid_total = [&](double v) {
    const double b = block_sum(v, red);
    double* P = partials + (size_t)buf * gridDim.x;
    if (threadIdx.x == 0) P[blockIdx.x] = b;
    coop_barrier(bar);
    double s = 0.0;
    for (unsigned i = 0; i < gridDim.x; ++i) s += __ldcg(P + i);
    buf ^= 1;  // the next total writes the other buffer while this one is read
    return s;
  };
  const int64_t j0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                stride = (int64_t)gridDim.x * blockDim.x;
  // r1 = constraint - sum (p1/du + q1/dl)
  double v = 0.0;
  for (int64_t j = j0; j < n; j += stride) {
    const MmaSub s = mma_sub(x[j], grad[j], low[j], upp[j], o.cgrad, o.move, o.xmin, o.xmax);
    v += s.p1 / (s.upp - s.x) + s.q1 / (s.x - s.low);
  }
  const double r1 = constraint - grid_total(v);
  auto constraint_at = [&](double lambda) {  // optim.cpp:110-118
    double w = 0.0;
    for (int64_t j = j0; j < n; j += stride) {
      const MmaSub s = mma_sub(x[j], grad[j], low[j], upp[j], o.cgrad, o.move, o.xmin, o.xmax);
      const double xi = mma_primal(s, lambda);
      w += s.p1 / (s.upp - xi) + s.q1 / (xi - s.low);
    }
    return r1 + grid_total(w);
  };
  double lambda = 0.0, status = 0.0, lo = 0.0, hi = 1.0;
  if (constraint_at(0.0) > 0.0) {
    int expand = 0;
    while (constraint_at(hi) > 0.0) {
      lo = hi;
      hi *= 2.0;
      if (++expand > 80) {
        status = 1.0;
        break;
      }
    }
    if (status == 0.0) {
      for (int it = 0; it < 128; ++it) {
        lambda = 0.5 * (lo + hi);
        if (constraint_at(lambda) > 0.0) lo = lambda;
        else hi = lambda;
      }
      lambda = hi;  // feasible side of the bracket
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = lambda;
    out[1] = status;
    out[2] = hi;
  }
}

// x_new = clamp(x(lambda), 0, 1) (optim.cpp:210-212, :318) and per-CTA
// partial max |x_new - x|
__global__ void __launch_bounds__(kMmaThreads) k_mma_primal(const double* __restrict__ x,
                                                            const double* __restrict__ grad,
                                                            const double* __restrict__ low,
                                                            const double* __restrict__ upp,
                                                            int64_t n, const double* lam,
                                                            MmaParams o, double* xnew,
                                                            double* partials) {
  __shared__ double red[32];
  const double lambda = lam[0];
  double m = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const MmaSub s = mma_sub(x[j], grad[j], low[j], upp[j], o.cgrad, o.move, o.xmin, o.xmax);
    const double xn = fmin(fmax(mma_primal(s, lambda), 0.0), 1.0);
    xnew[j] = xn;
    m = fmax(m, fabs(xn - x[j]));
  }
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b = fmax(b, red[w]);
    partials[blockIdx.x] = b;
  }
}

__global__ void k_max_partials(const double* partials, int n, double* out) {
  if (threadIdx.x != 0) return;
  double m = 0.0;
  for (int i = 0; i < n; ++i) m = fmax(m, partials[i]);
  out[0] = m;
}

// ------------------------------------------------------------ launchers

static int mma_grid() {  // per device: co-resident CTAs of the cooperative dual
  const int per = device_occupancy(k_mma_dual, kMmaThreads, 0);
  return device_sm_count() * (per < 2 ? per : 2);
}

int mma_partials_doubles() { return 2 * mma_grid() + 8; }

void launch_heat_source(const GridParams& g, int cb, const double* x, double* f, double f0, int p,
                        cudaStream_t s) {
  (void)cb;
  const int64_t C = brick_cells(g), m = g.nbo * C;
  int64_t b = (m + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  k_heat_source<<<(unsigned)(b < 1 ? 1 : b), 256, 0, s>>>(x, f, g.b0 * C, m, f0, p);
}

void launch_mma_asymptotes(const double* x, const double* xp, const double* xp2, double* low,
                           double* upp, int64_t n, int iteration, const MmaParams& o,
                           cudaStream_t s) {
  k_mma_asymptotes<<<mma_grid(), kMmaThreads, 0, s>>>(x, xp, xp2, low, upp, n, iteration, o);
}

void launch_mma_dual(const double* x, const double* grad, const double* low, const double* upp,
                     int64_t n, double constraint, const MmaParams& o, double* partials,
                     unsigned int* bar, double* out, cudaStream_t s) {
  void* args[] = {(void*)&x, (void*)&grad, (void*)&low, (void*)&upp, (void*)&n,
                  (void*)&constraint, (void*)&o, (void*)&partials, (void*)&bar, (void*)&out};
  launch_check(cudaLaunchCooperativeKernel((const void*)k_mma_dual, dim3(mma_grid()),
                                           dim3(kMmaThreads), args, 0, s),
               "k_mma_dual (cooperative) launch");
}

void launch_mma_primal(const double* x, const double* grad, const double* low, const double* upp,
                       int64_t n, const double* lam, const MmaParams& o, double* xnew,
                       double* partials, double* dx_out, cudaStream_t s) {
  k_mma_primal<<<mma_grid(), kMmaThreads, 0, s>>>(x, grad, low, upp, n, lam, o, xnew, partials);
  k_max_partials<<<1, 32, 0, s>>>(partials, mma_grid(), dx_out);
}

}  // namespace tmg
