// Seeded synthetic designs on the device (§8(d)
// "Synthetic inputs"): bit-identical to paper_2410_06850_b200/inputs.py
// box_filter_design and the oracle's orc_box_filter_design.
//   1. u_i = Lcg64(seed).next_uniform(), i = 0..M-1 (rng.hpp:17-25), by
//      jump-ahead: state_{i+1} = a^{i+1} seed + c (a^i + ... + 1) mod 2^64;
//   2. `passes` box means of radius r over the clipped (2r+1)^3 window:
//      window sums along x, then y, then z, each accumulated from 0 in
//      increasing offset order, then divided by (count_x count_y) count_z;
//   3. the ceil(vf M) largest values -> 1, ties by lower index (rng.cpp:39-51):
//      an MSB-first 8-bit radix select of the (order-preserving) bit patterns
//      of the nonnegative values, then a block-ordered prefix count of the
//      values equal to the threshold.
// Host-side generation at 512^3 takes ~37 s; this path is HBM-bound.
#include "kernels.h"

namespace tmg {

namespace {
constexpr uint64_t kLcgA = 6364136223846793005ULL, kLcgC = 1442695040888963407ULL;
constexpr int kGenThreads = 256;

// (A, C) with state_e = A seed + C after e steps
__device__ __forceinline__ void lcg_jump(uint64_t e, uint64_t& A, uint64_t& C) {
  uint64_t ra = 1, rc = 0, pa = kLcgA, pc = kLcgC;  // result, power-of-two step
  while (e) {
    if (e & 1) {  // apply step (pa, pc) after the current result
      rc = pa * rc + pc;
      ra = pa * ra;
    }
    pc = pa * pc + pc;  // compose the step with itself
    pa = pa * pa;
    e >>= 1;
  }
  A = ra;
  C = rc;
}
}  // namespace

// each thread: G consecutive uniforms
__global__ void k_lcg_uniforms(double* out, int64_t n, uint64_t seed, int G) {
  const int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * G;
  if (i0 >= n) return;
  uint64_t A, C;
  lcg_jump((uint64_t)i0, A, C);
  uint64_t st = A * seed + C;  // state after i0 steps
  for (int g = 0; g < G && i0 + g < n; ++g) {
    st = kLcgA * st + kLcgC;
    out[i0 + g] = (double)(st >> 11) * 0x1.0p-53;
  }
}

// out = window sum of in along `axis` (0 = x), radius r; with denom, out /=
// (cx cy) cz of the clipped window (the last axis of a pass)
__global__ void k_window_sum(const double* __restrict__ in, double* out, int64_t nx, int64_t ny,
                             int64_t nz, int axis, int r, int divide) {
  const int64_t m = nx * ny * nz;
  const int64_t stride = axis == 0 ? 1 : axis == 1 ? nx : nx * ny;
  const int64_t na = axis == 0 ? nx : axis == 1 ? ny : nz;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = s % nx, j = (s / nx) % ny, k = s / (nx * ny);
    const int64_t a = axis == 0 ? i : axis == 1 ? j : k;
    double acc = 0.0;
    for (int d = -r; d <= r; ++d) {
      const int64_t b = a + d;
      if (b < 0 || b >= na) continue;
      acc += in[s + d * stride];
    }
    if (divide) {
      auto cnt = [r](int64_t c, int64_t n) {
        const int64_t lo = c - r < 0 ? 0 : c - r, hi = c + r > n - 1 ? n - 1 : c + r;
        return (double)(hi - lo + 1);
      };
      acc = acc / ((cnt(i, nx) * cnt(j, ny)) * cnt(k, nz));
    }
    out[s] = acc;
  }
}

// radix select: histogram of the digit at `shift` over keys matching prefix
__global__ void k_radix_hist(const double* __restrict__ f, int64_t m, const uint64_t* sel,
                             int shift, unsigned long long* hist) {
  __shared__ unsigned int h[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const uint64_t prefix = sel[0], mask = sel[1];
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = (uint64_t)__double_as_longlong(f[s]);
    if ((key & mask) == prefix) atomicAdd(&h[(key >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    if (h[b]) atomicAdd(&hist[b], (unsigned long long)h[b]);
}

// walk the bins from the largest digit; sel = {prefix, mask, k (rank still
// to take among the keys matching the prefix)}
__global__ void k_radix_pick(unsigned long long* hist, uint64_t* sel, int shift) {
  if (threadIdx.x != 0) return;
  uint64_t k = sel[2], cum = 0;
  for (int b = 255; b >= 0; --b) {
    const uint64_t h = hist[b];
    if (cum + h >= k) {
      sel[0] |= (uint64_t)b << shift;
      sel[1] |= (uint64_t)255 << shift;
      sel[2] = k - cum;
      break;
    }
    cum += h;
  }
  for (int b = 0; b < 256; ++b) hist[b] = 0;
}

// rho = key > threshold; per-chunk counts of keys equal to it
__global__ void k_mark_greater(const double* __restrict__ f, int64_t m, const uint64_t* sel,
                               int64_t chunk, double* rho, unsigned long long* eq_count) {
  __shared__ unsigned int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const uint64_t thr = sel[0];
  const int64_t a = blockIdx.x * chunk, b = a + chunk < m ? a + chunk : m;
  unsigned int mine = 0;
  for (int64_t s = a + threadIdx.x; s < b; s += blockDim.x) {
    const uint64_t key = (uint64_t)__double_as_longlong(f[s]);
    rho[s] = key > thr ? 1.0 : 0.0;
    mine += key == thr;
  }
  if (mine) atomicAdd(&cnt, mine);
  __syncthreads();
  if (threadIdx.x == 0) eq_count[blockIdx.x] = cnt;
}

__global__ void k_exclusive_scan(unsigned long long* v, int n) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long s = 0;
  for (int i = 0; i < n; ++i) {
    const unsigned long long t = v[i];
    v[i] = s;
    s += t;
  }
}

// the first k' keys equal to the threshold (lowest indices) -> 1
__global__ void k_mark_equal(const double* __restrict__ f, int64_t m, const uint64_t* sel,
                             int64_t chunk, const unsigned long long* eq_base, double* rho) {
  __shared__ unsigned int wsum[kGenThreads / 32];
  __shared__ unsigned long long base;
  const uint64_t thr = sel[0], take = sel[2];
  if (threadIdx.x == 0) base = eq_base[blockIdx.x];
  __syncthreads();
  if (base >= take) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t a = blockIdx.x * chunk, b = a + chunk < m ? a + chunk : m;
  for (int64_t t0 = a; t0 < b; t0 += blockDim.x) {
    const int64_t s = t0 + threadIdx.x;
    const bool eq = s < b && (uint64_t)__double_as_longlong(f[s]) == thr;
    const unsigned bal = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    unsigned before = 0, total = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      if (i < w) before += wsum[i];
      total += wsum[i];
    }
    const unsigned rank = before + __popc(bal & ((1u << lane) - 1u));
    if (eq && base + rank < take) rho[s] = 1.0;
    __syncthreads();
    if (threadIdx.x == 0) base += total;
    __syncthreads();
  }
}

size_t gen_scratch_bytes(int64_t m) {
  const int64_t chunks = (m + 65535) / 65536;
  return sizeof(double) * (size_t)m + sizeof(unsigned long long) * (size_t)(256 + chunks) +
         sizeof(uint64_t) * 4;
}

// Tree-like field (BASELINE configs[4], no reference generator; DESIGN.md
// §6 and inputs.tree_design): f = max over the seeded branch segments of the
// capsule profile (1 - d / w)_+ plus amp * u, u the LCG noise already in f.
// d is the distance from the cell centre to the segment, evaluated with
// explicitly rounded FP64 operations (no contraction) so the host restatement
// is bit-identical.
__global__ void k_tree_field(double* f, int64_t nx, int64_t ny, int64_t nz, double hx, double hy,
                             double hz, const double* __restrict__ seg, int nseg, double amp) {
  extern __shared__ double sseg[];  // 7 doubles per segment: a, b, w
  for (int i = threadIdx.x; i < 7 * nseg; i += blockDim.x) sseg[i] = seg[i];
  __syncthreads();
  const int64_t m = nx * ny * nz;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = s % nx, j = (s / nx) % ny, k = s / (nx * ny);
    const double px = __dmul_rn((double)i + 0.5, hx), py = __dmul_rn((double)j + 0.5, hy),
                 pz = __dmul_rn((double)k + 0.5, hz);
    double best = 0.0;
    for (int q = 0; q < nseg; ++q) {
      const double* g = sseg + 7 * q;
      const double ex = __dsub_rn(g[3], g[0]), ey = __dsub_rn(g[4], g[1]), ez = __dsub_rn(g[5], g[2]);
      const double wx = __dsub_rn(px, g[0]), wy = __dsub_rn(py, g[1]), wz = __dsub_rn(pz, g[2]);
      const double ee = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
      const double we = __dadd_rn(__dadd_rn(__dmul_rn(wx, ex), __dmul_rn(wy, ey)), __dmul_rn(wz, ez));
      double t = __ddiv_rn(we, ee);
      t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
      const double dx = __dsub_rn(wx, __dmul_rn(t, ex)), dy = __dsub_rn(wy, __dmul_rn(t, ey)),
                   dz = __dsub_rn(wz, __dmul_rn(t, ez));
      const double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                            __dmul_rn(dz, dz)));
      const double v = __dsub_rn(1.0, __ddiv_rn(d, g[6]));
      best = v > best ? v : best;
    }
    f[s] = __dadd_rn(best, __dmul_rn(amp, f[s]));
  }
}

static void filter_select(int64_t nx, int64_t ny, int64_t nz, double vf, int passes, int radius,
                          double* rho, double* f, void* scratch, cudaStream_t s);
static void select_top(int64_t m, double vf, double* rho, const double* f, void* scratch,
                       cudaStream_t s);
static void lcg_fill(double* f, int64_t m, uint64_t seed, cudaStream_t s);

// One 7-point averaging sweep of frozen_bench_design (rng.cpp:21-37): the
// cell and its in-domain face neighbours summed in the reference's order
// (self, x-, x+, y-, y+, z-, z+), divided by their count.
__global__ void k_star_average(const double* __restrict__ in, double* out, int64_t nx, int64_t ny,
                               int64_t nz) {
  const int64_t m = nx * ny * nz, sy = nx, sz = nx * ny;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = s % nx, j = (s / nx) % ny, k = s / sz;
    double sum = in[s];
    int n = 1;
    if (i > 0) { sum += in[s - 1]; ++n; }
    if (i < nx - 1) { sum += in[s + 1]; ++n; }
    if (j > 0) { sum += in[s - sy]; ++n; }
    if (j < ny - 1) { sum += in[s + sy]; ++n; }
    if (k > 0) { sum += in[s - sz]; ++n; }
    if (k < nz - 1) { sum += in[s + sz]; ++n; }
    out[s] = sum / n;
  }
}

// frozen_bench_design (rng.cpp:16-53): LCG uniforms, `passes` 7-point
// averaging sweeps, the ceil(vstar M) largest -> 1 (ties by lower index).
void launch_frozen_design(int64_t nx, int64_t ny, int64_t nz, double vstar, uint64_t seed,
                          int passes, double* rho, double* f, void* scratch, cudaStream_t s) {
  const int64_t m = nx * ny * nz;
  lcg_fill(f, m, seed, s);
  double* t = (double*)scratch;  // the first m doubles of the scratch
  int64_t gb = (m + kGenThreads - 1) / kGenThreads;
  if (gb > 148 * 64) gb = 148 * 64;
  for (int p = 0; p < passes; ++p) {
    k_star_average<<<(unsigned)gb, kGenThreads, 0, s>>>(f, t, nx, ny, nz);
    cudaMemcpyAsync(f, t, sizeof(double) * (size_t)m, cudaMemcpyDeviceToDevice, s);
  }
  select_top(m, vstar, rho, f, scratch, s);
}

static void lcg_fill(double* f, int64_t m, uint64_t seed, cudaStream_t s) {
  const int G = 16;
  const int64_t nthreads = (m + G - 1) / G;
  k_lcg_uniforms<<<(unsigned)((nthreads + kGenThreads - 1) / kGenThreads), kGenThreads, 0, s>>>(
      f, m, seed, G);
}

// rho (x-fastest, M = nx ny nz doubles) from the seeded generator; scratch of
// gen_scratch_bytes(M); f is a second M-double work array.
void launch_box_filter_design(int64_t nx, int64_t ny, int64_t nz, double vf, uint64_t seed,
                              int passes, int radius, double* rho, double* f, void* scratch,
                              cudaStream_t s) {
  lcg_fill(f, nx * ny * nz, seed, s);
  filter_select(nx, ny, nz, vf, passes, radius, rho, f, scratch, s);
}

// The tree-like design: noise (as above), k_tree_field over the segments
// (device array, 7 doubles each), then the same box means and top-k select.
void launch_tree_design(int64_t nx, int64_t ny, int64_t nz, double lx, double ly, double lz,
                        double vf, uint64_t seed, int passes, int radius, const double* seg,
                        int nseg, double amp, double* rho, double* f, void* scratch,
                        cudaStream_t s) {
  const int64_t m = nx * ny * nz;
  lcg_fill(f, m, seed, s);
  int64_t gb = (m + kGenThreads - 1) / kGenThreads;
  if (gb > 148 * 64) gb = 148 * 64;
  k_tree_field<<<(unsigned)gb, kGenThreads, sizeof(double) * 7 * nseg, s>>>(
      f, nx, ny, nz, lx / (double)nx, ly / (double)ny, lz / (double)nz, seg, nseg, amp);
  filter_select(nx, ny, nz, vf, passes, radius, rho, f, scratch, s);
}

static void filter_select(int64_t nx, int64_t ny, int64_t nz, double vf, int passes, int radius,
                          double* rho, double* f, void* scratch, cudaStream_t s) {
  const int64_t m = nx * ny * nz;
  double* t = (double*)scratch;
  int64_t gb = (m + kGenThreads - 1) / kGenThreads;
  if (gb > 148 * 64) gb = 148 * 64;
  for (int p = 0; p < passes; ++p) {
    k_window_sum<<<(unsigned)gb, kGenThreads, 0, s>>>(f, t, nx, ny, nz, 0, radius, 0);
    k_window_sum<<<(unsigned)gb, kGenThreads, 0, s>>>(t, rho, nx, ny, nz, 1, radius, 0);
    k_window_sum<<<(unsigned)gb, kGenThreads, 0, s>>>(rho, f, nx, ny, nz, 2, radius, 1);
  }
  select_top(m, vf, rho, f, scratch, s);
}

// rho = the ceil(vf M) largest values of f -> 1, ties by lower index
// (rng.cpp:39-51); f is not modified.
static void select_top(int64_t m, double vf, double* rho, const double* f, void* scratch,
                       cudaStream_t s) {
  double* t = (double*)scratch;
  unsigned long long* hist = (unsigned long long*)(t + m);
  const int64_t chunk = 65536, chunks = (m + chunk - 1) / chunk;
  unsigned long long* eq = hist + 256;
  uint64_t* sel = (uint64_t*)(eq + chunks);
  int64_t gb = (m + kGenThreads - 1) / kGenThreads;
  if (gb > 148 * 64) gb = 148 * 64;
  // solid = min(M, ceil(vf M)) largest (rng.cpp:39-51)
  int64_t solid = (int64_t)ceil(vf * (double)m);
  if (solid > m) solid = m;
  if (solid <= 0) {
    cudaMemsetAsync(rho, 0, sizeof(double) * (size_t)m, s);
    return;
  }
  const uint64_t init[3] = {0, 0, (uint64_t)solid};
  cudaMemcpyAsync(sel, init, sizeof init, cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * 256, s);
  for (int shift = 56; shift >= 0; shift -= 8) {
    k_radix_hist<<<(unsigned)gb, kGenThreads, 0, s>>>(f, m, sel, shift, hist);
    k_radix_pick<<<1, 32, 0, s>>>(hist, sel, shift);
  }
  k_mark_greater<<<(unsigned)chunks, kGenThreads, 0, s>>>(f, m, sel, chunk, rho, eq);
  k_exclusive_scan<<<1, 32, 0, s>>>(eq, (int)chunks);
  k_mark_equal<<<(unsigned)chunks, kGenThreads, 0, s>>>(f, m, sel, chunk, eq, rho);
}

}  // namespace tmg
