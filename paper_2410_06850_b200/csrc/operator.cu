// Fine-grid elementwise / stencil kernels: layout permutation at the C-ABI
// boundary, SIMP conductivity, Dirichlet face masks, the right-hand side, the
// matrix-free TPFA apply and the Jacobi diagonal.
#include "kernels.h"
#include "stencil.cuh"

namespace tmg {

// global x-fastest index of brick-layout slot s (bricks of g.bx x g.by x g.bz
// cells, x-fastest inside)
__device__ __forceinline__ int64_t brick_to_global(const GridParams& g, int64_t s) {
  const int64_t c = brick_cells(g);
  const int64_t b = s / c;
  const int l = (int)(s % c);
  const int64_t bi = b % g.nbx, bj = (b / g.nbx) % g.nby, bk = b / (g.nbx * g.nby);
  const int li = l % g.bx, lj = (l / g.bx) % g.by, lk = l / (g.bx * g.by);
  const int64_t i = bi * g.bx + li, j = bj * g.by + lj, k = bk * g.bz + lk;
  return i + g.nx * (j + g.ny * k);
}

// src/dst: x-fastest cells of this context's z-slab (global index - xoff).
__global__ void k_to_brick(GridParams g, const double* __restrict__ src, double* dst,
                           int64_t s0, int64_t m, int64_t xoff) {
  for (int64_t s = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < s0 + m;
       s += (int64_t)gridDim.x * blockDim.x)
    dst[s] = src[brick_to_global(g, s) - xoff];
}

__global__ void k_from_brick(GridParams g, const double* __restrict__ src, double* dst,
                             int64_t s0, int64_t m, int64_t xoff) {
  for (int64_t s = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < s0 + m;
       s += (int64_t)gridDim.x * blockDim.x)
    dst[brick_to_global(g, s) - xoff] = src[s];
}

// interpolate_design (grid.cpp:220-241): piecewise-constant prolongation of a
// field on an (nxl, nyl, nzl) grid by integer factors, into this context's
// own cells (brick layout).
__global__ void k_interpolate(GridParams g, const double* __restrict__ lo, int64_t nxl,
                              int64_t nyl, int64_t fx, int64_t fy, int64_t fz, double* dst,
                              int64_t s0, int64_t m) {
  for (int64_t s = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < s0 + m;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gx = brick_to_global(g, s);
    const int64_t i = gx % g.nx, j = (gx / g.nx) % g.ny, k = gx / (g.nx * g.ny);
    dst[s] = lo[(i / fx) + nxl * ((j / fy) + nyl * (k / fz))];
  }
}

// material.cpp:45-59 — kappa = lo + x^p (hi - lo), repeated multiply
__global__ void k_conductivity(const double* __restrict__ x, double* kappa, int64_t s0, int64_t m,
                               double lo, double hi, int p) {
  const double dk = hi - lo;
  for (int64_t s = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < s0 + m;
       s += (int64_t)gridDim.x * blockDim.x) {
    double r = 1.0;
    for (int i = 0; i < p; ++i) r = __dmul_rn(r, x[s]);
    kappa[s] = __dadd_rn(lo, __dmul_rn(r, dk));
  }
}

struct PatchSet {
  int n;
  Patch p[kMaxPatches];
  double lx, ly, lz;
};

// grid.cpp:61-75 (face-centre containment, inclusive bounds)
__device__ bool dirichlet_value(const GridParams& g, const PatchSet& ps, int64_t i, int64_t j,
                                int64_t k, int face, double* value) {
  bool on = false;
  switch (face) {
    case 0: on = i == 0; break;
    case 1: on = i == g.nx - 1; break;
    case 2: on = j == 0; break;
    case 3: on = j == g.ny - 1; break;
    case 4: on = k == 0; break;
    default: on = k == g.nz - 1; break;
  }
  if (!on) return false;
  const double cx = __dmul_rn((double)i + 0.5, g.hx);
  const double cy = __dmul_rn((double)j + 0.5, g.hy);
  const double cz = __dmul_rn((double)k + 0.5, g.hz);
  double u, v;
  if (face <= 1) { u = cy; v = cz; }
  else if (face <= 3) { u = cx; v = cz; }
  else { u = cx; v = cy; }
  for (int q = 0; q < ps.n; ++q) {
    const Patch& p = ps.p[q];
    if (p.face != face) continue;
    if (u >= p.u0 && u <= p.u1 && v >= p.v0 && v <= p.v1) {
      if (value) *value = p.value;
      return true;
    }
  }
  return false;
}

// Per-cell Dirichlet face bits (brick layout) and the rhs
// b = f*vol + sum_D t_D * T_D in the reference face order (fvm.cpp:63-112).
__global__ void k_boundary(GridParams g, PatchSet ps, const double* __restrict__ kappa,
                           const double* __restrict__ source, uint8_t* dmask, double* rhs,
                           int64_t s0, int64_t m, unsigned long long* count) {
  for (int64_t s = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < s0 + m;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = brick_cells(g);
    const int64_t b = s / c;
    const int l = (int)(s % c);
    const int64_t bi = b % g.nbx, bj = (b / g.nbx) % g.nby, bk = b / (g.nbx * g.nby);
    const int64_t i = bi * g.bx + l % g.bx, j = bj * g.by + (l / g.bx) % g.by,
                  k = bk * g.bz + l / (g.bx * g.by);
    unsigned mask = 0;
    double bval = source ? __dmul_rn(source[s], g.vol) : 0.0;
    const bool bnd = i == 0 || j == 0 || k == 0 || i == g.nx - 1 || j == g.ny - 1 || k == g.nz - 1;
    if (bnd) {
      for (int f = 0; f < 6; ++f) {
        double td = 0.0;
        if (dirichlet_value(g, ps, i, j, k, f, &td)) {
          mask |= 1u << f;
          const double t = __dmul_rn(__dmul_rn(2.0, kappa[s]), g.cpl[f >> 1]);
          bval = __dadd_rn(bval, __dmul_rn(t, td));
        }
      }
      if (mask && count) atomicAdd(count, (unsigned long long)__popc(mask));
    }
    dmask[s] = (uint8_t)mask;
    if (rhs) rhs[s] = bval;
  }
}

// sensitivity (optim.cpp:21-84): adjoint gradient of the mean temperature per
// cell, face by face, in the reference's operation order (no contraction:
// bitwise). rho = design x, t = state, u = adjoint (brick layout, ghosts of
// t and u filled), kappa = the system's conductivity.
__global__ void k_sensitivity(GridParams g, PatchSet ps, const double* __restrict__ rho,
                              const double* __restrict__ kappa, const double* __restrict__ t,
                              const double* __restrict__ u, double kappa_lo, double kappa_hi,
                              double f0, int p, double* grad, int64_t s0, int64_t m) {
  const int64_t C = brick_cells(g);
  const int bd[3] = {g.bx, g.by, g.bz};
  const double dkm = __dsub_rn(kappa_hi, kappa_lo), pd = (double)p;
  for (int64_t s = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < s0 + m;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = s / C;
    const int l = (int)(s % C);
    const int64_t bi = b % g.nbx, bj = (b / g.nbx) % g.nby, bk = b / (g.nbx * g.nby);
    const int li = l % g.bx, lj = (l / g.bx) % g.by, lk = l / (g.bx * g.by);
    const int64_t ijk[3] = {bi * g.bx + li, bj * g.by + lj, bk * g.bz + lk};
    const int64_t n_axis[3] = {g.nx, g.ny, g.nz};
    // material_derivatives (material.cpp:61-74)
    double xp1 = 1.0;
    if (p >= 2)
      for (int q = 0; q < p - 1; ++q) xp1 = __dmul_rn(xp1, rho[s]);
    const double dk = __dmul_rn(__dmul_rn(pd, xp1), dkm);
    const double dsrc = __dmul_rn(__dmul_rn(-pd, xp1), f0);
    const double uc = u[s], tc = t[s];
    double value = __dmul_rn(__dmul_rn(uc, dsrc), g.vol);
    if (dk != 0.0) {
      const double kc = kappa[s];
      const int st_in[3] = {1, g.bx, g.bx * g.by};
      const int64_t st_b[3] = {1, g.nbx, g.nbx * g.nby};
      const int lc3[3] = {li, lj, lk};
      for (int a = 0; a < 3; ++a) {
        for (int side = 0; side < 2; ++side) {
          const bool exists = side == 0 ? ijk[a] > 0 : ijk[a] < n_axis[a] - 1;
          if (!exists) continue;
          // neighbour's storage index: inside the brick or across its face
          int64_t ns;
          if (side == 0)
            ns = lc3[a] > 0 ? s - st_in[a] : (b - st_b[a]) * C + (l + (bd[a] - 1) * st_in[a]);
          else
            ns = lc3[a] < bd[a] - 1 ? s + st_in[a] : (b + st_b[a]) * C + (l - (bd[a] - 1) * st_in[a]);
          const double kf = face_t(kc, kappa[ns]);
          const double ratio = __ddiv_rn(kf, kc);
          const double dt =
              __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(0.5, ratio), ratio), dk), g.cpl[a]);
          value = __dsub_rn(value, __dmul_rn(__dmul_rn(dt, __dsub_rn(uc, u[ns])),
                                             __dsub_rn(tc, t[ns])));
        }
        for (int side = 0; side < 2; ++side) {
          double td = 0.0;
          if (dirichlet_value(g, ps, ijk[0], ijk[1], ijk[2], 2 * a + side, &td)) {
            const double dt = __dmul_rn(__dmul_rn(2.0, g.cpl[a]), dk);
            value = __dadd_rn(value, __dmul_rn(__dmul_rn(dt, uc), __dsub_rn(td, tc)));
          }
        }
      }
    }
    grad[s] = value;
  }
}

// y = A x from the precomputed coefficients (bitwise SparseOperator::apply),
// optionally dinv = 1/diag (JacobiPreconditioner, solver.cpp:21-29).
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_apply(GridParams g, const double* __restrict__ coef,
                                                       int64_t M, const double* __restrict__ x,
                                                       double* y, double* dinv) {
  __shared__ CoefSmem<CB> cs;
  __shared__ double xt[Tile<CB>::N];
  constexpr int C = CB * CB * CB;
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  load_coefs<CB>(coef, M, cs, g, bc);
  if (x) load_tile<CB, true>(x, xt, g, bc);
  __syncthreads();
  const int t = threadIdx.x, li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
  const size_t s = bofs(bc.b, C) + t;
  if (y) y[s] = apply_coef<CB>(cs, xt, li, lj, lk);
  if (dinv) dinv[s] = 1.0 / cs.dg[t];  // solver.cpp:27
}

// y = |A| |x|: every term of the row sum made nonnegative (the scale of the
// rounding error of b - A x, eps |A||x|).
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_apply_abs(GridParams g,
                                                           const double* __restrict__ coef,
                                                           int64_t M, const double* __restrict__ x,
                                                           double* y) {
  __shared__ CoefSmem<CB> cs;
  __shared__ double xt[Tile<CB>::N];
  constexpr int C = CB * CB * CB;
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  load_coefs<CB>(coef, M, cs, g, bc);
  load_tile<CB, true>(x, xt, g, bc);
  __syncthreads();
  const int t = threadIdx.x, li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
  constexpr int E = Tile<CB>::E;
  const int ti = Tile<CB>::idx(li, lj, lk);
  const double* pz = lk > 0 ? cs.cz + (t - CB * CB) : cs.hz + (li + CB * lj);
  const double* py = lj > 0 ? cs.cy + (t - CB) : cs.hy + (li + CB * lk);
  const double* px = li > 0 ? cs.cx + (t - 1) : cs.hx + (lj + CB * lk);
  double v = fabs(*pz * xt[ti - E * E]) + fabs(*py * xt[ti - E]) + fabs(*px * xt[ti - 1]) +
             fabs(cs.dg[t] * xt[ti]) + fabs(cs.cx[t] * xt[ti + 1]) + fabs(cs.cy[t] * xt[ti + E]) +
             fabs(cs.cz[t] * xt[ti + E * E]);
  y[bofs(bc.b, C) + t] = v;
}

static int grid1d(int64_t m) {
  int64_t b = (m + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (int)b;
}

// own cells of the context: brick-layout [b0*C, (b0+nbo)*C); x-fastest slab
// arrays start at global cell (b0 / (nbx*nby)) * bz * nx * ny
static int64_t slab_xoff(const GridParams& g) {
  return (g.b0 / (g.nbx * g.nby)) * g.bz * g.nx * g.ny;
}
void launch_to_brick(const GridParams& g, int cb, const double* src, double* dst, cudaStream_t s) {
  const int64_t C = brick_cells(g), m = g.nbo * C;
  k_to_brick<<<grid1d(m), 256, 0, s>>>(g, src, dst, g.b0 * C, m, slab_xoff(g));
}
void launch_from_brick(const GridParams& g, int cb, const double* src, double* dst,
                       cudaStream_t s) {
  const int64_t C = brick_cells(g), m = g.nbo * C;
  k_from_brick<<<grid1d(m), 256, 0, s>>>(g, src, dst, g.b0 * C, m, slab_xoff(g));
}
void launch_interpolate(const GridParams& g, int cb, const double* lo, const int64_t* nlo,
                        double* dst, cudaStream_t s) {
  const int64_t C = brick_cells(g), m = g.nbo * C;
  k_interpolate<<<grid1d(m), 256, 0, s>>>(g, lo, nlo[0], nlo[1], g.nx / nlo[0], g.ny / nlo[1],
                                          g.nz / nlo[2], dst, g.b0 * C, m);
}
void launch_conductivity(const GridParams& g, int cb, const double* x, double* kappa, double lo,
                         double hi, int p, cudaStream_t s) {
  const int64_t C = brick_cells(g), m = g.nbo * C;
  k_conductivity<<<grid1d(m), 256, 0, s>>>(x, kappa, g.b0 * C, m, lo, hi, p);
}
void launch_boundary(const GridParams& g, int cb, const Patch* patches, int npatch, double lx,
                     double ly, double lz, const double* kappa, const double* source,
                     uint8_t* dmask, double* rhs, unsigned long long* count, cudaStream_t s) {
  PatchSet ps{};
  ps.n = npatch;
  for (int i = 0; i < npatch && i < kMaxPatches; ++i) ps.p[i] = patches[i];
  ps.lx = lx; ps.ly = ly; ps.lz = lz;
  const int64_t C = brick_cells(g), m = g.nbo * C;
  k_boundary<<<grid1d(m), 256, 0, s>>>(g, ps, kappa, source, dmask, rhs, g.b0 * C, m, count);
}
void launch_sensitivity(const GridParams& g, int cb, const Patch* patches, int npatch, double lx,
                        double ly, double lz, const double* rho, const double* kappa,
                        const double* t, const double* u, double kappa_lo, double kappa_hi,
                        double f0, int p, double* grad, cudaStream_t s) {
  PatchSet ps{};
  ps.n = npatch;
  for (int i = 0; i < npatch && i < kMaxPatches; ++i) ps.p[i] = patches[i];
  ps.lx = lx; ps.ly = ly; ps.lz = lz;
  const int64_t C = brick_cells(g), m = g.nbo * C;
  k_sensitivity<<<grid1d(m), 256, 0, s>>>(g, ps, rho, kappa, t, u, kappa_lo, kappa_hi, f0, p,
                                          grad, g.b0 * C, m);
}
void launch_apply_abs(const GridParams& g, int cb, const double* coef, const double* x, double* y,
                      cudaStream_t s) {
  const int64_t M = g.mst;
  if (cb == 0)
    launch_g_apply(g, coef, x, y, nullptr, 1, s);
  else if (cb == 8)
    k_apply_abs<8><<<(unsigned)g.nbo, 512, 0, s>>>(g, coef, M, x, y);
  else
    k_apply_abs<4><<<(unsigned)g.nbo, 64, 0, s>>>(g, coef, M, x, y);
}
void launch_apply(const GridParams& g, int cb, const double* coef, const double* x, double* y,
                  double* dinv, cudaStream_t s) {
  const int64_t M = g.mst;
  if (cb == 0)
    launch_g_apply(g, coef, x, y, dinv, 0, s);
  else if (cb == 8)
    k_apply<8><<<(unsigned)g.nbo, 512, 0, s>>>(g, coef, M, x, y, dinv);
  else
    k_apply<4><<<(unsigned)g.nbo, 64, 0, s>>>(g, coef, M, x, y, dinv);
}

}  // namespace tmg
