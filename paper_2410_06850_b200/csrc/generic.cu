// Generic brick shapes: the whole MMG / PCG path for any coarse-cell extent
// (SURVEY.md §8 row A20).
//
// The reference accepts any HierarchicalGrid (grid.cpp:191-218): per axis
// cells_per_c = n / (ncc sd), so coarse cells are c_x x c_y x c_z boxes of any
// size -- 2^3 at the coarsest level of a three-level optimize() run, 12^3 for a
// 96^3 grid with ncc = 4, sd = 2, non-cubic for non-cubic grids -- and above
// 4096 cells per box the local eigenproblem switches to Lanczos
// (coarse_space.cpp:61-198, 229-230). The tuned kernels (pcg.cu, smoother.cuh,
// spectral.cu) are templated on cubic 4^3 / 8^3 bricks; every other shape runs
// here, on the same brick layout (bricks of g.bx x g.by x g.bz cells,
// x-fastest inside), the same device-side CG scalars (pcg_fin.cuh) and the
// same coarse and coarse-coarse levels (coarse.cu, coarse_large.cu,
// acc_planes.cu, which never see the brick shape). The launchers in pcg.cu /
// operator.cu / block_jacobi.cu route cb = 0 here.
//
// * Operator: one thread per cell; the row is summed in the reference's
//   sorted-column order without contraction, so y = A x stays bitwise equal
//   to SparseOperator::apply (sparse.cpp:71-84).
// * Fine smoother: exact block solves on boxes (the bricks, or the cc
//   elements of fine_blocks_by_cc, solver.cpp:353-361) by block Thomas over the
//   box's z planes with explicit Schur-complement inverses
//       G_0 = A_00^-1, G_k = (A_kk - D_k G_{k-1} D_k)^-1,
//       y_k = G_k (r_k + D_k y_{k-1}),  x_k = y_k + G_k D_{k+1} x_{k+1},
//   the inverses batched over boxes on the FP64 tensor cores
//   (dense_spd_inverse_batched), the LDL^T pivots of every plane folded into
//   one per-box extremum for the reference's singular-pivot rule
//   (solver.cpp:86-92). The apply is one launch per plane step, grid (column
//   slices, boxes).
// * Local bases: Chebyshev-filtered subspace iteration (the algorithm of
//   spectral.cu) with the 8-vector block in global scratch instead of
//   registers, so one CTA handles a box of any size -- the same eigenpairs the
//   reference's dense (n <= 4096) and Lanczos (n > 4096) paths return, to the
//   solver tolerance. Boxes of fewer than 8 cells are solved densely.
// * A_c / Bc blocks, literal restriction, prolongation, residuals: per brick
//   or per cell, the definitions of coarse.cu / block_jacobi.cu.
#include <algorithm>

#include "eig_small.cuh"
#include "kernels.h"
#include "pcg_fin.cuh"
#include "stencil.cuh"

namespace tmg {

namespace {

constexpr int kGT = 256;  // CTA size of the generic kernels
constexpr int kGLc = 6;   // largest L_c (same bound as the tuned kernels)

struct GCell {
  int64_t b;        // brick
  int l;            // cell inside the brick (x-fastest)
  int li, lj, lk;   // its brick-local coordinates
  int64_t i, j, k;  // global coordinates
};

__device__ __forceinline__ GCell gcell(const GridParams& g, int64_t s) {
  const int64_t C = brick_cells(g);
  GCell c;
  c.b = s / C;
  c.l = (int)(s - c.b * C);
  const int64_t bi = c.b % g.nbx, bj = (c.b / g.nbx) % g.nby, bk = c.b / (g.nbx * g.nby);
  c.li = c.l % g.bx;
  c.lj = (c.l / g.bx) % g.by;
  c.lk = c.l / (g.bx * g.by);
  c.i = bi * g.bx + c.li;
  c.j = bj * g.by + c.lj;
  c.k = bk * g.bz + c.lk;
  return c;
}

// storage slot of global cell (i, j, k)
__device__ __forceinline__ int64_t gslot(const GridParams& g, int64_t i, int64_t j, int64_t k) {
  const int64_t bi = i / g.bx, bj = j / g.by, bk = k / g.bz;
  const int li = (int)(i - bi * g.bx), lj = (int)(j - bj * g.by), lk = (int)(k - bk * g.bz);
  return (bi + g.nbx * (bj + g.nby * bk)) * brick_cells(g) + li + g.bx * (lj + g.by * lk);
}

// slot of the neighbour across face f (0 x-lo .. 5 z-hi); -1 outside the domain
__device__ __forceinline__ int64_t gnbr(const GridParams& g, const GCell& c, int64_t s, int f) {
  switch (f) {
    case 0: return c.i == 0 ? -1 : (c.li > 0 ? s - 1 : gslot(g, c.i - 1, c.j, c.k));
    case 1: return c.i + 1 >= g.nx ? -1 : (c.li + 1 < g.bx ? s + 1 : gslot(g, c.i + 1, c.j, c.k));
    case 2: return c.j == 0 ? -1 : (c.lj > 0 ? s - g.bx : gslot(g, c.i, c.j - 1, c.k));
    case 3:
      return c.j + 1 >= g.ny ? -1 : (c.lj + 1 < g.by ? s + g.bx : gslot(g, c.i, c.j + 1, c.k));
    case 4:
      return c.k == 0 ? -1 : (c.lk > 0 ? s - (int64_t)g.bx * g.by : gslot(g, c.i, c.j, c.k - 1));
    default:
      return c.k + 1 >= g.nz ? -1
                             : (c.lk + 1 < g.bz ? s + (int64_t)g.bx * g.by
                                                : gslot(g, c.i, c.j, c.k + 1));
  }
}

// (A x)_s in the sorted-column order of SparseOperator::apply (z-lo, y-lo,
// x-lo, diag, x-hi, y-hi, z-hi), no contraction; missing neighbours
// contribute -0 * 0, as in apply_coef (stencil.cuh). val(slot) gives x.
template <typename V>
__device__ __forceinline__ double g_row(const GridParams& g, const double* __restrict__ coef,
                                        int64_t M, const GCell& c, int64_t s, V val) {
  int64_t nb[6];
#pragma unroll
  for (int f = 0; f < 6; ++f) nb[f] = gnbr(g, c, s, f);
  const double tzl = nb[4] >= 0 ? coef[2 * M + nb[4]] : 0.0, xzl = nb[4] >= 0 ? val(nb[4]) : 0.0;
  const double tyl = nb[2] >= 0 ? coef[M + nb[2]] : 0.0, xyl = nb[2] >= 0 ? val(nb[2]) : 0.0;
  const double txl = nb[0] >= 0 ? coef[nb[0]] : 0.0, xxl = nb[0] >= 0 ? val(nb[0]) : 0.0;
  const double xxh = nb[1] >= 0 ? val(nb[1]) : 0.0, xyh = nb[3] >= 0 ? val(nb[3]) : 0.0,
               xzh = nb[5] >= 0 ? val(nb[5]) : 0.0;
  double r = __dadd_rn(0.0, __dmul_rn(-tzl, xzl));
  r = __dadd_rn(r, __dmul_rn(-tyl, xyl));
  r = __dadd_rn(r, __dmul_rn(-txl, xxl));
  r = __dadd_rn(r, __dmul_rn(coef[3 * M + s], val(s)));
  r = __dadd_rn(r, __dmul_rn(-coef[s], xxh));
  r = __dadd_rn(r, __dmul_rn(-coef[M + s], xyh));
  r = __dadd_rn(r, __dmul_rn(-coef[2 * M + s], xzh));
  return r;
}

// grid of the per-cell kernels: their reductions leave K gridDim.x partials
// in the context's 4 nbo + 64 doubles
unsigned cell_grid(const GridParams& g) {
  const int64_t m = g.nbo * brick_cells(g);
  int64_t n = (m + kGT - 1) / kGT;
  n = std::min<int64_t>(n, 2 * g.nbo + 32);
  n = std::min<int64_t>(n, 148 * 16);
  return (unsigned)std::max<int64_t>(n, 1);
}

#define FOR_OWN_CELLS(s)                                                            \
  for (int64_t s = g.b0 * brick_cells(g) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x, \
               s##_end = (g.b0 + g.nbo) * brick_cells(g);                            \
       s < s##_end; s += (int64_t)gridDim.x * blockDim.x)

}  // namespace

// ------------------------------------------------------------ coefficients
// fvm.cpp:33-120: T = face_transmissibility(k_low, k_high) * area/h per
// interior face, 2 k_c area/h per Dirichlet face, diagonal in face order.
__global__ void __launch_bounds__(kGT) k_g_coefficients(GridParams g,
                                                       const double* __restrict__ kappa,
                                                       const uint8_t* __restrict__ dmask,
                                                       double* coef, int64_t M) {
  FOR_OWN_CELLS(s) {
    const GCell c = gcell(g, s);
    const double kc = kappa[s];
    const unsigned dm = dmask[s];
    double t[6], diag = 0.0;
    bool has[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int64_t nb = gnbr(g, c, s, f);
      const double cp = g.cpl[f >> 1];
      has[f] = nb >= 0;
      t[f] = 0.0;
      if (nb >= 0) {
        t[f] = __dmul_rn((f & 1) ? face_t(kc, kappa[nb]) : face_t(kappa[nb], kc), cp);
        diag = __dadd_rn(diag, t[f]);
      } else if (dm & (1u << f)) {
        t[f] = __dmul_rn(__dmul_rn(2.0, kc), cp);
        diag = __dadd_rn(diag, t[f]);
      }
    }
    coef[s] = has[1] ? t[1] : 0.0;
    coef[M + s] = has[3] ? t[3] : 0.0;
    coef[2 * M + s] = has[5] ? t[5] : 0.0;
    coef[3 * M + s] = diag;
  }
}

// y = A x (absval: |A| |x|), dinv = 1 / diag (JacobiPreconditioner)
__global__ void __launch_bounds__(kGT) k_g_apply(GridParams g, const double* __restrict__ coef,
                                                int64_t M, const double* __restrict__ x,
                                                double* y, double* dinv, int absval) {
  FOR_OWN_CELLS(s) {
    if (dinv) dinv[s] = 1.0 / coef[3 * M + s];  // solver.cpp:27
    if (!y) continue;
    const GCell c = gcell(g, s);
    if (!absval) {
      y[s] = g_row(g, coef, M, c, s, [&](int64_t n) { return x[n]; });
    } else {
      double v = fabs(coef[3 * M + s] * x[s]);
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        const int64_t nb = gnbr(g, c, s, f);
        if (nb < 0) continue;
        const double T = coef[(size_t)(f >> 1) * M + ((f & 1) ? s : nb)];
        v += fabs(T * x[nb]);
      }
      y[s] = v;
    }
  }
}

// ------------------------------------------------------------ CG kernels
// r = b - A x0 (or r = b, x = 0), b.b and r.r -> fin_init (solver.cpp:515-531)
__global__ void __launch_bounds__(kGT) k_g_init(GridParams g, const double* __restrict__ coef,
                                               int64_t M, const double* __restrict__ b, double* x,
                                               int has_x0, double* r, PcgState* st,
                                               double* partials) {
  __shared__ double red[80];
  __shared__ int flag;
  double v[2] = {0.0, 0.0};
  FOR_OWN_CELLS(s) {
    const double bv = b[s];
    double rv;
    if (has_x0) {
      const GCell c = gcell(g, s);
      rv = bv - g_row(g, coef, M, c, s, [&](int64_t n) { return x[n]; });
    } else {
      x[s] = 0.0;
      rv = bv;
    }
    r[s] = rv;
    v[0] += bv * bv;
    v[1] += rv * rv;
  }
  block_sum_k<kGT, 2>(v, red);
  double tot[2];
  if (grid_reduce_last_k<2>(v, partials, &st->ticket[0], tot, &flag, red) && threadIdx.x == 0) {
    if (g.dist) {
      st->loc[kRedInit] = tot[0];
      st->loc[kRedInit + 1] = tot[1];
    } else {
      fin_init(st, tot[0], tot[1]);
    }
  }
}

// p = z + beta p_old (z on the first iteration), q = A p, p.q -> fin_search
// (solver.cpp:538-549, 565-567); neighbours' p is recomputed from z, p_old
__global__ void __launch_bounds__(kGT) k_g_search(GridParams g, const double* __restrict__ coef,
                                                 int64_t M, const double* __restrict__ z,
                                                 const double* __restrict__ p_old, double* p,
                                                 double* q, PcgState* st, double* partials) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  __shared__ double red[80];
  __shared__ int flag;
  const bool first = st->first;
  const double beta = st->beta;
  auto pv = [&](int64_t n) { return first ? z[n] : z[n] + beta * p_old[n]; };
  double v[1] = {0.0};
  FOR_OWN_CELLS(s) {
    const GCell c = gcell(g, s);
    const double ps = pv(s);
    const double qs = g_row(g, coef, M, c, s, pv);
    p[s] = ps;
    q[s] = qs;
    v[0] += ps * qs;
  }
  block_sum_k<kGT, 1>(v, red);
  double tot[1];
  if (grid_reduce_last_k<1>(v, partials, &st->ticket[1], tot, &flag, red) && threadIdx.x == 0) {
    if (g.dist) st->loc[kRedSearch] = tot[0];
    else fin_search(st, tot[0]);
  }
}

// x += alpha p, r -= alpha q, z = D^-1 r (or r), r.r and r.z (k_jacobi_step)
__global__ void __launch_bounds__(kGT) k_g_jacobi_step(GridParams g,
                                                      const double* __restrict__ dinv, double* x,
                                                      const double* __restrict__ p,
                                                      const double* __restrict__ q, double* r,
                                                      double* z, PcgState* st, double* partials,
                                                      double* history, int init, int defer) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  __shared__ double red[80];
  __shared__ int flag;
  const double alpha = st->alpha;
  double v[2] = {0.0, 0.0};
  FOR_OWN_CELLS(s) {
    double rv = r[s];
    if (!init) {
      x[s] = x[s] + alpha * p[s];
      rv = rv - alpha * q[s];
      r[s] = rv;
    }
    const double zv = dinv ? rv * dinv[s] : rv;
    if (!defer) z[s] = zv;
    v[0] += rv * rv;
    v[1] += rv * zv;
  }
  block_sum_k<kGT, 2>(v, red);
  double tot[2];
  if (grid_reduce_last_k<2>(v, partials, &st->ticket[4], tot, &flag, red) && threadIdx.x == 0) {
    if (defer) {
      if (g.dist) st->loc[kRedUpdate] = tot[0];
      else finish_rr(st, tot[0], history);
    } else if (g.dist) {
      st->loc[kRedJacobi] = tot[0];
      st->loc[kRedJacobi + 1] = tot[1];
    } else {
      fin_jacobi(st, tot[0], tot[1], init, history);
    }
  }
}

// t = r - A x (solver.cpp:285, 327)
__global__ void __launch_bounds__(kGT) k_g_resid(GridParams g, const double* __restrict__ coef,
                                                int64_t M, const double* __restrict__ r,
                                                const double* __restrict__ x, double* t,
                                                const PcgState* st) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  FOR_OWN_CELLS(s) {
    const GCell c = gcell(g, s);
    t[s] = r[s] - g_row(g, coef, M, c, s, [&](int64_t n) { return x[n]; });
  }
}

// r2 = r1 + R_c^T ec (solver.cpp:307-309)
__global__ void __launch_bounds__(kGT) k_g_prolong_add(GridParams g, const double* __restrict__ phi,
                                                      const double* __restrict__ r1,
                                                      const double* __restrict__ ec, double* r2,
                                                      const PcgState* st) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  const int64_t C = brick_cells(g);
  const int lc = g.lc;
  FOR_OWN_CELLS(s) {
    const int64_t b = s / C, l = s - b * C;
    double v = r1[s];
    for (int a = 0; a < lc; ++a) v = fma(phi[(b * lc + a) * C + l], ec[b * lc + a], v);
    r2[s] = v;
  }
}

// out = add + y; with rdot, rdot . out -> fin_post (k_add_finish)
__global__ void __launch_bounds__(kGT) k_g_add_finish(GridParams g, const double* __restrict__ y,
                                                     const double* __restrict__ add, double* out,
                                                     const double* __restrict__ rdot, PcgState* st,
                                                     double* partials, int init) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  __shared__ double red[80];
  __shared__ int flag;
  double v[1] = {0.0};
  FOR_OWN_CELLS(s) {
    const double o = add ? add[s] + y[s] : y[s];
    out[s] = o;
    if (rdot) v[0] += rdot[s] * o;
  }
  if (!rdot) return;
  block_sum_k<kGT, 1>(v, red);
  double tot[1];
  if (grid_reduce_last_k<1>(v, partials, &st->ticket[5], tot, &flag, red) && threadIdx.x == 0) {
    if (g.dist) st->loc[kRedPost] = tot[0];
    else fin_post(st, tot[0], init);
  }
}

// rc = R_c (r - A r1), one CTA per brick (solver.cpp:285-289)
__global__ void __launch_bounds__(kGT) k_g_restrict(GridParams g, const double* __restrict__ coef,
                                                   int64_t M, const double* __restrict__ phi,
                                                   const double* __restrict__ r,
                                                   const double* __restrict__ r1, double* rc,
                                                   const PcgState* st) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  __shared__ double red[80];
  const int64_t C = brick_cells(g), b = g.b0 + blockIdx.x;
  const int lc = g.lc;
  double v[kGLc] = {};
  for (int64_t l = threadIdx.x; l < C; l += blockDim.x) {
    const int64_t s = b * C + l;
    const GCell c = gcell(g, s);
    const double w = r[s] - g_row(g, coef, M, c, s, [&](int64_t n) { return r1[n]; });
#pragma unroll
    for (int a = 0; a < kGLc; ++a)
      if (a < lc) v[a] = fma(phi[(b * lc + a) * C + l], w, v[a]);
  }
  block_sum_k<kGT, kGLc>(v, red);
  if ((int)threadIdx.x < lc) rc[b * lc + threadIdx.x] = v[threadIdx.x];
}

// ------------------------------------------------------ A_c and Bc blocks
// Ac[b][dir][a][b'] = Phi_b^T A_{b,dir} Phi_dir and Bc[b] = Phi_b^T diag(e)
// Phi_b (e: faces leaving the cc element + Dirichlet terms): the definitions
// of k_coarse_blocks (coarse.cu), one CTA per brick, the blocks one at a time.
__global__ void __launch_bounds__(kGT) k_g_coarse_blocks(GridParams g,
                                                        const double* __restrict__ kappa,
                                                        const uint8_t* __restrict__ dmask,
                                                        const double* __restrict__ coef, int64_t M,
                                                        const double* __restrict__ phi, double* Ac,
                                                        double* Bc) {
  constexpr int K2 = kGLc * kGLc;
  __shared__ double red[K2 * (kGT / 32) + K2 + 8];
  const int64_t C = brick_cells(g), b = g.b0 + blockIdx.x;
  const int lc = g.lc;
  const int64_t bco[3] = {b % g.nbx, (b / g.nbx) % g.nby, b / (g.nbx * g.nby)};
  const int bd[3] = {g.bx, g.by, g.bz};
  const int st_in[3] = {1, g.bx, g.bx * g.by};
  auto ph = [&](int64_t bb, int a, int64_t l) { return phi[(bb * lc + a) * C + l]; };
  for (int pass = 0; pass < 8; ++pass) {
    double v[K2];
#pragma unroll
    for (int e = 0; e < K2; ++e) v[e] = 0.0;
    for (int64_t l = threadIdx.x; l < C; l += blockDim.x) {
      const int64_t s = b * C + l;
      const GCell c = gcell(g, s);
      const int co[3] = {c.li, c.lj, c.lk};
      double f[kGLc];
#pragma unroll
      for (int a = 0; a < kGLc; ++a) f[a] = a < lc ? ph(b, a, l) : 0.0;
      if (pass == 0) {  // self block: diag f f^T - sum over in-brick +axis faces
        const double d = coef[3 * M + s];
#pragma unroll
        for (int a = 0; a < kGLc; ++a)
#pragma unroll
          for (int bb = 0; bb < kGLc; ++bb) v[a * kGLc + bb] += d * f[a] * f[bb];
        for (int ax = 0; ax < 3; ++ax) {
          if (co[ax] + 1 >= bd[ax]) continue;
          const int64_t j = l + st_in[ax];
          const double T = coef[(size_t)ax * M + s];
          double fj[kGLc];
#pragma unroll
          for (int a = 0; a < kGLc; ++a) fj[a] = a < lc ? ph(b, a, j) : 0.0;
#pragma unroll
          for (int a = 0; a < kGLc; ++a)
#pragma unroll
            for (int bb = 0; bb < kGLc; ++bb)
              v[a * kGLc + bb] -= T * (f[a] * fj[bb] + fj[a] * f[bb]);
        }
      } else if (pass <= 6) {  // face block dir = pass: -T f_a(l) Phi_nb,b(l')
        const int fc = pass - 1, ax = fc >> 1;
        const bool hi = fc & 1;
        const bool on_face = hi ? co[ax] == bd[ax] - 1 : co[ax] == 0;
        if (!on_face) continue;
        const int64_t ns = gnbr(g, c, s, fc);
        if (ns < 0) continue;
        const double T = coef[(size_t)ax * M + (hi ? s : ns)];
        const int64_t nbb = ns / C, nl = ns - nbb * C;
#pragma unroll
        for (int bb = 0; bb < kGLc; ++bb) {
          const double pj = bb < lc ? ph(nbb, bb, nl) : 0.0;
#pragma unroll
          for (int a = 0; a < kGLc; ++a) v[a * kGLc + bb] += -T * f[a] * pj;
        }
      } else {  // Bc: faces crossing the cc-element boundary + Dirichlet faces
        double e = 0.0;
        const unsigned dm = dmask[s];
        for (int fc = 0; fc < 6; ++fc) {
          const int ax = fc >> 1;
          const bool hi = fc & 1;
          const bool on_face = hi ? co[ax] == bd[ax] - 1 : co[ax] == 0;
          if (!on_face) continue;
          const int64_t ns = gnbr(g, c, s, fc);
          if (ns >= 0) {
            const bool crosses = hi ? ((bco[ax] + 1) % g.sd == 0) : (bco[ax] % g.sd == 0);
            if (crosses) e += coef[(size_t)ax * M + (hi ? s : ns)];
          } else if (dm & (1u << fc)) {
            e += __dmul_rn(__dmul_rn(2.0, kappa[s]), g.cpl[ax]);
          }
        }
#pragma unroll
        for (int a = 0; a < kGLc; ++a)
#pragma unroll
          for (int bb = 0; bb < kGLc; ++bb) v[a * kGLc + bb] += e * f[a] * f[bb];
      }
    }
    block_sum_k<kGT, K2>(v, red);
    const int t = threadIdx.x;
    if (t < lc * lc) {
      const double val = v[(t / lc) * kGLc + t % lc];
      if (pass < 7) Ac[(b * 7 + pass) * lc * lc + t] = val;
      else Bc[b * lc * lc + t] = val;
    }
  }
}

// ------------------------------------------------------ local spectral bases
namespace {
constexpr int kEigK = 8;                  // subspace block
constexpr int kEigNP = kEigK * (kEigK + 1) / 2;

// Gram of the K-vector blocks A, B ([K][C] in global memory):
// g = (A^T B + B^T A) / 2 (same: A^T A). Symmetric, in gs (row-major K x K).
__device__ void gram_g(const double* A, const double* B, bool same, int64_t C, double* red,
                       double* gs) {
  double acc[kEigNP];
#pragma unroll
  for (int e = 0; e < kEigNP; ++e) acc[e] = 0.0;
  for (int64_t l = threadIdx.x; l < C; l += blockDim.x) {
    double a[kEigK], bv[kEigK];
#pragma unroll
    for (int k = 0; k < kEigK; ++k) {
      a[k] = A[k * C + l];
      bv[k] = same ? a[k] : B[k * C + l];
    }
    int e = 0;
#pragma unroll
    for (int i = 0; i < kEigK; ++i)
#pragma unroll
      for (int j = i; j < kEigK; ++j, ++e)
        acc[e] += same ? a[i] * a[j] : 0.5 * (a[i] * bv[j] + bv[i] * a[j]);
  }
  block_sum_k<kGT, kEigNP>(acc, red);
  if (threadIdx.x == 0) {
    int e = 0;
    for (int i = 0; i < kEigK; ++i)
      for (int j = i; j < kEigK; ++j, ++e) gs[i * kEigK + j] = gs[j * kEigK + i] = acc[e];
  }
  __syncthreads();
}

// y = B x for the K vectors, B = M^-1/2 S_loc M^-1/2 from the box's interior
// faces: TF[ax][l] = T between cell l and its +ax neighbour inside the box
// (0 at the box surface), SL = M^-1/2, SLL = sum of the cell's interior T's.
__device__ void bmatvec_g(const GridParams& g, const double* X, double* Y, const double* SL,
                          const double* SLL, const double* TF, int64_t C) {
  __syncthreads();
  const int st[3] = {1, g.bx, g.bx * g.by};
  for (int64_t l = threadIdx.x; l < C; l += blockDim.x) {
    const int co[3] = {(int)(l % g.bx), (int)((l / g.bx) % g.by), (int)(l / (g.bx * g.by))};
    const int bd[3] = {g.bx, g.by, g.bz};
    int64_t nb[6];
    double tf[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int ax = f >> 1;
      const bool hi = f & 1;
      const bool ex = hi ? co[ax] + 1 < bd[ax] : co[ax] > 0;
      nb[f] = ex ? (hi ? l + st[ax] : l - st[ax]) : -1;
      tf[f] = ex ? TF[ax * C + (hi ? l : l - st[ax])] : 0.0;
    }
    const double sl = SL[l], sll = SLL[l];
#pragma unroll
    for (int k = 0; k < kEigK; ++k) {
      double s = sll * (sl * X[k * C + l]);
#pragma unroll
      for (int f = 0; f < 6; ++f)
        if (nb[f] >= 0) s -= tf[f] * (SL[nb[f]] * X[k * C + nb[f]]);
      Y[k * C + l] = sl * s;
    }
  }
  __syncthreads();
}

// Cholesky G = R^T R by warp 0 into rsm (upper, row-major); false if G is
// not numerically positive definite (cholqr_apply of spectral.cu)
__device__ bool chol_g(const double* gs, double* rsm, int* okflag) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double a[kEigK];
#pragma unroll
    for (int i = 0; i < kEigK; ++i) a[i] = lane < kEigK ? gs[i * kEigK + lane] : 0.0;
    double gmax = lane < kEigK ? gs[lane * kEigK + lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    bool ok = true;
#pragma unroll
    for (int k = 0; k < kEigK; ++k) {
      const double d = __shfl_sync(0xffffffffu, a[k], k);
      ok = ok && (d > 1e-28 * gmax);
      const double rkk = ok ? sqrt(d) : 1.0;
      const double rkj = lane >= k && lane < kEigK ? a[k] / rkk : 0.0;
      if (lane < kEigK) rsm[k * kEigK + lane] = lane >= k ? rkj : 0.0;
#pragma unroll
      for (int i = k + 1; i < kEigK; ++i) {
        const double rki = __shfl_sync(0xffffffffu, rkj, i);
        if (lane > k) a[i] -= rki * rkj;
      }
    }
    if (lane == 0) *okflag = ok;
  }
  __syncthreads();
  return *okflag;
}
}  // namespace

// One CTA per brick (chunk [bfirst, bfirst + gridDim.x) of the owned bricks);
// scratch per CTA: X, Y, W [K][C], SL, SLL [C], TF [3][C].
__global__ void __launch_bounds__(kGT) k_g_local_basis(GridParams g,
                                                      const double* __restrict__ kappa,
                                                      const double* __restrict__ phi0, double* phi,
                                                      double* evals, int* iters_out, double tol,
                                                      int degree, int max_outer, double* scratch,
                                                      int64_t bfirst) {
  constexpr int K = kEigK;
  __shared__ double red[kEigNP * (kGT / 32) + kEigNP + 8];
  __shared__ double gs[K * K], qv[K * K], rsm[K * K], scal[K + 8];
  __shared__ int okflag, convflag;
  const int64_t C = brick_cells(g);
  const int64_t b = g.b0 + bfirst + blockIdx.x;
  double* X = scratch + (int64_t)blockIdx.x * (3 * K + 5) * C;
  double* Y = X + K * C;
  double* W = Y + K * C;
  double* SL = W + K * C;
  double* SLL = SL + C;
  double* TF = SLL + C;
  const int t = threadIdx.x;
  const int bd[3] = {g.bx, g.by, g.bz};
  const int st[3] = {1, g.bx, g.bx * g.by};
  // interior-face transmissibilities (box_interior_stiffness, coarse_space.cpp:238-277)
  for (int64_t l = t; l < C; l += blockDim.x) {
    const int co[3] = {(int)(l % g.bx), (int)((l / g.bx) % g.by), (int)(l / (g.bx * g.by))};
    const double kc = kappa[b * C + l];
    for (int ax = 0; ax < 3; ++ax)
      TF[ax * C + l] =
          co[ax] + 1 < bd[ax] ? face_t(kc, kappa[b * C + l + st[ax]]) * g.cpl[ax] : 0.0;
    SL[l] = 1.0 / sqrt(kc * g.vol);
  }
  __syncthreads();
  double gr = 0.0;
  for (int64_t l = t; l < C; l += blockDim.x) {
    const int co[3] = {(int)(l % g.bx), (int)((l / g.bx) % g.by), (int)(l / (g.bx * g.by))};
    double sll = 0.0, off = 0.0;
    for (int f = 0; f < 6; ++f) {
      const int ax = f >> 1;
      const bool hi = f & 1;
      if (hi ? co[ax] + 1 >= bd[ax] : co[ax] == 0) continue;
      const int64_t n = hi ? l + st[ax] : l - st[ax];
      const double T = TF[ax * C + (hi ? l : n)];
      sll += T;
      off += T * SL[n];
    }
    SLL[l] = sll;
    gr = fmax(gr, SL[l] * sll * SL[l] + SL[l] * off);  // Gershgorin bound of B
  }
  for (int o = 16; o > 0; o >>= 1) gr = fmax(gr, __shfl_xor_sync(0xffffffffu, gr, o));
  if ((t & 31) == 0) red[t >> 5] = gr;
  __syncthreads();
  if (t == 0) {
    double m = 0.0;
    for (int w = 0; w < kGT / 32; ++w) m = fmax(m, red[w]);
    scal[K] = m > 0.0 ? m : 1.0;
  }
  __syncthreads();
  const double bmax = scal[K];
  __syncthreads();
  constexpr int kWarmOuter = 20;
  double* theta = scal;  // Ritz values (shared, written by thread 0)
  int outer = 0, outer_total = 0;
  bool converged = false;
  for (int attempt = 0; attempt < (phi0 ? 2 : 1) && !converged; ++attempt) {
    const bool warm = phi0 && attempt == 0;
    for (int64_t l = t; l < C; l += blockDim.x) {
      const double sm_ = 1.0 / SL[l];  // sqrt(mass)
      X[l] = sm_;
      for (int k = 1; k < K; ++k) X[k * C + l] = hash_uniform(b, l, k);
      if (warm)
        for (int k = 0; k < g.lc && k < K; ++k) X[k * C + l] = sm_ * phi0[(b * g.lc + k) * C + l];
    }
    __syncthreads();
    double a_cut = 0.5 * bmax;
    const int outer_cap = warm && kWarmOuter < max_outer ? kWarmOuter : max_outer;
    for (outer = 0; outer <= outer_cap; ++outer) {
      // orthonormalise (CholQR twice)
      for (int pass = 0; pass < 2; ++pass) {
        gram_g(X, X, true, C, red, gs);
        const bool ok = chol_g(gs, rsm, &okflag);
#ifdef TMG_EIG_DEBUG
        if (t == 0 && blockIdx.x == 0 && !ok) printf("[eig b=%lld] outer %d pass %d rank loss\n", (long long)b, outer, pass);
#endif
        for (int64_t l = t; l < C; l += blockDim.x) {
          double x[K];
#pragma unroll
          for (int k = 0; k < K; ++k) x[k] = X[k * C + l];
          if (ok) {
#pragma unroll
            for (int j = 0; j < K; ++j) {
              double s = x[j];
#pragma unroll
              for (int k = 0; k < j; ++k) s -= x[k] * rsm[k * K + j];
              x[j] = s / rsm[j * K + j];
            }
          } else {  // rank loss: perturb the trailing vectors
#pragma unroll
            for (int k = 1; k < K; ++k) x[k] += 1e-3 * hash_uniform(b + 7777, l, k + 31 * outer);
          }
#pragma unroll
          for (int k = 0; k < K; ++k) X[k * C + l] = x[k];
        }
        __syncthreads();
      }
      // Rayleigh-Ritz
      bmatvec_g(g, X, Y, SL, SLL, TF, C);
      gram_g(X, Y, false, C, red, gs);
      if (t < 32) {
        warp_jacobi_small<K>(gs, rsm);
        if (t == 0) {
          int ord[K];
          for (int i = 0; i < K; ++i) ord[i] = i;
          for (int i = 0; i < K; ++i)
            for (int j = i + 1; j < K; ++j)
              if (gs[ord[j] * K + ord[j]] < gs[ord[i] * K + ord[i]]) {
                const int tmp = ord[i];
                ord[i] = ord[j];
                ord[j] = tmp;
              }
          for (int c = 0; c < K; ++c) {
            scal[c] = gs[ord[c] * K + ord[c]];
            for (int r = 0; r < K; ++r) qv[r * K + c] = rsm[r * K + ord[c]];
          }
        }
      }
      __syncthreads();
      // X <- X Q, Y <- Y Q; W = Y - X theta (residuals)
      for (int64_t l = t; l < C; l += blockDim.x) {
        double x[K], y[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          x[k] = X[k * C + l];
          y[k] = Y[k * C + l];
        }
#pragma unroll
        for (int c = 0; c < K; ++c) {
          double s = 0.0, s2 = 0.0;
#pragma unroll
          for (int r = 0; r < K; ++r) {
            s += x[r] * qv[r * K + c];
            s2 += y[r] * qv[r * K + c];
          }
          X[c * C + l] = s;
          Y[c * C + l] = s2;
          W[c * C + l] = s2 - theta[c] * s;
        }
      }
      __syncthreads();
      gram_g(W, W, true, C, red, gs);
      if (t == 0) {
        double w = 0.0;
        for (int c = 0; c < g.lc; ++c) w = fmax(w, sqrt(fmax(gs[c * K + c], 0.0)));
        scal[K + 1] = w;
        convflag = w <= tol * bmax;
      }
      __syncthreads();
#ifdef TMG_EIG_DEBUG
      const double worst = scal[K + 1];
      if (t == 0 && blockIdx.x == 0)
        printf("[eig b=%lld] outer %d worst/bmax %.3e bmax %.4e theta %.6e %.6e %.6e %.6e %.6e\n",
               (long long)b, outer, worst / bmax, bmax, theta[0], theta[1], theta[2], theta[3],
               theta[K - 1]);
#endif
      if (convflag) {
        converged = true;
        break;
      }
      if (outer == outer_cap) break;
      // Chebyshev filter damping [a_cut, bmax], normalised at 0 (spectral.cu)
      a_cut = fmin(fmax(theta[K - 1], 1e-6 * bmax), 0.95 * bmax);
      __syncthreads();  // every thread has read theta before the next Rayleigh-Ritz
      const double e = 0.5 * (bmax - a_cut), c0 = 0.5 * (bmax + a_cut);
      const double sigma1 = e / (0.0 - c0);
      const double gam = 2.0 / sigma1;
      double sigma = sigma1;
      // x0 = X, y = (B X - c0 X) sigma1 / e
      bmatvec_g(g, X, Y, SL, SLL, TF, C);
      for (int64_t i = t; i < K * C; i += blockDim.x) Y[i] = (Y[i] - c0 * X[i]) * (sigma1 / e);
      double* x0 = X;
      double* yg = Y;
      double* by = W;
      // degree: enough to damp the interval by ~1e6 relative to 0, no more
      // (a stronger filter collapses the block onto the lowest modes when the
      // wanted eigenvalues are not small against ||B||: boxes of a few dozen
      // cells); up to `degree`, and up to 1024 once three rounds have not
      // converged (a box whose wanted eigenvalues sit ~1e-5 ||B|| above 0,
      // where a degree-32 filter barely separates them)
      const int dcap = outer < 3 ? degree : 1024;
      const int dd = max(2, min(dcap, (int)ceil(acosh(1e6) / acosh(c0 / e))));
      for (int d = 2; d <= dd; ++d) {
        const double sig2 = 1.0 / (gam - sigma);
        bmatvec_g(g, yg, by, SL, SLL, TF, C);
        // ynew -> by's slot; x0 <- yg (by pointer rotation)
        for (int64_t i = t; i < K * C; i += blockDim.x)
          by[i] = (by[i] - c0 * yg[i]) * (2.0 * sig2 / e) - (sigma * sig2) * x0[i];
        double* tmp = x0;
        x0 = yg;
        yg = by;
        by = tmp;
        sigma = sig2;
      }
      __syncthreads();
      if (yg != X)
        for (int64_t i = t; i < K * C; i += blockDim.x) X[i] = yg[i];
      __syncthreads();
    }
    outer_total += outer;
  }
  // sign convention: sum of each basis vector >= 0; phi = M^-1/2 x
  double sg[K];
#pragma unroll
  for (int k = 0; k < K; ++k) sg[k] = 0.0;
  for (int64_t l = t; l < C; l += blockDim.x)
#pragma unroll
    for (int k = 0; k < K; ++k) sg[k] += X[k * C + l] * SL[l];
  block_sum_k<kGT, K>(sg, red);
  // Above dense_threshold (4096 cells) the reference's Lanczos path returns
  // the pairs in descending order (coarse_space.cpp:145-147 store the j-th
  // largest Ritz value of sigma I - B at count - 1 - j); R_c's rows follow it.
  const bool descending = C > 4096;
  for (int a = 0; a < g.lc; ++a) {
    const int src = descending ? g.lc - 1 - a : a;
    const double sgn = sg[src] < 0.0 ? -1.0 : 1.0;
    for (int64_t l = t; l < C; l += blockDim.x)
      phi[(b * g.lc + a) * C + l] = sgn * SL[l] * X[src * C + l];
  }
  if (t == 0) {
    for (int a = 0; a < g.lc; ++a) evals[b * g.lc + a] = theta[descending ? g.lc - 1 - a : a];
    iters_out[b] = converged ? outer_total : -outer_total - 1;
  }
}

// Boxes of fewer than kEigK cells: dense B (n x n) and cyclic Jacobi, one
// thread per brick.
__global__ void k_g_local_basis_tiny(GridParams g, const double* __restrict__ kappa, double* phi,
                                     double* evals, int* iters_out) {
  constexpr int NMAX = kEigK;
  const int64_t bl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (bl >= g.nbo) return;
  const int64_t b = g.b0 + bl;
  const int n = (int)brick_cells(g);
  double a[NMAX * NMAX], v[NMAX * NMAX], sl[NMAX];
  const int bd[3] = {g.bx, g.by, g.bz};
  const int st[3] = {1, g.bx, g.bx * g.by};
  for (int i = 0; i < n * n; ++i) a[i] = 0.0;
  for (int l = 0; l < n; ++l) sl[l] = 1.0 / sqrt(kappa[b * n + l] * g.vol);
  for (int l = 0; l < n; ++l) {
    const int co[3] = {l % g.bx, (l / g.bx) % g.by, l / (g.bx * g.by)};
    for (int ax = 0; ax < 3; ++ax) {
      if (co[ax] + 1 >= bd[ax]) continue;
      const int j = l + st[ax];
      const double T = face_t(kappa[b * n + l], kappa[b * n + j]) * g.cpl[ax];
      a[l * n + l] += T * sl[l] * sl[l];
      a[j * n + j] += T * sl[j] * sl[j];
      a[l * n + j] -= T * sl[l] * sl[j];
      a[j * n + l] -= T * sl[l] * sl[j];
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) v[i * n + j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n * n; ++i) {
      tot += a[i] * a[i];
      if (i / n != i % n) off += a[i] * a[i];
    }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (apq == 0.0) continue;
        const double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
        const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
        for (int k = 0; k < n; ++k) {
          const double akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = c * akp - s * akq;
          a[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = c * apk - s * aqk;
          a[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = c * vkp - s * vkq;
          v[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  int ord[NMAX];
  for (int i = 0; i < n; ++i) ord[i] = i;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (a[ord[j] * n + ord[j]] < a[ord[i] * n + ord[i]]) {
        const int tmp = ord[i];
        ord[i] = ord[j];
        ord[j] = tmp;
      }
  for (int c = 0; c < g.lc; ++c) {
    double sum = 0.0;
    for (int l = 0; l < n; ++l) sum += v[l * n + ord[c]] * sl[l];
    const double sgn = sum < 0.0 ? -1.0 : 1.0;
    for (int l = 0; l < n; ++l) phi[(b * g.lc + c) * n + l] = sgn * sl[l] * v[l * n + ord[c]];
    evals[b * g.lc + c] = a[ord[c] * n + ord[c]];
  }
  iters_out[b] = 0;
}

// ------------------------------------------------- exact box block solves
namespace {
struct BoxDims {
  int X, Y, Z;
};
__host__ __device__ __forceinline__ BoxDims box_dims(const GridParams& g, int kind) {
  return kind == 0 ? BoxDims{g.bx, g.by, g.bz}
                   : BoxDims{g.sd * g.bx, g.sd * g.by, g.sd * g.bz};
}
// slot of cell (i, j, k) of box `box` (kind 0: brick index, 1: cc element)
__device__ __forceinline__ int64_t box_slot(const GridParams& g, int kind, int64_t box, int i,
                                            int j, int k) {
  int64_t oi, oj, ok;
  if (kind == 0) {
    oi = (box % g.nbx) * g.bx;
    oj = ((box / g.nbx) % g.nby) * g.by;
    ok = (box / (g.nbx * g.nby)) * g.bz;
  } else {
    oi = (box % g.ncx) * g.sd * g.bx;
    oj = ((box / g.ncx) % g.ncy) * g.sd * g.by;
    ok = (box / (g.ncx * g.ncy)) * g.sd * g.bz;
  }
  return gslot(g, oi + i, oj + j, ok + k);
}
__host__ __device__ __forceinline__ int64_t box_first(const GridParams& g, int kind) { return kind == 0 ? g.b0 : g.e0; }
__host__ __device__ __forceinline__ int64_t box_count(const GridParams& g, int kind) { return kind == 0 ? g.nbo : g.neo; }
}  // namespace

// Plane k's matrix A_kk - D_k G_{k-1} D_k of boxes [c0, c0 + nc) (local
// indices; G_{k-1} already inverted in place). Plane-major storage
// G[k][box][P][P].
__global__ void __launch_bounds__(kGT) k_box_assemble(GridParams g, int kind,
                                                     const double* __restrict__ coef, int64_t M,
                                                     const double* __restrict__ Gp, double* Gk,
                                                     int k, int64_t c0, int64_t nc) {
  const BoxDims d = box_dims(g, kind);
  const int64_t P = (int64_t)d.X * d.Y, PP = P * P;
  const int64_t first = box_first(g, kind);
  for (int64_t idx = c0 * PP + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (c0 + nc) * PP;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bl = idx / PP, e = idx - bl * PP, box = first + bl;
    const int a = (int)(e / P), bcol = (int)(e % P);
    const int ia = a % d.X, ja = a / d.X, ib = bcol % d.X, jb = bcol / d.X;
    double v = 0.0;
    if (a == bcol) {
      v = coef[3 * M + box_slot(g, kind, box, ia, ja, k)];
    } else if (ja == jb && (ib == ia + 1 || ia == ib + 1)) {
      v = -coef[box_slot(g, kind, box, min(ia, ib), ja, k)];
    } else if (ia == ib && (jb == ja + 1 || ja == jb + 1)) {
      v = -coef[M + box_slot(g, kind, box, ia, min(ja, jb), k)];
    }
    if (k > 0) {
      const double da = coef[2 * M + box_slot(g, kind, box, ia, ja, k - 1)];
      const double db = coef[2 * M + box_slot(g, kind, box, ib, jb, k - 1)];
      v -= da * Gp[idx] * db;
    }
    Gk[idx] = v;
  }
}

// fold one batch's plane pivots into the per-box extrema (min pivot, max |pivot|)
__global__ void k_box_fold(const double* __restrict__ work, int64_t stride, int64_t off,
                           int64_t P, double* ext, int k, int64_t c0) {
  const int64_t bl = c0 + blockIdx.x;
  const double* piv = work + blockIdx.x * stride + off;
  __shared__ double rmn[32], rmx[32];
  double mn = 1e300, mx = 0.0;
  for (int64_t i = threadIdx.x; i < P; i += blockDim.x) {
    mn = fmin(mn, piv[i]);
    mx = fmax(mx, fabs(piv[i]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    rmn[threadIdx.x >> 5] = mn;
    rmx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      mn = fmin(mn, rmn[w]);
      mx = fmax(mx, rmx[w]);
    }
    if (k == 0) {
      ext[2 * bl] = mn;
      ext[2 * bl + 1] = mx;
    } else {
      ext[2 * bl] = fmin(ext[2 * bl], mn);
      ext[2 * bl + 1] = fmax(ext[2 * bl + 1], mx);
    }
  }
}

// the reference's singular-pivot rule over the whole block (solver.cpp:86-92)
__global__ void k_box_check(const double* __restrict__ ext, int64_t n, int* status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!(ext[2 * i] > 1e-14 * ext[2 * i + 1])) atomicExch(status, 1);
}

// One plane step of the block Thomas apply, grid (column slices of 64) x
// boxes on gridDim.x, 256 threads = 4 row groups x 64 columns; v (P values)
// in dynamic smem.
//   fwd: y_k = G_k (in_k + D_k y_{k-1})      -> ybuf plane k
//   bwd: x_k = y_k + G_k (D_{k+1} x_{k+1})   -> ybuf plane k
__global__ void __launch_bounds__(kGT) k_box_step(GridParams g, int kind,
                                                 const double* __restrict__ coef, int64_t M,
                                                 const double* __restrict__ G,
                                                 const double* __restrict__ in, double* ybuf,
                                                 const PcgState* st, int k, int bwd) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  extern __shared__ double vsm[];
  __shared__ double part[4][64];
  const BoxDims d = box_dims(g, kind);
  const int P = d.X * d.Y, t = threadIdx.x, nsl = (P + 63) / 64;
  const int64_t nb = box_count(g, kind), bl = blockIdx.x / nsl, box = box_first(g, kind) + bl;
  const int slice = (int)(blockIdx.x % nsl);
  for (int q = t; q < P; q += blockDim.x) {
    const int i = q % d.X, j = q / d.X;
    double val;
    if (!bwd) {
      val = in[box_slot(g, kind, box, i, j, k)];
      if (k > 0) {
        const int64_t sp = box_slot(g, kind, box, i, j, k - 1);
        val += coef[2 * M + sp] * ybuf[sp];
      }
    } else {
      val = coef[2 * M + box_slot(g, kind, box, i, j, k)] *
            ybuf[box_slot(g, kind, box, i, j, k + 1)];
    }
    vsm[q] = val;
  }
  __syncthreads();
  const int col = slice * 64 + (t & 63), rg = t >> 6;
  const int rows = (P + 3) / 4, q0 = rg * rows, q1 = min(P, q0 + rows);
  double s0 = 0.0, s1 = 0.0;
  if (col < P) {
    const double* Gk = G + ((size_t)k * nb + bl) * (size_t)P * P + col;
    int q = q0;
    for (; q + 1 < q1; q += 2) {
      s0 = fma(Gk[(size_t)q * P], vsm[q], s0);
      s1 = fma(Gk[(size_t)(q + 1) * P], vsm[q + 1], s1);
    }
    if (q < q1) s0 = fma(Gk[(size_t)q * P], vsm[q], s0);
  }
  part[rg][t & 63] = s0 + s1;
  __syncthreads();
  if (t < 64 && col < P) {
    const double tot = (part[0][t] + part[1][t]) + (part[2][t] + part[3][t]);
    const int64_t so = box_slot(g, kind, box, col % d.X, col / d.X, k);
    ybuf[so] = bwd ? ybuf[so] + tot : tot;
  }
}

// ---------------------------------------------------------------- launchers
void launch_g_coefficients(const GridParams& g, const double* kappa, const uint8_t* dmask,
                           double* coef, cudaStream_t s) {
  k_g_coefficients<<<cell_grid(g), kGT, 0, s>>>(g, kappa, dmask, coef, g.mst);
}
void launch_g_apply(const GridParams& g, const double* coef, const double* x, double* y,
                    double* dinv, int absval, cudaStream_t s) {
  k_g_apply<<<cell_grid(g), kGT, 0, s>>>(g, coef, g.mst, x, y, dinv, absval);
}
void launch_g_init(const GridParams& g, const double* coef, const double* b, double* x,
                   int has_x0, double* r, PcgState* st, double* partials, cudaStream_t s) {
  k_g_init<<<cell_grid(g), kGT, 0, s>>>(g, coef, g.mst, b, x, has_x0, r, st, partials);
}
void launch_g_search(const GridParams& g, const double* coef, const double* z, const double* p_old,
                     double* p, double* q, PcgState* st, double* partials, cudaStream_t s) {
  launch_pdl(k_g_search, dim3(cell_grid(g)), dim3(kGT), 0, s, g, coef, g.mst, z, p_old, p, q, st,
             partials);
}
void launch_g_jacobi_step(const GridParams& g, const double* dinv, double* x, const double* p,
                          const double* q, double* r, double* z, PcgState* st, double* partials,
                          double* history, int init, int defer, cudaStream_t s) {
  launch_pdl(k_g_jacobi_step, dim3(cell_grid(g)), dim3(kGT), 0, s, g, dinv, x, p, q, r, z, st,
             partials, history, init, defer);
}
void launch_g_resid(const GridParams& g, const double* coef, const double* r, const double* x,
                    double* t, const PcgState* st, cudaStream_t s) {
  launch_pdl(k_g_resid, dim3(cell_grid(g)), dim3(kGT), 0, s, g, coef, g.mst, r, x, t, st);
}
void launch_g_prolong_add(const GridParams& g, const double* phi, const double* r1,
                          const double* ec, double* r2, const PcgState* st, cudaStream_t s) {
  launch_pdl(k_g_prolong_add, dim3(cell_grid(g)), dim3(kGT), 0, s, g, phi, r1, ec, r2, st);
}
void launch_g_add_finish(const GridParams& g, const double* y, const double* add, double* out,
                         const double* rdot, PcgState* st, double* partials, int init,
                         cudaStream_t s) {
  launch_pdl(k_g_add_finish, dim3(cell_grid(g)), dim3(kGT), 0, s, g, y, add, out, rdot, st,
             partials, init);
}
void launch_g_restrict(const GridParams& g, const double* coef, const double* phi, const double* r,
                       const double* r1, double* rc, const PcgState* st, cudaStream_t s) {
  launch_pdl(k_g_restrict, dim3((unsigned)g.nbo), dim3(kGT), 0, s, g, coef, g.mst, phi, r, r1, rc,
             st);
}
void launch_g_coarse_blocks(const GridParams& g, const double* kappa, const uint8_t* dmask,
                            const double* coef, const double* phi, double* Ac, double* Bc,
                            cudaStream_t s) {
  k_g_coarse_blocks<<<(unsigned)g.nbo, kGT, 0, s>>>(g, kappa, dmask, coef, g.mst, phi, Ac, Bc);
}

// bricks per local-basis launch: scratch of (3 K + 5) C doubles per brick
// within kGenericScratchDoubles
constexpr int64_t kGenericScratchDoubles = 64LL << 20;  // 512 MB
int64_t g_local_basis_scratch_doubles(const GridParams& g) {
  const int64_t C = brick_cells(g);
  if (C < kEigK) return 0;
  const int64_t per = (3 * kEigK + 5) * C;
  const int64_t nb = std::max<int64_t>(1, std::min<int64_t>(g.nbo, kGenericScratchDoubles / per));
  return nb * per;
}
void launch_g_local_basis(const GridParams& g, const double* kappa, const double* phi0,
                          double* phi, double* evals, int* iters, double tol, int degree,
                          int max_outer, double* scratch, cudaStream_t s) {
  const int64_t C = brick_cells(g);
  if (C < kEigK) {
    k_g_local_basis_tiny<<<(unsigned)((g.nbo + 63) / 64), 64, 0, s>>>(g, kappa, phi, evals, iters);
    return;
  }
  const int64_t per = (3 * kEigK + 5) * C;
  const int64_t chunk = std::max<int64_t>(1, g_local_basis_scratch_doubles(g) / per);
  if (C > 4096) tol = std::min(tol, 1e-10);  // the Lanczos path's 1e-10 sigma (coarse_space.cpp:106)
  for (int64_t b0 = 0; b0 < g.nbo; b0 += chunk) {
    const int64_t n = std::min(chunk, g.nbo - b0);
    k_g_local_basis<<<(unsigned)n, kGT, 0, s>>>(g, kappa, phi0, phi, evals, iters, tol, degree,
                                                max_outer, scratch, b0);
  }
}

int64_t box_doubles(const GridParams& g, int kind) {
  const BoxDims d = box_dims(g, kind);
  const int64_t P = (int64_t)d.X * d.Y;
  return (int64_t)d.Z * P * P;
}
int box_plane_cells(const GridParams& g, int kind) {
  const BoxDims d = box_dims(g, kind);
  return d.X * d.Y;
}
int box_apply_kernels(const GridParams& g, int kind) { return 2 * box_dims(g, kind).Z; }

// boxes per batched inverse: the grid's z extent and a bounded work buffer
static int64_t box_batch(const GridParams& g, int kind) {
  const int64_t per = dense_inverse_work_doubles(box_plane_cells(g, kind));
  return std::max<int64_t>(1, std::min<int64_t>({box_count(g, kind), (int64_t)32768,
                                                 kGenericScratchDoubles / per}));
}
int64_t box_factor_work_doubles(const GridParams& g, int kind) {
  return box_batch(g, kind) * dense_inverse_work_doubles(box_plane_cells(g, kind)) +
         2 * box_count(g, kind);
}

void launch_box_factor(const GridParams& g, int kind, const double* coef, double* G, int* status,
                       double* work, cudaStream_t s) {
  const BoxDims d = box_dims(g, kind);
  const int64_t P = (int64_t)d.X * d.Y, nb = box_count(g, kind), batch = box_batch(g, kind);
  const int64_t wper = dense_inverse_work_doubles(P);
  double* ext = work + batch * wper;
  const int64_t plane = nb * P * P;
  for (int k = 0; k < d.Z; ++k) {
    double* Gk = G + k * plane;
    const double* Gp = k ? Gk - plane : nullptr;
    for (int64_t c0 = 0; c0 < nb; c0 += batch) {
      const int64_t nc = std::min(batch, nb - c0);
      const int64_t ent = nc * P * P;
      const unsigned grid = (unsigned)std::min<int64_t>((ent + kGT - 1) / kGT, 148 * 64);
      k_box_assemble<<<grid, kGT, 0, s>>>(g, kind, coef, g.mst, Gp, Gk, k, c0, nc);
      dense_spd_inverse_batched(Gk + c0 * P * P, P, nc, work, status, s);
      k_box_fold<<<(unsigned)nc, 256, 0, s>>>(work, wper, dense_inverse_pivots(work, P, 0) - work, P,
                                              ext, k, c0);
    }
  }
  k_box_check<<<(unsigned)std::min<int64_t>((nb + 255) / 256, 1024), 256, 0, s>>>(ext, nb, status);
}

void launch_box_apply(const GridParams& g, int kind, const double* coef, const double* G,
                      const double* in, const double* add, double* out, const double* rdot,
                      PcgState* st, double* partials, int init, double* ybuf, cudaStream_t s) {
  const BoxDims d = box_dims(g, kind);
  const int P = d.X * d.Y;
  const int64_t nb = box_count(g, kind);
  const dim3 grid((unsigned)(((P + 63) / 64) * nb));
  const size_t smem = sizeof(double) * (size_t)P;
  ensure_dyn_smem(k_box_step, smem);
  for (int k = 0; k < d.Z; ++k)
    launch_pdl(k_box_step, grid, dim3(kGT), smem, s, g, kind, coef, g.mst, G, in, ybuf,
               (const PcgState*)st, k, 0);
  for (int k = d.Z - 2; k >= 0; --k)
    launch_pdl(k_box_step, grid, dim3(kGT), smem, s, g, kind, coef, g.mst, G, in, ybuf,
               (const PcgState*)st, k, 1);
  launch_g_add_finish(g, ybuf, add, out, rdot, st, partials, init, s);
}

}  // namespace tmg
