// Fused PCG + V-cycle fine-level kernels (north_star items 1, 2, 3, 5).
//
// One PCG iteration of the reference (proj/core/src/solver.cpp:539-568) with
// the MultiscaleHierarchy::apply V-cycle (:272-334) is executed as
//   K1 search   p = z + beta p ; q = A p ; p.q            (grid reduction -> alpha)
//   K2 update   x += alpha p ; r -= alpha q ; r.r ;        (-> convergence test)
//               r1 = S(r)                (pre-smooth, exact per-coarse-cell solve)
//   K3 restrict rc = R_c (r - A r1)
//   coarse      rc0, rcc (k_coarse_down) ; ecc = A_cc^-1 rcc (GEMV) ; ec (k_coarse_up)
//   K4 post     r2 = r1 + R_c^T ec ; z = r2 + S(r - A r2) ; r.z  (-> beta)
// Every kernel is one CTA per brick, stages its brick (+ face halo) in shared
// memory, and reads the CG scalars from device memory; the CTA that finishes
// a grid reduction last computes alpha / beta / the stopping rule and flags
// `done`, after which every later kernel returns immediately. No host round
// trip is needed inside an iteration; the host only polls `done` between
// chunks of captured iterations.
#include "kernels.h"
#include "smoother.cuh"

namespace tmg {

constexpr int LCP = 4;  // compiled L_c (see coarse.cu)

__device__ __forceinline__ bool is_finite(double v) { return isfinite(v); }

// ------------------------------------------------------------------ K0 init
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_init(GridParams g, const double* __restrict__ kappa,
                                                      const uint8_t* __restrict__ dmask,
                                                      const double* __restrict__ b, double* x,
                                                      int has_x0, double* r, PcgState* st,
                                                      double* partials) {
  constexpr int C = CB * CB * CB;
  __shared__ double kt[Tile<CB>::N];
  __shared__ double xt[Tile<CB>::N];
  __shared__ double red[80];
  __shared__ int flag;
  const BrickCoord bc = brick_coord(g, blockIdx.x);
  const int t = threadIdx.x, li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
  const int64_t s = bc.b * C + t;
  const double bv = b[s];
  double rv;
  if (has_x0) {
    load_tile<CB, true>(kappa, kt, g, bc);
    load_tile<CB, true>(x, xt, g, bc);
    __syncthreads();
    const unsigned dm = brick_on_boundary(g, bc) ? dmask[s] : 0u;
    const FaceSet fs = cell_faces<CB>(kt, li, lj, lk, g, bc, dm);
    rv = bv - apply_row<CB>(fs, xt, li, lj, lk);
  } else {
    x[s] = 0.0;
    rv = bv;
  }
  r[s] = rv;
  double v[2] = {bv * bv, rv * rv};
  block_sum_k<C, 2>(v, red);
  double tot[2];
  if (grid_reduce_last_k<2>(v, partials, &st->ticket[0], tot, &flag, red) && t == 0) {
    const double bnorm = sqrt(tot[0]), rnorm = sqrt(tot[1]);
    st->bnorm = bnorm;
    st->rnorm = rnorm;
    st->it = 0;
    st->first = 0;
    if (bnorm == 0.0) {
      st->status = kStatusZeroRhs;
      st->done = 1;
    } else if (rnorm / bnorm <= st->rtol) {
      st->status = kStatusConverged;
      st->done = 1;
    } else {
      st->status = kStatusRunning;
      st->done = 0;
    }
  }
}

// --------------------------------------------------------------- K1 search
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_search(GridParams g, const double* __restrict__ kappa,
                                                        const uint8_t* __restrict__ dmask,
                                                        const double* __restrict__ z,
                                                        const double* __restrict__ p_old, double* p,
                                                        double* q, PcgState* st, double* partials) {
  // p_old and p are distinct buffers: neighbouring CTAs read p_old's halo while
  // this CTA writes the new search direction.
  if (st->done) return;
  constexpr int C = CB * CB * CB;
  __shared__ double kt[Tile<CB>::N];
  __shared__ double pt[Tile<CB>::N];
  __shared__ double zt[Tile<CB>::N];
  __shared__ double red[80];
  __shared__ int flag;
  const BrickCoord bc = brick_coord(g, blockIdx.x);
  const int t = threadIdx.x, li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
  const bool first = st->first;
  const double beta = st->beta;
  load_tile<CB, true>(kappa, kt, g, bc);
  load_tile<CB, true>(z, zt, g, bc);
  if (!first) load_tile<CB, true>(p_old, pt, g, bc);
  __syncthreads();
  // p = z + beta p over the whole tile (solver.cpp:565-567)
  for (int e = t; e < Tile<CB>::N; e += C) pt[e] = first ? zt[e] : zt[e] + beta * pt[e];
  __syncthreads();
  const int64_t s = bc.b * C + t;
  const unsigned dm = brick_on_boundary(g, bc) ? dmask[s] : 0u;
  const FaceSet fs = cell_faces<CB>(kt, li, lj, lk, g, bc, dm);
  const double pv = pt[Tile<CB>::idx(li, lj, lk)];
  const double qv = apply_row<CB>(fs, pt, li, lj, lk);
  p[s] = pv;
  q[s] = qv;
  double v[1] = {pv * qv};
  block_sum_k<C, 1>(v, red);
  double tot[1];
  if (grid_reduce_last_k<1>(v, partials, &st->ticket[1], tot, &flag, red) && t == 0) {
    const double pq = tot[0];
    st->pq = pq;
    st->first = 0;
    if (!(pq > 0.0)) {  // solver.cpp:541-548
      st->status = kStatusIndefinite;
      st->done = 1;
    } else {
      st->alpha = st->rho / pq;
    }
  }
}

// ------------------------------------------------- K2 update + pre-smooth
template <int CB>
__device__ __forceinline__ void finish_rr(PcgState* st, double rr, double* history) {
  const int it = st->it + 1;
  const double rel = sqrt(rr) / st->bnorm;
  st->it = it;
  st->rnorm = sqrt(rr);
  history[it - 1] = rel;
  if (!is_finite(rel)) {
    st->status = kStatusNonFinite;
    st->done = 1;
  } else if (rel <= st->rtol) {  // solver.cpp:557-560
    st->status = kStatusConverged;
    st->done = 1;
  } else if (it >= st->maxit) {
    st->status = kStatusMaxIt;
    st->done = 1;
  }
}

template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_update(GridParams g, const double* __restrict__ kappa,
                                                        const double* __restrict__ Gf, double* x,
                                                        const double* __restrict__ p,
                                                        const double* __restrict__ q, double* r,
                                                        double* r1, PcgState* st, double* partials,
                                                        double* history, int init) {
  if (st->done) return;
  constexpr int C = CB * CB * CB, P = CB * CB;
  extern __shared__ double sm[];
  double* tv = sm;            // C
  double* tz = tv + C;        // C
  double* u = tz + C;         // C
  double* xs = u + C;         // C
  double* w = xs + C;         // P
  double* gbuf = w + P;       // PP
  __shared__ double kb[C];
  __shared__ double red[80];
  __shared__ int flag;
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x, lk = t / (CB * CB);
  const int64_t s = b * C + t;
  double rv = r[s];
  if (!init) {
    const double alpha = st->alpha;
    x[s] = x[s] + alpha * p[s];  // solver.cpp:550-553
    rv = rv - alpha * q[s];
    r[s] = rv;
  }
  tv[t] = rv;
  kb[t] = kappa[s];
  __syncthreads();
  tz[t] = lk > 0 ? face_t(kb[t - P], kb[t]) * g.cpl[2] : 0.0;
  __syncthreads();
  thomas_solve<CB>(Gf + b * Thomas<CB>::PER_BRICK, tv, tz, u, xs, gbuf, w);
  r1[s] = xs[t];
  if (!init) {
    double v[1] = {rv * rv};
    block_sum_k<C, 1>(v, red);
    double tot[1];
    if (grid_reduce_last_k<1>(v, partials, &st->ticket[2], tot, &flag, red) && t == 0)
      finish_rr<CB>(st, tot[0], history);
  }
}

// ------------------------------------------------------------ K3 restrict
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_restrict(GridParams g, const double* __restrict__ kappa,
                                                          const uint8_t* __restrict__ dmask,
                                                          const double* __restrict__ phi,
                                                          const double* __restrict__ r,
                                                          const double* __restrict__ r1, double* rc,
                                                          const PcgState* st) {
  if (st->done) return;
  constexpr int C = CB * CB * CB;
  __shared__ double kt[Tile<CB>::N];
  __shared__ double xt[Tile<CB>::N];
  __shared__ double red[LCP * (C / 32) + LCP + 8];
  const BrickCoord bc = brick_coord(g, blockIdx.x);
  const int t = threadIdx.x, li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
  load_tile<CB, true>(kappa, kt, g, bc);
  load_tile<CB, true>(r1, xt, g, bc);
  __syncthreads();
  const int64_t s = bc.b * C + t;
  const unsigned dm = brick_on_boundary(g, bc) ? dmask[s] : 0u;
  const FaceSet fs = cell_faces<CB>(kt, li, lj, lk, g, bc, dm);
  const double wv = r[s] - apply_row<CB>(fs, xt, li, lj, lk);  // solver.cpp:285-288
  double v[LCP];
#pragma unroll
  for (int a = 0; a < LCP; ++a) v[a] = phi[(bc.b * LCP + a) * C + t] * wv;  // :289
  block_sum_k<C, LCP>(v, red);
  if (t < LCP) rc[bc.b * LCP + t] = v[t];
}

// ---------------------------------------------------------------- K4 post
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_post(GridParams g, const double* __restrict__ kappa,
                                                      const uint8_t* __restrict__ dmask,
                                                      const double* __restrict__ phi,
                                                      const double* __restrict__ Gf,
                                                      const double* __restrict__ r,
                                                      const double* __restrict__ r1,
                                                      const double* __restrict__ ec, double* z,
                                                      PcgState* st, double* partials, int init) {
  if (st->done) return;
  constexpr int C = CB * CB * CB, P = CB * CB, F = CB * CB;
  extern __shared__ double sm[];
  double* kt = sm;                      // tile
  double* r2 = kt + Tile<CB>::N;        // tile
  double* tv = r2 + Tile<CB>::N;        // C
  double* tz = tv + C;                  // C
  double* u = tz + C;                   // C
  double* xs = u + C;                   // C
  double* w = xs + C;                   // P
  double* gbuf = w + P;                 // PP
  __shared__ double red[80];
  __shared__ int flag;
  const BrickCoord bc = brick_coord(g, blockIdx.x);
  const int t = threadIdx.x, li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
  load_tile<CB, true>(kappa, kt, g, bc);
  // r2 = r1 + R_c^T ec over the brick and its face halo (solver.cpp:322-324)
  {
    const int64_t s = bc.b * C + t;
    double v = r1[s];
#pragma unroll
    for (int a = 0; a < LCP; ++a) v += phi[(bc.b * LCP + a) * C + t] * ec[bc.b * LCP + a];
    r2[Tile<CB>::idx(li, lj, lk)] = v;
    for (int hs = t; hs < 6 * F; hs += C) {
      const int f = hs / F, qq = hs % F;
      const int uu = qq % CB, ww = qq / CB;
      int64_t nbk = -1;
      int ni = 0, nj = 0, nk = 0, ti = 0, tj = 0, tk = 0;
      switch (f) {
        case 0: if (bc.bi > 0) nbk = bc.b - 1; ni = CB - 1; nj = uu; nk = ww; ti = -1; tj = uu; tk = ww; break;
        case 1: if (bc.bi + 1 < g.nbx) nbk = bc.b + 1; ni = 0; nj = uu; nk = ww; ti = CB; tj = uu; tk = ww; break;
        case 2: if (bc.bj > 0) nbk = bc.b - g.nbx; ni = uu; nj = CB - 1; nk = ww; ti = uu; tj = -1; tk = ww; break;
        case 3: if (bc.bj + 1 < g.nby) nbk = bc.b + g.nbx; ni = uu; nj = 0; nk = ww; ti = uu; tj = CB; tk = ww; break;
        case 4: if (bc.bk > 0) nbk = bc.b - g.nbx * g.nby; ni = uu; nj = ww; nk = CB - 1; ti = uu; tj = ww; tk = -1; break;
        default: if (bc.bk + 1 < g.nbz) nbk = bc.b + g.nbx * g.nby; ni = uu; nj = ww; nk = 0; ti = uu; tj = ww; tk = CB; break;
      }
      double hv = 0.0;
      if (nbk >= 0) {
        const int nl = ni + CB * (nj + CB * nk);
        hv = r1[nbk * C + nl];
#pragma unroll
        for (int a = 0; a < LCP; ++a) hv += phi[(nbk * LCP + a) * C + nl] * ec[nbk * LCP + a];
      }
      r2[Tile<CB>::idx(ti, tj, tk)] = hv;
    }
  }
  __syncthreads();
  const int64_t s = bc.b * C + t;
  const unsigned dm = brick_on_boundary(g, bc) ? dmask[s] : 0u;
  const FaceSet fs = cell_faces<CB>(kt, li, lj, lk, g, bc, dm);
  const double rv = r[s];
  tv[t] = rv - apply_row<CB>(fs, r2, li, lj, lk);  // solver.cpp:327-330
  tz[t] = lk > 0 ? fs.t[4] : 0.0;
  __syncthreads();
  thomas_solve<CB>(Gf + bc.b * Thomas<CB>::PER_BRICK, tv, tz, u, xs, gbuf, w);
  const double zv = r2[Tile<CB>::idx(li, lj, lk)] + xs[t];  // :331-333
  z[s] = zv;
  double v[1] = {rv * zv};
  block_sum_k<C, 1>(v, red);
  double tot[1];
  if (grid_reduce_last_k<1>(v, partials, &st->ticket[3], tot, &flag, red) && t == 0) {
    const double rz = tot[0];
    if (init) {
      st->rho = rz;  // solver.cpp:537
      st->beta = 0.0;
      st->first = 1;
    } else {
      st->beta = rz / st->rho;  // :562-564
      st->rho = rz;
    }
  }
}

// ---------------------------------------- Jacobi / identity preconditioner
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_jacobi_step(GridParams g, const double* __restrict__ dinv,
                                                             double* x, const double* __restrict__ p,
                                                             const double* __restrict__ q, double* r,
                                                             double* z, PcgState* st,
                                                             double* partials, double* history,
                                                             int init) {
  if (st->done) return;
  constexpr int C = CB * CB * CB;
  __shared__ double red[80];
  __shared__ int flag;
  const int t = threadIdx.x;
  const int64_t s = blockIdx.x * (int64_t)C + t;
  double rv = r[s];
  if (!init) {
    const double alpha = st->alpha;
    x[s] = x[s] + alpha * p[s];
    rv = rv - alpha * q[s];
    r[s] = rv;
  }
  const double zv = dinv ? rv * dinv[s] : rv;  // solver.cpp:35 / :18
  z[s] = zv;
  double v[2] = {rv * rv, rv * zv};
  block_sum_k<C, 2>(v, red);
  double tot[2];
  if (grid_reduce_last_k<2>(v, partials, &st->ticket[4], tot, &flag, red) && t == 0) {
    if (init) {
      st->rho = tot[1];
      st->beta = 0.0;
      st->first = 1;
    } else {
      finish_rr<CB>(st, tot[0], history);
      if (!st->done) {
        st->beta = tot[1] / st->rho;
        st->rho = tot[1];
      }
    }
  }
}

// ---------------------------------------------------------------- launchers

size_t update_smem(int cb) {
  const int C = cb * cb * cb, P = cb * cb, PP = P * (P + 1) / 2;
  return sizeof(double) * (size_t)(4 * C + P + PP);
}
size_t post_smem(int cb) {
  const int N = (cb + 2) * (cb + 2) * (cb + 2);
  return sizeof(double) * (size_t)(2 * N) + update_smem(cb);
}

template <int CB>
static void set_attrs() {
  cudaFuncSetAttribute(k_update<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)update_smem(CB));
  cudaFuncSetAttribute(k_post<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)post_smem(CB));
}

// Called once per context creation (outside any stream capture).
void init_kernel_attributes() {
  set_attrs<8>();
  set_attrs<4>();
}

void launch_init(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                 const double* b, double* x, int has_x0, double* r, PcgState* st, double* partials,
                 cudaStream_t s) {
  if (cb == 8) k_init<8><<<(unsigned)g.nb, 512, 0, s>>>(g, kappa, dmask, b, x, has_x0, r, st, partials);
  else k_init<4><<<(unsigned)g.nb, 64, 0, s>>>(g, kappa, dmask, b, x, has_x0, r, st, partials);
}
void launch_search(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                   const double* z, const double* p_old, double* p, double* q, PcgState* st,
                   double* partials, cudaStream_t s) {
  if (cb == 8) k_search<8><<<(unsigned)g.nb, 512, 0, s>>>(g, kappa, dmask, z, p_old, p, q, st, partials);
  else k_search<4><<<(unsigned)g.nb, 64, 0, s>>>(g, kappa, dmask, z, p_old, p, q, st, partials);
}
void launch_update(const GridParams& g, int cb, const double* kappa, const double* Gf, double* x,
                   const double* p, const double* q, double* r, double* r1, PcgState* st,
                   double* partials, double* history, int init, cudaStream_t s) {
  if (cb == 8) {
    k_update<8><<<(unsigned)g.nb, 512, update_smem(8), s>>>(g, kappa, Gf, x, p, q, r, r1, st, partials, history, init);
  } else {
    k_update<4><<<(unsigned)g.nb, 64, update_smem(4), s>>>(g, kappa, Gf, x, p, q, r, r1, st, partials, history, init);
  }
}
void launch_restrict(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                     const double* phi, const double* r, const double* r1, double* rc,
                     const PcgState* st, cudaStream_t s) {
  if (cb == 8) k_restrict<8><<<(unsigned)g.nb, 512, 0, s>>>(g, kappa, dmask, phi, r, r1, rc, st);
  else k_restrict<4><<<(unsigned)g.nb, 64, 0, s>>>(g, kappa, dmask, phi, r, r1, rc, st);
}
void launch_post(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                 const double* phi, const double* Gf, const double* r, const double* r1,
                 const double* ec, double* z, PcgState* st, double* partials, int init,
                 cudaStream_t s) {
  if (cb == 8) {
    k_post<8><<<(unsigned)g.nb, 512, post_smem(8), s>>>(g, kappa, dmask, phi, Gf, r, r1, ec, z, st, partials, init);
  } else {
    k_post<4><<<(unsigned)g.nb, 64, post_smem(4), s>>>(g, kappa, dmask, phi, Gf, r, r1, ec, z, st, partials, init);
  }
}
void launch_jacobi_step(const GridParams& g, int cb, const double* dinv, double* x, const double* p,
                        const double* q, double* r, double* z, PcgState* st, double* partials,
                        double* history, int init, cudaStream_t s) {
  if (cb == 8) k_jacobi_step<8><<<(unsigned)g.nb, 512, 0, s>>>(g, dinv, x, p, q, r, z, st, partials, history, init);
  else k_jacobi_step<4><<<(unsigned)g.nb, 64, 0, s>>>(g, dinv, x, p, q, r, z, st, partials, history, init);
}

}  // namespace tmg
