// Fused PCG + V-cycle fine-level kernels (north_star items 1, 2, 3, 5).
//
// One PCG iteration of the reference (proj/core/src/solver.cpp:539-568) with
// the MultiscaleHierarchy::apply V-cycle (:272-334) is executed as
//   K1 search   p = z + beta p ; q = A p ; p.q            (grid reduction -> alpha)
//   K2 update   x += alpha p ; r -= alpha q ; r.r ;        (-> convergence test)
//               r1 = S(r)                (pre-smooth, exact per-coarse-cell solve)
//   K3 restrict rc = R_c (r - A r1)
//   coarse      rc0, rcc ; ecc = A_cc^-1 rcc (GEMV) ; ec   (coarse.cu, dense.cu)
//   K4 post     r2 = r1 + R_c^T ec ; z = r2 + S(r - A r2) ; r.z  (-> beta)
// Every kernel is one CTA per brick, stages its brick (+ face halo) in shared
// memory, and reads the CG scalars from device memory; the CTA that finishes
// a grid reduction last computes alpha / beta / the stopping rule and flags
// `done`, after which every later kernel returns immediately. No host round
// trip is needed inside an iteration; the host only polls `done` between
// chunks of captured iterations.
#include <type_traits>

#include "kernels.h"
#include "pcg_fin.cuh"
#include "smoother.cuh"

namespace tmg {

// L_c (basis vectors per coarse cell) is a template parameter of the fine
// kernels that touch Phi: 1..kMaxLcFine, dispatched at launch (lc_dispatch).
constexpr int kMaxLcFine = 6;
template <typename F>
static void lc_dispatch(int lc, F&& f) {
  switch (lc) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 5: f(std::integral_constant<int, 5>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    default: throw std::runtime_error("L_c outside 1..6");
  }
}

// ------------------------------------------------------------ coefficients
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_coefficients(GridParams g,
                                                              const double* __restrict__ kappa,
                                                              const uint8_t* __restrict__ dmask,
                                                              double* coef, int64_t M) {
  constexpr int C = CB * CB * CB;
  __shared__ StencilSmem<CB> ss;
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  load_tile<CB, true>(kappa, ss.kt, g, bc);
  __syncthreads();
  tile_faces<CB>(ss.kt, ss.fx, ss.fy, ss.fz, g, bc);
  __syncthreads();
  const int t = threadIdx.x, li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
  const size_t s = bofs(bc.b, C) + t;
  const unsigned dm = brick_on_boundary(g, bc) ? dmask[s] : 0u;
  const FaceSet fs = cell_faces<CB>(ss.fx, ss.fy, ss.fz, ss.kt[Tile<CB>::idx(li, lj, lk)], li, lj,
                                    lk, g, bc, dm);
  coef[s] = (fs.nbmask & 2) ? fs.t[1] : 0.0;
  coef[M + s] = (fs.nbmask & 8) ? fs.t[3] : 0.0;
  coef[2 * M + s] = (fs.nbmask & 32) ? fs.t[5] : 0.0;
  coef[3 * M + s] = fs.diag;
}

__global__ void k_finalize(FinArgs a, int which, int init) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x != 0) return;
  if (which != kRedInit && a.st[0]->done) return;  // every slab holds the same flag
  const int nv = (which == kRedInit || which == kRedJacobi) ? 2 : 1;
  double tot[2] = {0.0, 0.0};
  for (int j = 0; j < a.ns; ++j)
    for (int v = 0; v < nv; ++v) tot[v] += a.st[j]->loc[which + v];
  for (int j = 0; j < a.ns; ++j) {
    PcgState* st = a.st[j];
    switch (which) {
      case kRedInit: fin_init(st, tot[0], tot[1]); break;
      case kRedSearch: fin_search(st, tot[0]); break;
      case kRedUpdate: finish_rr(st, tot[0], a.hist[j]); break;
      case kRedPost: fin_post(st, tot[0], init); break;
      default: fin_jacobi(st, tot[0], tot[1], init, a.hist[j]); break;
    }
  }
}

void launch_finalize(const FinArgs& a, int which, int init, cudaStream_t s) {
  launch_pdl(k_finalize, dim3(1), dim3(32), 0, s, a, which, init);
}

// Face-major T of every brick face slot (set-up): tf[b][f][q] = T of the face
// between face cell q of face f and the neighbour brick's cell, 0 on the
// domain boundary. The boundary-form kernels read these 6 CB^2 values
// coalesced instead of gathering one coefficient per 32-byte sector from the
// x faces (stride CB) and from the neighbours' coefficient arrays.
template <int CB>
__global__ void k_face_t(GridParams g, const double* __restrict__ coef, int64_t M, double* tf) {
  constexpr int C = CB * CB * CB, F = CB * CB;
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  const size_t ob = bofs(bc.b, C);
  for (int h = threadIdx.x; h < 6 * F; h += blockDim.x) {
    int f, ti, nl;
    halo_slot<CB>(h, f, ti, nl);
    const int nb = nbr_brick(g, bc, f);
    double v = 0.0;
    if (nb >= 0) {
      const int q = h % F, u = q % CB, w = q / CB, ax = f >> 1;
      const bool hi = f & 1;
      const int e = hi ? CB - 1 : 0;
      const int c = ax == 0 ? e + CB * (u + CB * w) : ax == 1 ? u + CB * (e + CB * w) : u + CB * (w + CB * e);
      v = coef[(size_t)ax * M + (hi ? ob + c : bofs(nb, C) + nl)];
    }
    tf[(size_t)bc.b * 6 * F + h] = v;
  }
}

// ------------------------------------------------------------------ K0 init
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_init(GridParams g, const double* __restrict__ coef,
                                                      int64_t M, const double* __restrict__ b,
                                                      double* x, int has_x0, double* r,
                                                      PcgState* st, double* partials) {
  constexpr int C = CB * CB * CB;
  __shared__ CoefSmem<CB> cs;
  __shared__ double xt[Tile<CB>::N];
  __shared__ double red[80];
  __shared__ int flag;
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  const int t = threadIdx.x, li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
  const size_t s = bofs(bc.b, C) + t;
  const double bv = b[s];
  double rv;
  if (has_x0) {
    load_coefs<CB>(coef, M, cs, g, bc);
    load_tile<CB, true>(x, xt, g, bc);
    __syncthreads();
    rv = bv - apply_coef<CB>(cs, xt, li, lj, lk);  // solver.cpp:518-521
  } else {
    x[s] = 0.0;
    rv = bv;
  }
  r[s] = rv;
  double v[2] = {bv * bv, rv * rv};
  block_sum_k<C, 2>(v, red);
  double tot[2];
  if (grid_reduce_last_k<2>(v, partials, &st->ticket[0], tot, &flag, red) && t == 0) {
    if (g.dist) {
      st->loc[kRedInit] = tot[0];
      st->loc[kRedInit + 1] = tot[1];
    } else {
      fin_init(st, tot[0], tot[1]);
    }
  }
}

// Grid sum of an iteration kernel's per-CTA partials (fixed order:
// thread-strided, warp tree, warps in sequence), then the scalar step of
// pcg() that follows it: `which` = kRedSearch (p.q -> alpha, solver.cpp:541-549),
// kRedUpdate (r.r -> stopping rule, :554-560) or kRedPost (r.z -> beta,
// :562-564). The producers end with their last store: no device-scope fence,
// no ticket, no CTA waiting to learn whether it was the last one. One CTA;
// with PDL it is resident while the producer drains.
__global__ void __launch_bounds__(1024) k_reduce_fin(const double* __restrict__ partials,
                                                     unsigned int n, PcgState* st, int dist,
                                                     int which, int init, double* history) {
  pdl_trigger();
  __shared__ double red[32];
  pdl_wait();
  if (st->done) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // four loads in flight per thread
  unsigned int i = threadIdx.x;
  for (; i + 3 * 1024 < n; i += 4 * 1024) {
    s0 += partials[i];
    s1 += partials[i + 1024];
    s2 += partials[i + 2 * 1024];
    s3 += partials[i + 3 * 1024];
  }
  for (; i < n; i += 1024) s0 += partials[i];
  double sum = (s0 + s1) + (s2 + s3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < 32; ++w) tot += red[w];
    if (dist) st->loc[which] = tot;
    else if (which == kRedSearch) fin_search(st, tot);
    else if (which == kRedUpdate) finish_rr(st, tot, history);
    else fin_post(st, tot, init);
  }
}

// CTA sum of v in a fixed order into partials[blockIdx.x] (for k_reduce_fin).
template <int NT>
__device__ __forceinline__ void cta_partial(double v, double* red, double* partials) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int w = 0; w < NT / 32; ++w) sum += red[w];
    partials[blockIdx.x] = sum;
  }
}

// --------------------------------------------------------------- K1 search
constexpr int kStencilThreads = 256;  // CTA size of the stencil kernels (2 cells/thread at CB = 8)

template <int CB>
#ifndef TMG_SEARCH_MINB
#define TMG_SEARCH_MINB 6
#endif
#ifndef TMG_FINE_DEFER  // 1: r.r / r.z of k_update / k_post_bnd summed by k_reduce_fin (no tickets)
#define TMG_FINE_DEFER 1
#endif
#ifndef TMG_SEARCH_DIAG  // 1: every brick reads the stored diagonal (A/B)
#define TMG_SEARCH_DIAG 0
#endif
#ifndef TMG_SEARCH_DEFER  // 1: p.q summed by k_reduce_fin instead of the last CTA (ticket)
#define TMG_SEARCH_DEFER 1
#endif
__global__ void __launch_bounds__(kStencilThreads, TMG_SEARCH_MINB) k_search(GridParams g, const double* __restrict__ coef,
                                                              int64_t M, const double* __restrict__ z,
                                                              const double* __restrict__ p_old, double* p,
                                                              double* q, PcgState* st, double* partials) {
  // p_old and p are distinct buffers: neighbouring CTAs read p_old's halo while
  // this CTA writes the new search direction.
  pdl_trigger();
  constexpr int C = CB * CB * CB, NT = kStencilThreads < C / 2 ? kStencilThreads : C / 2;
  constexpr int KPT = C / (2 * NT);  // x-adjacent cell pairs per thread
  __shared__ CoefSmem<CB> cs;
  __shared__ double pt[Tile<CB>::N];
  __shared__ double red[80];
  __shared__ int flag;
  const int t = threadIdx.x;
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  pdl_wait();
  if (st->done) return;
  const bool first = st->first;
  const double beta = st->beta;
  // coefficients + p = z + beta p over the tile (solver.cpp:565-567). Bricks
  // off the domain boundary (no Dirichlet faces; single-slab contexts) do not
  // read the diagonal: it is the sum of the six face coefficients (56 instead
  // of 64 B/cell).
  const bool with_dg = TMG_SEARCH_DIAG || g.dist || brick_on_boundary(g, bc);
  load_coefs_tile_axpy<CB, NT>(coef, M, cs, z, p_old, beta, first, pt, g, bc, with_dg);
  __syncthreads();
  double pq = 0.0;
  auto rows = [&](auto dgc) {
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const int c = 2 * (t + k * NT), li = c % CB, lj = (c / CB) % CB, lk = c / (CB * CB);
      const size_t s = bofs(bc.b, C) + c;
      const int ti = Tile<CB>::idx(li, lj, lk);
      const double2 pv = make_double2(pt[ti], pt[ti + 1]);
      const double2 qv = make_double2(apply_coef<CB, decltype(dgc)::value>(cs, pt, li, lj, lk),
                                      apply_coef<CB, decltype(dgc)::value>(cs, pt, li + 1, lj, lk));  // solver.cpp:540
      *reinterpret_cast<double2*>(p + s) = pv;
      *reinterpret_cast<double2*>(q + s) = qv;
      pq += pv.x * qv.x;
      pq += pv.y * qv.y;
    }
  };
  if (with_dg) rows(std::true_type{});
  else rows(std::false_type{});
#if TMG_SEARCH_DEFER
  cta_partial<NT>(pq, red, partials);  // the grid sum is k_reduce_fin's
#else
  double v[1] = {pq};
  block_sum_k<NT, 1>(v, red);
  double tot[1];
  if (grid_reduce_last_k<1>(v, partials, &st->ticket[1], tot, &flag, red) && t == 0) {
    if (g.dist) st->loc[kRedSearch] = tot[0];
    else fin_search(st, tot[0]);
  }
#endif
}

// K1 from the conductivity (opt-in, TMG_SEARCH_KAPPA=1; slower, abi.cu
// search()): the tile's face transmissibilities
// and diagonals are recomputed from kappa (8 B/cell, plus the Dirichlet bits
// on boundary bricks) with the expressions of k_coefficients instead of
// streaming the four coefficient arrays (32 B/cell), 40 instead of 64 B/cell;
// the faces (constant) are formed before the grid dependency wait. q is
// bitwise the q of k_search: the same coefficients, the row summed in the
// same order (apply_row / apply_coef differ only in the sign of a zero).
template <int CB>
__global__ void __launch_bounds__(kStencilThreads, TMG_SEARCH_MINB) k_search_kappa(
    GridParams g, const double* __restrict__ kappa, const uint8_t* __restrict__ dmask,
    const double* __restrict__ z, const double* __restrict__ p_old, double* p, double* q,
    PcgState* st, double* partials) {
  pdl_trigger();
  constexpr int C = CB * CB * CB, NT = kStencilThreads < C / 2 ? kStencilThreads : C / 2;
  constexpr int KPT = C / (2 * NT);  // x-adjacent cell pairs per thread
  __shared__ StencilSmem<CB> ss;
  __shared__ double pt[Tile<CB>::N];
  __shared__ double red[80];
  __shared__ int flag;
  const int t = threadIdx.x;
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  load_tile<CB, true>(kappa, ss.kt, g, bc);
  __syncthreads();
  tile_faces<CB>(ss.kt, ss.fx, ss.fy, ss.fz, g, bc);  // fvm.cpp:73-76, 91-94
  pdl_wait();
  if (st->done) return;
  const bool first = st->first;
  const double beta = st->beta;
  load_tile_axpy<CB>(z, p_old, beta, first, pt, g, bc);  // solver.cpp:565-567
  __syncthreads();
  const bool bnd = brick_on_boundary(g, bc);
  double pq = 0.0;
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int c = 2 * (t + k * NT), li = c % CB, lj = (c / CB) % CB, lk = c / (CB * CB);
    const size_t s = bofs(bc.b, C) + c;
    const int ti = Tile<CB>::idx(li, lj, lk);
    const unsigned dm0 = bnd ? dmask[s] : 0u, dm1 = bnd ? dmask[s + 1] : 0u;
    const FaceSet f0 = cell_faces<CB>(ss.fx, ss.fy, ss.fz, ss.kt[ti], li, lj, lk, g, bc, dm0);
    const FaceSet f1 = cell_faces<CB>(ss.fx, ss.fy, ss.fz, ss.kt[ti + 1], li + 1, lj, lk, g, bc, dm1);
    const double2 pv = make_double2(pt[ti], pt[ti + 1]);
    const double2 qv = make_double2(apply_row<CB>(f0, pt, li, lj, lk),
                                    apply_row<CB>(f1, pt, li + 1, lj, lk));  // solver.cpp:540
    *reinterpret_cast<double2*>(p + s) = pv;
    *reinterpret_cast<double2*>(q + s) = qv;
    pq += pv.x * qv.x;
    pq += pv.y * qv.y;
  }
  double v[1] = {pq};
  block_sum_k<NT, 1>(v, red);
  double tot[1];
  if (grid_reduce_last_k<1>(v, partials, &st->ticket[1], tot, &flag, red) && t == 0) {
    if (g.dist) st->loc[kRedSearch] = tot[0];
    else fin_search(st, tot[0]);
  }
}

// ------------------------------------------------- K2 update + pre-smooth
template <int CB>
struct UpdateSmem {
  double slots[kSlots][Thomas<CB>::PLANE];
  ThomasSmem<CB> th;
  double tv[CB * CB * CB];
  double tz[CB * CB * CB];
  double red[80];
  int flag;
};

// CTA size Thomas<CB>::NT (288 at CB = 8: one thread per mat-vec block row);
// brick cells are strided over the threads.
template <int CB>
__global__ void __launch_bounds__(Thomas<CB>::NT, 4) k_update(GridParams g, const double* __restrict__ coef,
                                                             int64_t M, const FineFactors Gf,
                                                             double* x, const double* __restrict__ p,
                                                             const double* __restrict__ q, double* r,
                                                             double* r1, double* r1f, PcgState* st,
                                                             double* partials, double* history, int init) {
  pdl_trigger();
  constexpr int C = CB * CB * CB, P = CB * CB, NT = Thomas<CB>::NT;
  extern __shared__ __align__(128) unsigned char smraw[];
  UpdateSmem<CB>& sm = *reinterpret_cast<UpdateSmem<CB>*>(smraw);
  const int b = (int)(blockIdx.x + g.b0);
  const GSlot gsl = Gf.map[b];
  // uniform bricks (slot < 0): no factor, fast diagonalisation (brick_inverse)
  const double* G = gsl.slot < 0 ? nullptr : Gf.G + (size_t)gsl.slot * Thomas<CB>::PER_BRICK;
  sm.th.slots = sm.slots;
  thomas_init<CB>(sm.th);
  __syncthreads();
  thomas_prefetch<CB>(sm.th, G);  // G is constant: stream it before the wait
  pdl_wait();
  if (st->done) {
    thomas_drain<CB>(sm.th, G);  // no bulk copy may land after the CTA exits
    return;
  }
  const int t = threadIdx.x;
  const double alpha = init ? 0.0 : st->alpha;
  double rr = 0.0;
  {
    // every global load of the thread's cells first, then the updates and
    // stores (x and r are read and written: in one rolled loop the stores
    // fence the next cell's loads and the brick pays one DRAM round trip per
    // NT cells)
    constexpr int KC = (C + NT - 1) / NT;
    double rv[KC], xv[KC], pv[KC], qv[KC], tzv[KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      const int c = t + k * NT, cc = c < C ? c : t;
      const size_t s = bofs(b, C) + cc;
      rv[k] = r[s];
      xv[k] = init ? 0.0 : x[s];
      pv[k] = init ? 0.0 : p[s];
      qv[k] = init ? 0.0 : q[s];
      tzv[k] = (G && cc >= P) ? __ldg(coef + 2 * M + s - P) : 0.0;  // T_z to the cell below
    }
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      const int c = t + k * NT;
      if (c < C) {
        const size_t s = bofs(b, C) + c;
        double v = rv[k];
        if (!init) {
          x[s] = xv[k] + alpha * pv[k];  // solver.cpp:550-553
          v = v - alpha * qv[k];
          r[s] = v;
          rr += v * v;
        }
        sm.tv[c] = v;
        sm.tz[c] = tzv[k];
      }
    }
  }
  brick_inverse<CB>(sm.th, G, sm.tv, sm.tz, gsl.scale, g);  // r1 = S(r), solver.cpp:280-281
  if (TMG_R1_FULL)
    for (int c = t; c < C; c += NT) r1[bofs(b, C) + c] = sm.tv[c];
  // the face layers of r1, face-major: all the boundary-form kernels read
  for (int h = t; h < 6 * P; h += NT) {
    const int f = h / P, q = h % P, u = q % CB, w = q / CB, ax = f >> 1, e = (f & 1) ? CB - 1 : 0;
    const int c = ax == 0 ? e + CB * (u + CB * w) : ax == 1 ? u + CB * (e + CB * w) : u + CB * (w + CB * e);
    r1f[(size_t)b * 6 * P + h] = sm.tv[c];
  }
  if (!init) {
#if TMG_FINE_DEFER
    cta_partial<NT>(rr, sm.red, partials);  // r.r and the stopping rule: k_reduce_fin
#else
    double v[1] = {rr};
    block_sum_k<NT, 1>(v, sm.red);
    double tot[1];
    if (grid_reduce_last_k<1>(v, partials, &st->ticket[2], tot, &sm.flag, sm.red) && t == 0) {
      if (g.dist) st->loc[kRedUpdate] = tot[0];
      else finish_rr(st, tot[0], history);  // :554-560
    }
#endif
  }
}

// ------------------------------------------------------------ K3 restrict
template <int CB, int LCP>
__global__ void __launch_bounds__(kStencilThreads, 6) k_restrict(GridParams g, const double* __restrict__ coef,
                                                                int64_t M, const double* __restrict__ phi,
                                                                const double* __restrict__ r,
                                                                const double* __restrict__ r1, double* rc,
                                                                const PcgState* st) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  constexpr int C = CB * CB * CB, NT = kStencilThreads < C ? kStencilThreads : C;
  constexpr int KPT = C / NT;
  __shared__ CoefSmem<CB> cs;
  __shared__ double xt[Tile<CB>::N];
  __shared__ double red[LCP * (NT / 32) + LCP + 8];
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  const int t = threadIdx.x;
  load_coefs<CB>(coef, M, cs, g, bc);
  load_tile<CB, true>(r1, xt, g, bc);
  double rv[KPT], ph[KPT][LCP];
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int c = t + k * NT;
    rv[k] = r[bofs(bc.b, C) + c];
#pragma unroll
    for (int a = 0; a < LCP; ++a) ph[k][a] = phi[((size_t)bc.b * LCP + a) * C + c];
  }
  __syncthreads();
  double v[LCP] = {};
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int c = t + k * NT, li = c % CB, lj = (c / CB) % CB, lk = c / (CB * CB);
    const double wv = rv[k] - apply_coef<CB>(cs, xt, li, lj, lk);  // solver.cpp:285-288
#pragma unroll
    for (int a = 0; a < LCP; ++a) v[a] = fma(ph[k][a], wv, v[a]);  // :289
  }
  block_sum_k<NT, LCP>(v, red);
  if (t < LCP) rc[(size_t)bc.b * LCP + t] = v[t];
}

// Boundary form of K3 for the default fine blocks (one exact block per brick).
// With r1_I = A_II^{-1} r_I, (r - A r1)_I = r_I - A_II r1_I - A_{I,nb} r1_nb
// = -A_{I,nb} r1_nb up to the rounding of the block solve: only the brick's
// surface cells carry a residual, T_f r1 across each face f (A's off-diagonal
// entries are -T). So rc_I = sum over the 6*CB^2 face slots of
// Phi_I(c_f) T_f r1_nb(f) — the same algebra as solver.cpp:285-289 without
// the brick's own r, r1 and the interior stencil (43% fewer bytes). Not valid
// for cc-element fine blocks, which keep k_restrict.
#ifndef TMG_RESTRICT_MINB
#define TMG_RESTRICT_MINB 8
#endif
template <int CB, int LCP>
__global__ void __launch_bounds__(CB == 8 ? kStencilThreads : 96, TMG_RESTRICT_MINB) k_restrict_bnd(
    GridParams g, const double* __restrict__ tfa, int64_t M, const double* __restrict__ phif,
    const double* __restrict__ r1f, double* rc, const PcgState* st) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  constexpr int C = CB * CB * CB, F = CB * CB, NS = 6 * F;
  constexpr int NT = kStencilThreads < NS ? kStencilThreads : NS;
  constexpr int KS = (NS + NT - 1) / NT;
  __shared__ double red[LCP * (NT / 32) + LCP + 8];
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  const int t = threadIdx.x;
  const size_t ob = bofs(bc.b, C);
  // every load of the thread's face slots first (unconditional, clamped
  // indices), then the products: one DRAM round trip per brick
  double tfv[KS], r1v[KS], phv[KS][LCP];
  bool ok[KS];
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    const int h = t + k * NT, hc = h < NS ? h : 0, f = hc / F, q = hc % F;
    const int nb = nbr_brick(g, bc, f);
    ok[k] = h < NS && nb >= 0;  // domain boundary: Dirichlet terms live in the diagonal
    tfv[k] = __ldg(tfa + (size_t)bc.b * 6 * F + hc);  // T of the face (face-major copy, k_face_t)
    r1v[k] = __ldg(r1f + ((size_t)(nb >= 0 ? nb : bc.b) * 6 + (f ^ 1)) * F + q);  // r1 on the neighbour's face
#pragma unroll
    for (int a = 0; a < LCP; ++a)  // own face f (face-major phif)
      phv[k][a] = __ldg(phif + (((size_t)bc.b * 6 + f) * LCP + a) * F + q);
  }
  double v[LCP] = {};
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    const double val = ok[k] ? tfv[k] * r1v[k] : 0.0;
#pragma unroll
    for (int a = 0; a < LCP; ++a) v[a] = fma(phv[k][a], val, v[a]);
  }
  block_sum_k<NT, LCP>(v, red);
#pragma unroll
  for (int a = 0; a < LCP; ++a)
    if (t == a) rc[(size_t)bc.b * LCP + a] = v[a];
}

// ---------------------------------------------------------------- K4 post
template <int CB>
struct PostSmem {
  union {  // stencil tiles are dead once the block solve starts streaming G
    double slots[kSlots][Thomas<CB>::PLANE];
    struct {
      CoefSmem<CB> cs;
      double r2[Tile<CB>::N];
    } st;
  } u;
  ThomasSmem<CB> th;
  double tv[CB * CB * CB];
  double tz[CB * CB * CB];
  double red[80];
  int flag;
};

template <int CB, int LCP>
__global__ void __launch_bounds__(Thomas<CB>::NT, 4) k_post(GridParams g, const double* __restrict__ coef,
                                                           const double* __restrict__ /*tfa*/,
                                                           int64_t M, const double* __restrict__ phi,
                                                           const FineFactors Gf,
                                                           const double* __restrict__ r,
                                                           const double* __restrict__ r1,
                                                           const double* __restrict__ ec, double* z,
                                                           PcgState* st, double* partials, int init) {
  pdl_trigger();
  constexpr int C = CB * CB * CB, NT = Thomas<CB>::NT;
  extern __shared__ __align__(128) unsigned char smraw[];
  PostSmem<CB>& sm = *reinterpret_cast<PostSmem<CB>*>(smraw);
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  const GSlot gsl = Gf.map[bc.b];
  // uniform bricks (slot < 0): no factor, fast diagonalisation (brick_inverse)
  const double* G = gsl.slot < 0 ? nullptr : Gf.G + (size_t)gsl.slot * Thomas<CB>::PER_BRICK;
  if (threadIdx.x == 0 && G)  // warm L2 with the first G planes (constant) before the wait
    prefetch_l2(G, (uint32_t)(2 * Thomas<CB>::PLANE * sizeof(double)));
  pdl_wait();
  if (st->done) return;
  sm.th.slots = sm.u.slots;
  thomas_init<CB>(sm.th);
  const int t = threadIdx.x;
  load_coefs<CB>(coef, M, sm.u.st.cs, g, bc);
  // r2 = r1 + R_c^T ec over the brick and its face halo (solver.cpp:322-324)
  {
    double ecb[LCP];
#pragma unroll
    for (int a = 0; a < LCP; ++a) ecb[a] = ec[(size_t)bc.b * LCP + a];
    for (int c = t; c < C; c += NT) {
      double v = r1[bofs(bc.b, C) + c];
#pragma unroll
      for (int a = 0; a < LCP; ++a) v += phi[((size_t)bc.b * LCP + a) * C + c] * ecb[a];
      sm.u.st.r2[Tile<CB>::idx(c % CB, (c / CB) % CB, c / (CB * CB))] = v;
    }
    for (int hs = t; hs < 6 * CB * CB; hs += NT) {
      int f, ti, nl;
      halo_slot<CB>(hs, f, ti, nl);
      const int nb = nbr_brick(g, bc, f);
      double hv = 0.0;
      if (nb >= 0) {
        hv = r1[bofs(nb, C) + nl];
#pragma unroll
        for (int a = 0; a < LCP; ++a) hv += phi[((size_t)nb * LCP + a) * C + nl] * ec[(size_t)nb * LCP + a];
      }
      sm.u.st.r2[ti] = hv;
    }
  }
  __syncthreads();
  constexpr int KPT = (C + NT - 1) / NT;  // cells per thread
  double r2own[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int c = t + k * NT;
    if (c < C) {
      const int li = c % CB, lj = (c / CB) % CB, lk = c / (CB * CB);
      r2own[k] = sm.u.st.r2[Tile<CB>::idx(li, lj, lk)];
      sm.tv[c] = r[bofs(bc.b, C) + c] - apply_coef<CB>(sm.u.st.cs, sm.u.st.r2, li, lj, lk);  // solver.cpp:327-330
      sm.tz[c] = lk > 0 ? coef_tz_below<CB>(sm.u.st.cs, c) : 0.0;
    }
  }
  __syncthreads();  // stencil tiles dead: the slots may now be filled
  thomas_prefetch<CB>(sm.th, G);
  brick_inverse<CB>(sm.th, G, sm.tv, sm.tz, gsl.scale, g);
  double rz = 0.0;
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int c = t + k * NT;
    if (c < C) {
      const size_t s = bofs(bc.b, C) + c;
      const double zv = r2own[k] + sm.tv[c];  // :331-333
      z[s] = zv;
      rz += r[s] * zv;
    }
  }
  double v[1] = {rz};
  block_sum_k<NT, 1>(v, sm.red);
  double tot[1];
  if (grid_reduce_last_k<1>(v, partials, &st->ticket[3], tot, &sm.flag, sm.red) && t == 0) {
    if (g.dist) st->loc[kRedPost] = tot[0];
    else fin_post(st, tot[0], init);
  }
}

// Boundary form of K4 for the default fine blocks (one exact block per brick).
// z = r2 + S(r - A r2) with r2 = r1 + R_c^T ec and r1_I = A_II^{-1} r_I gives
//   z_I = A_II^{-1} r_I - r2_I + r2_I + A_II^{-1} (-A_{I,nb} r2_nb)
//       = A_II^{-1} (r_I + t_I),   t_c = sum_{surface faces f of c} T_f r2_nb(f),
// the same algebra as solver.cpp:322-333 without the brick's own Phi, its
// coefficients and the interior stencil. r2 is needed on the face halo only
// (r1 + Phi ec of the neighbouring bricks). The shared memory no longer holds
// stencil tiles, so the first G planes stream from kernel entry.
template <int CB>
struct PostBSmem {
  double slots[kSlots][Thomas<CB>::PLANE];
  ThomasSmem<CB> th;
  double tv[CB * CB * CB];
  double tz[CB * CB * CB];
  double red[80];
  int flag;
};

template <int CB, int LCP>
__global__ void __launch_bounds__(Thomas<CB>::NT, 4) k_post_bnd(GridParams g, const double* __restrict__ coef,
                                                               const double* __restrict__ tfa,
                                                               int64_t M, const double* __restrict__ phif,
                                                               const FineFactors Gf,
                                                               const double* __restrict__ r,
                                                               const double* __restrict__ r1f,
                                                               const double* __restrict__ ec, double* z,
                                                               PcgState* st, double* partials, int init) {
  pdl_trigger();
  constexpr int C = CB * CB * CB, F = CB * CB, NT = Thomas<CB>::NT;
  extern __shared__ __align__(128) unsigned char smraw[];
  PostBSmem<CB>& sm = *reinterpret_cast<PostBSmem<CB>*>(smraw);
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  const GSlot gsl = Gf.map[bc.b];
  // uniform bricks (slot < 0): no factor, fast diagonalisation (brick_inverse)
  const double* G = gsl.slot < 0 ? nullptr : Gf.G + (size_t)gsl.slot * Thomas<CB>::PER_BRICK;
  sm.th.slots = sm.slots;
  thomas_init<CB>(sm.th);
  __syncthreads();
  thomas_prefetch<CB>(sm.th, G);  // G is constant: stream it before the wait
  pdl_wait();
  if (st->done) {
    thomas_drain<CB>(sm.th, G);
    return;
  }
  const int t = threadIdx.x;
  const size_t ob = bofs(bc.b, C);
  // surface terms T_f r2_nb(f), r2 = r1 + R_c^T ec on the halo (solver.cpp:
  // 322-324): every global load of the thread first -- unconditional, on
  // clamped indices, so none of them waits behind a branch or a dependent
  // FMA chain (one DRAM round trip per brick instead of one per face slot
  // and cell) -- then the arithmetic. The neighbours' ec go through shared
  // memory (24 values, sm.red is free until the final sum).
  constexpr int NS = 6 * F, KS = (NS + NT - 1) / NT, KC = (C + NT - 1) / NT;
  if (t < 6 * LCP) {
    const int nb = nbr_brick(g, bc, t / LCP);
    sm.red[t] = nb >= 0 ? __ldg(ec + (size_t)nb * LCP + t % LCP) : 0.0;
  }
  double r1v[KS], tfv[KS], phv[KS][LCP], rown[KC], tzv[KC];
  int face[KS];  // face of slot k, or -1: no neighbour / no slot
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    const int h = t + k * NT, hc = h < NS ? h : 0, f = hc / F, q = hc % F;
    const int nb = nbr_brick(g, bc, f);
    face[k] = (h < NS && nb >= 0) ? f : -1;
    const size_t fb = ((size_t)(nb >= 0 ? nb : bc.b) * 6 + (f ^ 1));  // the neighbour's face f^1 (face-major)
    r1v[k] = __ldg(r1f + fb * F + q);
#pragma unroll
    for (int a = 0; a < LCP; ++a) phv[k][a] = __ldg(phif + (fb * LCP + a) * F + q);
    tfv[k] = __ldg(tfa + (size_t)bc.b * 6 * F + hc);  // face-major T (k_face_t)
  }
  // z_I = A_II^{-1} (r_I + t_I) = r1_I + A_II^{-1} t_I: the solve takes r + t
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int c = t + k * NT, cc = c < C ? c : t;
    rown[k] = __ldg(r + ob + cc);
    tzv[k] = (G && cc >= F) ? __ldg(coef + 2 * M + ob + cc - F) : 0.0;  // T_z to the cell below
  }
  __syncthreads();  // ec of the six neighbours
  double val[KS];
  int cell[KS], axis[KS];
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    const int f = face[k] < 0 ? 0 : face[k], q = (t + k * NT) % F, u = q % CB, w = q / CB, ax = f >> 1;
    const int e = (f & 1) ? CB - 1 : 0;
    double r2 = r1v[k];
#pragma unroll
    for (int a = 0; a < LCP; ++a) r2 += phv[k][a] * sm.red[f * LCP + a];
    val[k] = face[k] < 0 ? 0.0 : tfv[k] * r2;
    axis[k] = face[k] < 0 ? -1 : ax;
    cell[k] = ax == 0 ? e + CB * (u + CB * w) : ax == 1 ? u + CB * (e + CB * w) : u + CB * (w + CB * e);
  }
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int c = t + k * NT;
    if (c < C) {
      sm.tv[c] = rown[k];
      sm.tz[c] = tzv[k];
    } else {
      rown[k] = 0.0;
    }
  }
  // t_c, one axis per pass (the two faces of a pass touch disjoint cells;
  // edge and corner cells sum x, then y, then z)
  for (int ax = 0; ax < 3; ++ax) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KS; ++k)
      if (axis[k] == ax) sm.tv[cell[k]] += val[k];
  }
  __syncthreads();  // the solve's first step reads plane 0 of t from other threads
  brick_inverse<CB>(sm.th, G, sm.tv, sm.tz, gsl.scale, g);  // z = A_II^{-1} (r + t), solver.cpp:331-333
  double rz = 0.0;
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int c = t + k * NT;
    if (c < C) {
      const double zv = sm.tv[c];
      z[ob + c] = zv;
      rz += rown[k] * zv;
    }
  }
#if TMG_FINE_DEFER
  cta_partial<NT>(rz, sm.red, partials);  // r.z and beta: k_reduce_fin
#else
  double v[1] = {rz};
  block_sum_k<NT, 1>(v, sm.red);
  double tot[1];
  if (grid_reduce_last_k<1>(v, partials, &st->ticket[3], tot, &sm.flag, sm.red) && t == 0) {
    if (g.dist) st->loc[kRedPost] = tot[0];
    else fin_post(st, tot[0], init);
  }
#endif
}

// --------------------------------- generic block solve (nu != 1 V-cycles)
// out = add + A_II^{-1} in on every owned brick (add nullable, may alias
// out); with rdot, rdot . out is reduced and finishes the iteration like K4
// (fin_post). One smoother sweep z += S (r - A z) of BlockJacobiSmoother
// (solver.cpp:221-243) for the per-coarse-cell blocks, composed with k_resid
// by the generic V-cycle (abi.cu enqueue_vcycle_nu).
template <int CB>
__global__ void __launch_bounds__(Thomas<CB>::NT, 4) k_brick_solve(GridParams g,
                                                                  const double* __restrict__ coef,
                                                                  int64_t M,
                                                                  const FineFactors Gf,
                                                                  const double* __restrict__ in,
                                                                  const double* add, double* out,
                                                                  const double* __restrict__ rdot,
                                                                  PcgState* st, double* partials,
                                                                  int init) {
  pdl_trigger();
  constexpr int C = CB * CB * CB, P = CB * CB, NT = Thomas<CB>::NT;
  extern __shared__ __align__(128) unsigned char smraw[];
  UpdateSmem<CB>& sm = *reinterpret_cast<UpdateSmem<CB>*>(smraw);
  const int b = (int)(blockIdx.x + g.b0);
  const GSlot gsl = Gf.map[b];
  // uniform bricks (slot < 0): no factor, fast diagonalisation (brick_inverse)
  const double* G = gsl.slot < 0 ? nullptr : Gf.G + (size_t)gsl.slot * Thomas<CB>::PER_BRICK;
  sm.th.slots = sm.slots;
  thomas_init<CB>(sm.th);
  __syncthreads();
  thomas_prefetch<CB>(sm.th, G);
  pdl_wait();
  if (st->done) {
    thomas_drain<CB>(sm.th, G);
    return;
  }
  const int t = threadIdx.x;
  for (int c = t; c < C; c += NT) {
    const size_t s = bofs(b, C) + c;
    sm.tv[c] = in[s];
    sm.tz[c] = c >= P ? __ldg(coef + 2 * M + s - P) : 0.0;  // T_z to the cell below
  }
  __syncthreads();
  brick_inverse<CB>(sm.th, G, sm.tv, sm.tz, gsl.scale, g);
  double rz = 0.0;
  for (int c = t; c < C; c += NT) {
    const size_t s = bofs(b, C) + c;
    const double o = add ? add[s] + sm.tv[c] : sm.tv[c];
    out[s] = o;
    if (rdot) rz += rdot[s] * o;
  }
  if (!rdot) return;
  double v[1] = {rz};
  block_sum_k<NT, 1>(v, sm.red);
  double tot[1];
  if (grid_reduce_last_k<1>(v, partials, &st->ticket[3], tot, &sm.flag, sm.red) && t == 0) {
    if (g.dist) st->loc[kRedPost] = tot[0];
    else fin_post(st, tot[0], init);
  }
}

// ---------------------------------------- Jacobi / identity preconditioner
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_jacobi_step(GridParams g, const double* __restrict__ dinv,
                                                             double* x, const double* __restrict__ p,
                                                             const double* __restrict__ q, double* r,
                                                             double* z, PcgState* st,
                                                             double* partials, double* history,
                                                             int init, int defer) {
  pdl_trigger();
  pdl_wait();
  if (st->done) return;
  constexpr int C = CB * CB * CB;
  __shared__ double red[80];
  __shared__ int flag;
  const int t = threadIdx.x;
  const size_t s = bofs((int)(blockIdx.x + g.b0), C) + t;
  double rv = r[s];
  if (!init) {
    const double alpha = st->alpha;
    x[s] = x[s] + alpha * p[s];
    rv = rv - alpha * q[s];
    r[s] = rv;
  }
  const double zv = dinv ? rv * dinv[s] : rv;  // solver.cpp:35 / :18
  if (!defer) z[s] = zv;  // defer: the block solve (block_jacobi.cu) writes z
  double v[2] = {rv * rv, rv * zv};
  block_sum_k<C, 2>(v, red);
  double tot[2];
  if (grid_reduce_last_k<2>(v, partials, &st->ticket[4], tot, &flag, red) && t == 0) {
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

// ---------------------------------------------------------------- launchers

// Grid for a persistent kernel: every resident CTA slot of every SM, capped
// at the number of bricks.
template <typename K>
static unsigned persist_grid(K kernel, int threads, size_t smem, int64_t nb) {
  const int64_t n = (int64_t)device_sm_count() * device_occupancy(kernel, threads, smem);
  return (unsigned)(n < nb ? n : nb);
}

size_t update_smem(int cb) { return cb == 8 ? sizeof(UpdateSmem<8>) : sizeof(UpdateSmem<4>); }
#ifndef TMG_POST_BND
#define TMG_POST_BND 1
#endif
#if TMG_POST_BND
#define K_POST k_post_bnd
size_t post_smem(int cb) { return cb == 8 ? sizeof(PostBSmem<8>) : sizeof(PostBSmem<4>); }
#else
#define K_POST k_post
size_t post_smem(int cb) { return cb == 8 ? sizeof(PostSmem<8>) : sizeof(PostSmem<4>); }
#endif

template <int CB>
static void set_attrs() {
  cudaFuncSetAttribute(k_update<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)update_smem(CB));
  cudaFuncSetAttribute(k_brick_solve<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)update_smem(CB));
  for (int lc = 1; lc <= kMaxLcFine; ++lc)
    lc_dispatch(lc, [](auto L) {
      cudaFuncSetAttribute(K_POST<CB, decltype(L)::value>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)post_smem(CB));
    });
}

// Called once per context creation (outside any stream capture).
void init_kernel_attributes() {
  set_attrs<8>();
  set_attrs<4>();
}

void launch_coefficients(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                         double* coef, cudaStream_t s) {
  const int64_t M = g.mst;
  if (cb == 0) return launch_g_coefficients(g, kappa, dmask, coef, s);
  if (cb == 8) k_coefficients<8><<<(unsigned)g.nbo, 512, 0, s>>>(g, kappa, dmask, coef, M);
  else k_coefficients<4><<<(unsigned)g.nbo, 64, 0, s>>>(g, kappa, dmask, coef, M);
}
void launch_brick_solve(const GridParams& g, int cb, const double* coef, const FineFactors& Gf,
                        const double* in, const double* add, double* out, const double* rdot,
                        PcgState* st, double* partials, int init, cudaStream_t s) {
  const int64_t M = g.mst;
  if (cb == 8)
    launch_pdl(k_brick_solve<8>, dim3((unsigned)g.nbo), dim3(Thomas<8>::NT), update_smem(cb), s, g,
               coef, M, Gf, in, add, out, rdot, st, partials, init);
  else
    launch_pdl(k_brick_solve<4>, dim3((unsigned)g.nbo), dim3(Thomas<4>::NT), update_smem(cb), s, g,
               coef, M, Gf, in, add, out, rdot, st, partials, init);
}
void launch_face_t(const GridParams& g, int cb, const double* coef, double* tf, cudaStream_t s) {
  const int64_t M = g.mst;
  if (cb == 8) k_face_t<8><<<(unsigned)g.nbo, 384, 0, s>>>(g, coef, M, tf);
  else k_face_t<4><<<(unsigned)g.nbo, 96, 0, s>>>(g, coef, M, tf);
}
void launch_init(const GridParams& g, int cb, const double* coef, const double* b, double* x,
                 int has_x0, double* r, PcgState* st, double* partials, cudaStream_t s) {
  const int64_t M = g.mst;
  if (cb == 0) return launch_g_init(g, coef, b, x, has_x0, r, st, partials, s);
  if (cb == 8) k_init<8><<<(unsigned)g.nbo, 512, 0, s>>>(g, coef, M, b, x, has_x0, r, st, partials);
  else k_init<4><<<(unsigned)g.nbo, 64, 0, s>>>(g, coef, M, b, x, has_x0, r, st, partials);
}
void launch_search(const GridParams& g, int cb, const double* coef, const double* z,
                   const double* p_old, double* p, double* q, PcgState* st, double* partials,
                   cudaStream_t s) {
  const int64_t M = g.mst;
  if (cb == 0) return launch_g_search(g, coef, z, p_old, p, q, st, partials, s);
  if (cb == 8) launch_pdl(k_search<8>, dim3((unsigned)g.nbo), dim3(kStencilThreads), 0, s, g, coef, M, z, p_old, p, q, st, partials);
  else launch_pdl(k_search<4>, dim3((unsigned)g.nbo), dim3(32), 0, s, g, coef, M, z, p_old, p, q, st, partials);
#if TMG_SEARCH_DEFER
  launch_pdl(k_reduce_fin, dim3(1), dim3(1024), 0, s, (const double*)partials, (unsigned int)g.nbo, st,
             (int)g.dist, (int)kRedSearch, 0, (double*)nullptr);
#endif
}
int search_kernels(int cb) { return cb != 0 && TMG_SEARCH_DEFER ? 2 : 1; }
void launch_search_kappa(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                         const double* z, const double* p_old, double* p, double* q, PcgState* st,
                         double* partials, cudaStream_t s) {
  if (cb == 8) launch_pdl(k_search_kappa<8>, dim3((unsigned)g.nbo), dim3(kStencilThreads), 0, s, g, kappa, dmask, z, p_old, p, q, st, partials);
  else launch_pdl(k_search_kappa<4>, dim3((unsigned)g.nbo), dim3(32), 0, s, g, kappa, dmask, z, p_old, p, q, st, partials);
}
int launch_update(const GridParams& g, int cb, const double* coef, const FineFactors& Gf, double* x,
                  const double* p, const double* q, double* r, double* r1, double* r1f, PcgState* st,
                  double* partials, double* history, int init, cudaStream_t s) {
  const int64_t M = g.mst;
  if (cb == 8) launch_pdl(k_update<8>, dim3((unsigned)g.nbo), dim3(Thomas<8>::NT), update_smem(cb), s, g, coef, M, Gf, x, p, q, r, r1, r1f, st, partials, history, init);
  else launch_pdl(k_update<4>, dim3((unsigned)g.nbo), dim3(Thomas<4>::NT), update_smem(cb), s, g, coef, M, Gf, x, p, q, r, r1, r1f, st, partials, history, init);
  if (!TMG_FINE_DEFER || init) return 1;
  launch_pdl(k_reduce_fin, dim3(1), dim3(1024), 0, s, (const double*)partials, (unsigned int)g.nbo, st,
             (int)g.dist, (int)kRedUpdate, 0, history);
  return 2;
}
void launch_restrict(const GridParams& g, int cb, const double* coef, const double* phi,
                     const double* r, const double* r1, double* rc, const PcgState* st,
                     cudaStream_t s) {
  const int64_t M = g.mst;
  if (cb == 0) return launch_g_restrict(g, coef, phi, r, r1, rc, st, s);
  lc_dispatch(g.lc, [&](auto L) {
    constexpr int LCP = decltype(L)::value;
    if (cb == 8) launch_pdl(k_restrict<8, LCP>, dim3((unsigned)g.nbo), dim3(kStencilThreads), 0, s, g, coef, M, phi, r, r1, rc, st);
    else launch_pdl(k_restrict<4, LCP>, dim3((unsigned)g.nbo), dim3(64), 0, s, g, coef, M, phi, r, r1, rc, st);
  });
}
void launch_restrict_bnd(const GridParams& g, int cb, const double* tf, const double* phif,
                         const double* r1f, double* rc, const PcgState* st, cudaStream_t s) {
  const int64_t M = g.mst;
  lc_dispatch(g.lc, [&](auto L) {
    constexpr int LCP = decltype(L)::value;
    if (cb == 8) launch_pdl(k_restrict_bnd<8, LCP>, dim3((unsigned)g.nbo), dim3(kStencilThreads), 0, s, g, tf, M, phif, r1f, rc, st);
    else launch_pdl(k_restrict_bnd<4, LCP>, dim3((unsigned)g.nbo), dim3(96), 0, s, g, tf, M, phif, r1f, rc, st);
  });
}

// Face-major copy of Phi for the boundary-form kernels: their Phi reads are
// whole 16-byte-coalesced face rows instead of stride-CB columns (x faces).
template <int CB, int LCP>
__global__ void __launch_bounds__(256) k_phi_faces(const double* __restrict__ phi, double* phif, int64_t b0) {
  constexpr int C = CB * CB * CB, F = CB * CB;
  const int64_t b = b0 + blockIdx.x;
  for (int i = threadIdx.x; i < 6 * LCP * F; i += blockDim.x) {
    const int f = i / (LCP * F), a = (i / F) % LCP, q = i % F, u = q % CB, w = q / CB, ax = f >> 1;
    const int e = (f & 1) ? CB - 1 : 0;
    const int c = ax == 0 ? e + CB * (u + CB * w) : ax == 1 ? u + CB * (e + CB * w) : u + CB * (w + CB * e);
    phif[(b * 6 + f) * LCP * F + a * F + q] = phi[(b * LCP + a) * C + c];
  }
}
void launch_phi_faces(const GridParams& g, int cb, const double* phi, double* phif, int64_t b0,
                      int64_t nb, cudaStream_t s) {
  lc_dispatch(g.lc, [&](auto L) {
    constexpr int LCP = decltype(L)::value;
    if (cb == 8) k_phi_faces<8, LCP><<<(unsigned)nb, 256, 0, s>>>(phi, phif, b0);
    else k_phi_faces<4, LCP><<<(unsigned)nb, 256, 0, s>>>(phi, phif, b0);
  });
}
int launch_post(const GridParams& g, int cb, const double* coef, const double* tf,
                const double* phi_full, const double* phif, const FineFactors& Gf, const double* r,
                const double* r1_full, const double* r1f, const double* ec, double* z, PcgState* st,
                double* partials, int init, cudaStream_t s) {
  const int64_t M = g.mst;
  const double* phi = TMG_POST_BND ? phif : phi_full;
  const double* r1 = TMG_POST_BND ? r1f : r1_full;
  lc_dispatch(g.lc, [&](auto L) {
    constexpr int LCP = decltype(L)::value;
    if (cb == 8) launch_pdl(K_POST<8, LCP>, dim3((unsigned)g.nbo), dim3(Thomas<8>::NT), post_smem(cb), s, g, coef, tf, M, phi, Gf, r, r1, ec, z, st, partials, init);
    else launch_pdl(K_POST<4, LCP>, dim3((unsigned)g.nbo), dim3(Thomas<4>::NT), post_smem(cb), s, g, coef, tf, M, phi, Gf, r, r1, ec, z, st, partials, init);
  });
  if (!(TMG_FINE_DEFER && TMG_POST_BND)) return 1;  // the literal k_post keeps its ticket
  launch_pdl(k_reduce_fin, dim3(1), dim3(1024), 0, s, (const double*)partials, (unsigned int)g.nbo, st,
             (int)g.dist, (int)kRedPost, init, (double*)nullptr);
  return 2;
}
void launch_jacobi_step(const GridParams& g, int cb, const double* dinv, double* x, const double* p,
                        const double* q, double* r, double* z, PcgState* st, double* partials,
                        double* history, int init, int defer, cudaStream_t s) {
  if (cb == 0)
    return launch_g_jacobi_step(g, dinv, x, p, q, r, z, st, partials, history, init, defer, s);
  if (cb == 8) launch_pdl(k_jacobi_step<8>, dim3((unsigned)g.nbo), dim3(512), 0, s, g, dinv, x, p, q, r, z, st, partials, history, init, defer);
  else launch_pdl(k_jacobi_step<4>, dim3((unsigned)g.nbo), dim3(64), 0, s, g, dinv, x, p, q, r, z, st, partials, history, init, defer);
}

}  // namespace tmg
