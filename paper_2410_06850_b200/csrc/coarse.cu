// Coarse and coarse-coarse levels (north_star items 3, 4 (second level), 6).
//
// A_c = R_c A R_c^T (solver.cpp:265, galerkin_product sparse.cpp:261-270) is a
// block 7-point operator because every R_c row lives in one coarse cell and A
// is 7-point: block (I, J) = Phi_I^T A_IJ Phi_J, stored as Ac[I][dir][a][b],
// dir = self, x-lo, x-hi, y-lo, y-hi, z-lo, z-hi. The coarse-coarse spectral
// problem of one cc element (coarse_coarse_basis, coarse_space.cpp:343-406) is
// P S_E P^T = A_c restricted to the element's children minus, on the diagonal
// blocks, the face terms that cross the element boundary and the Dirichlet
// terms (S_E uses only faces strictly inside the element); it is solved densely
// per element (cyclic Jacobi, one warp) and its L_cc lowest eigenvectors are
// the rows of R_cc. A_cc = R_cc A_c R_cc^T is again block 7-point at the cc
// level and is assembled densely for the direct solve.
#include <type_traits>

#include "kernels.h"
#include "stencil.cuh"
#include "symv.cuh"
#include "coarse_elem.cuh"

namespace tmg {

// ------------------------------------------------------------ A_c blocks

template <int CB, int LM>
__global__ void __launch_bounds__(CB * CB * CB) k_coarse_blocks(GridParams g,
                                                               const double* __restrict__ kappa,
                                                               const uint8_t* __restrict__ dmask,
                                                               const double* __restrict__ phi,
                                                               double* Ac, double* Bc) {
  constexpr int C = CB * CB * CB, NW = C / 32;
  __shared__ StencilSmem<CB> ss;
  constexpr int K2 = LM * LM;  // LM = L_c (template: exact register arrays)
  __shared__ double red[K2 * NW + K2 + 8];
  constexpr int lc = LM;
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  load_tile<CB, true>(kappa, ss.kt, g, bc);
  const int t = threadIdx.x, li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
  double f[LM];
#pragma unroll
  for (int a = 0; a < LM; ++a) f[a] = a < lc ? phi[((size_t)bc.b * lc + a) * C + t] : 0.0;
  // Phi at an in-brick neighbour j (read through L1; set-up only)
  auto ph = [&](int a, int j) { return a < lc ? __ldg(phi + ((size_t)bc.b * lc + a) * C + j) : 0.0; };
  __syncthreads();
  tile_faces<CB>(ss.kt, ss.fx, ss.fy, ss.fz, g, bc);
  __syncthreads();
  const unsigned dm = brick_on_boundary(g, bc) ? dmask[bofs(bc.b, C) + t] : 0u;
  const FaceSet fs = cell_faces<CB>(ss.fx, ss.fy, ss.fz, ss.kt[Tile<CB>::idx(li, lj, lk)], li, lj, lk, g, bc, dm);
  // --- self block: sum_l d_l f_a f_b - sum_{+x,+y,+z in brick} T (f_a(l) f_b(j) + f_a(j) f_b(l))
  {
    double v[K2];  // v[a * LM + b]; entries a, b >= lc stay 0
    const int st[3] = {1, CB, CB * CB};
    const int co[3] = {li, lj, lk};
#pragma unroll
    for (int a = 0; a < LM; ++a)
#pragma unroll
      for (int b = 0; b < LM; ++b) v[a * LM + b] = fs.diag * f[a] * f[b];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (co[ax] + 1 >= CB) continue;
      const int j = t + st[ax];
      const double T = fs.t[2 * ax + 1];
#pragma unroll
      for (int a = 0; a < LM; ++a)
#pragma unroll
        for (int b = 0; b < LM; ++b) v[a * LM + b] -= T * (f[a] * ph(b, j) + ph(a, j) * f[b]);
    }
    block_sum_k<C, K2>(v, red);
    if (t < lc * lc) Ac[((size_t)bc.b * 7 + 0) * lc * lc + t] = v[(t / lc) * LM + t % lc];
  }
  // --- face blocks: -T_lj f_a(l) phi_J,b(j) over the CB^2 face pairs
  int nbr[6];
#pragma unroll
  for (int f6 = 0; f6 < 6; ++f6) nbr[f6] = nbr_brick(g, bc, f6);
  const int co[3] = {li, lj, lk};
  for (int fc = 0; fc < 6; ++fc) {
    double v[K2];
#pragma unroll
    for (int e = 0; e < K2; ++e) v[e] = 0.0;
    const int ax = fc >> 1;
    const bool on_face = (fc & 1) ? co[ax] == CB - 1 : co[ax] == 0;
    if (nbr[fc] >= 0 && on_face) {
      // neighbour local index: mirror coordinate on this axis
      int nc3[3] = {li, lj, lk};
      nc3[ax] = (fc & 1) ? 0 : CB - 1;
      const int lj2 = nc3[0] + CB * (nc3[1] + CB * nc3[2]);
      const double T = fs.t[fc];
#pragma unroll
      for (int b = 0; b < LM; ++b) {
        const double pj = b < lc ? phi[((size_t)nbr[fc] * lc + b) * C + lj2] : 0.0;
#pragma unroll
        for (int a = 0; a < LM; ++a) v[a * LM + b] = -T * f[a] * pj;
      }
    }
    block_sum_k<C, K2>(v, red);
    if (t < lc * lc) Ac[((size_t)bc.b * 7 + 1 + fc) * lc * lc + t] = v[(t / lc) * LM + t % lc];
  }
  // --- cc-boundary correction: faces leaving the cc element + Dirichlet terms
  {
    const int bco[3] = {bc.bi, bc.bj, bc.bk};
    double e = 0.0;
#pragma unroll
    for (int fc = 0; fc < 6; ++fc) {
      const int ax = fc >> 1;
      const bool hi = fc & 1;
      const bool on_face = hi ? co[ax] == CB - 1 : co[ax] == 0;
      if (!on_face) continue;
      if (fs.nbmask & (1 << fc)) {
        const bool crosses = hi ? ((bco[ax] + 1) % g.sd == 0) : (bco[ax] % g.sd == 0);
        if (crosses) e += fs.t[fc];
      } else if (dm & (1u << fc)) {
        e += fs.t[fc];
      }
    }
    double v[K2];
#pragma unroll
    for (int a = 0; a < LM; ++a)
#pragma unroll
      for (int b = 0; b < LM; ++b) v[a * LM + b] = e * f[a] * f[b];
    block_sum_k<C, K2>(v, red);
    if (t < lc * lc) Bc[(size_t)bc.b * lc * lc + t] = v[(t / lc) * LM + t % lc];
  }
}

// One warp per cc element: projected matrix, eigenpairs, R_cc rows.
__global__ void k_cc_basis(GridParams g, const double* __restrict__ Ac,
                           const double* __restrict__ Bc, double* Rcc, double* cc_evals) {
  extern __shared__ double sm[];
  const int q = g.sd * g.sd * g.sd * g.lc;
  double* M = sm;
  double* V = M + q * q;
  const ElemCoord ec = elem_coord(g, blockIdx.x + g.e0);
  build_elem_matrix(g, ec, Ac, Bc, true, M, q);
  if (threadIdx.x < 32) warp_jacobi(M, V, q);
  __syncthreads();
  if (threadIdx.x == 0) {
    // selection of the lcc smallest (ascending, ties by index)
    int* used = (int*)(V + q * q);
    for (int i = 0; i < q; ++i) used[i] = 0;
    for (int k = 0; k < g.lcc; ++k) {
      int best = -1;
      for (int i = 0; i < q; ++i)
        if (!used[i] && (best < 0 || M[i * q + i] < M[best * q + best])) best = i;
      used[best] = 1;
      cc_evals[ec.e * g.lcc + k] = M[best * q + best];
      double s = 0.0;
      for (int r = 0; r < q; ++r) s += V[r * q + best];
      const double sg = s < 0.0 ? -1.0 : 1.0;
      for (int r = 0; r < q; ++r) Rcc[((int64_t)ec.e * g.lcc + k) * q + r] = sg * V[r * q + best];
    }
  }
}

// In-place Gauss-Jordan inversion of an SPD matrix in smem (block-wide).
// Records the pivots (LDL^T pivots) and applies the reference's rule.
__device__ bool smem_gj_inverse(double* M, int n, double* col, double* rowp, double* pivs) {
  for (int p = 0; p < n; ++p) {
    const double pv = M[p * n + p];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      col[i] = M[i * n + p];
      rowp[i] = M[p * n + i];
    }
    if (threadIdx.x == 0) pivs[p] = pv;
    __syncthreads();
    const double inv = 1.0 / pv;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e % n;
      double v;
      if (i == p && j == p) v = inv;
      else if (i == p) v = rowp[j] * inv;
      else if (j == p) v = -col[i] * inv;
      else v = M[e] - col[i] * (rowp[j] * inv);
      M[e] = v;
    }
    __syncthreads();
  }
  bool ok = true;
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int p = 0; p < n; ++p) mx = fmax(mx, fabs(pivs[p]));
    for (int p = 0; p < n; ++p)
      if (!(pivs[p] > 1e-14 * mx)) ok = false;
    pivs[n] = ok ? 1.0 : 0.0;
  }
  __syncthreads();
  ok = pivs[n] != 0.0;
  // symmetrise
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    if (i < j) {
      const double s = 0.5 * (M[i * n + j] + M[j * n + i]);
      M[i * n + j] = s;
      M[j * n + i] = s;
    }
  }
  __syncthreads();
  return ok;
}

// Coarse smoother: exact inverse of A_c over each cc element's rows
// (coarse_blocks_by_cc, solver.cpp:362-374) -> Winv[E][q][q].
__global__ void k_coarse_smoother(GridParams g, const double* __restrict__ Ac, double* Winv,
                                  int* status) {
  extern __shared__ double sm[];
  const int q = g.sd * g.sd * g.sd * g.lc;
  double* M = sm;
  double* col = M + q * q;
  double* rowp = col + q;
  double* pivs = rowp + q;
  const ElemCoord ec = elem_coord(g, blockIdx.x + g.e0);
  build_elem_matrix(g, ec, Ac, nullptr, false, M, q);
  const bool ok = smem_gj_inverse(M, q, col, rowp, pivs);
  if (!ok && threadIdx.x == 0) atomicExch(status, 2);
  for (int e = threadIdx.x; e < q * q; e += blockDim.x) Winv[(int64_t)ec.e * q * q + e] = M[e];
}

// A_cc block (E, F) for F in {E, 6 face neighbours}: sum over coupled child
// pairs (I in E, J in F) of R_E[:, I] Ac_IJ R_F[:, J]^T, written into the dense
// n_cc x n_cc matrix. grid = (m_cc, 7), block = lcc*lcc threads.
// planar (acc_planes.cu): Acc = ncz dense P x P plane blocks, C = the z-lo
// coupling blocks [element][L_cc][L_cc]; z-hi couplings are their transposes.
__global__ void k_acc_assemble(GridParams g, const double* __restrict__ Ac,
                               const double* __restrict__ Rcc, double* Acc, int64_t ldacc,
                               double* C, int planar) {
  const int q = g.sd * g.sd * g.sd * g.lc, nch = g.sd * g.sd * g.sd;
  const ElemCoord ec = elem_coord(g, blockIdx.x + g.e0);
  const int fdir = blockIdx.y;  // 0 self, 1..6 faces
  int64_t F = ec.e;
  if (fdir > 0) {
    const int64_t coords[3] = {ec.ei, ec.ej, ec.ek};
    const int64_t n3[3] = {g.ncx, g.ncy, g.ncz};
    const int ax = (fdir - 1) >> 1;
    const bool hi = (fdir - 1) & 1;
    if (hi ? coords[ax] + 1 >= n3[ax] : coords[ax] == 0) return;
    const int64_t strides[3] = {1, g.ncx, g.ncx * g.ncy};
    F = hi ? ec.e + strides[ax] : ec.e - strides[ax];
  }
  const ElemCoord fc = elem_coord(g, F);
  if (planar && fdir == 6) return;
  const int64_t nxy = g.ncx * g.ncy, P = nxy * g.lcc;
  for (int pr = threadIdx.x; pr < g.lcc * g.lcc; pr += blockDim.x) {
    const int bb = pr / g.lcc, bp = pr % g.lcc;
    const double* RE = Rcc + (ec.e * g.lcc + bb) * q;
    const double* RF = Rcc + (F * g.lcc + bp) * q;
    double acc = 0.0;
    for (int ci = 0; ci < nch; ++ci) {
      const int64_t I = child_brick(g, ec, ci);
      for (int dir = 0; dir < 7; ++dir) {
        int64_t J = dir == 0 ? I : brick_nbr(g, I, dir - 1);
        if (J < 0) continue;
        const int cj = child_index(g, fc, J);
        if (cj < 0) continue;
        const double* blk = Ac + (I * 7 + dir) * g.lc * g.lc;
        for (int a = 0; a < g.lc; ++a) {
          double s = 0.0;
          for (int b = 0; b < g.lc; ++b) s += blk[a * g.lc + b] * RF[cj * g.lc + b];
          acc += RE[ci * g.lc + a] * s;
        }
      }
    }
    if (!planar) {
      Acc[(ec.e * g.lcc + bb) * ldacc + F * g.lcc + bp] = acc;
    } else if (fdir == 5) {
      C[(ec.e * g.lcc + bb) * g.lcc + bp] = acc;
    } else {
      const int64_t eloc = ec.e - ec.ek * nxy, floc = F - ec.ek * nxy;
      Acc[ec.ek * P * P + (eloc * g.lcc + bb) * P + floc * g.lcc + bp] = acc;
    }
  }
}

// ------------------------------------------------ coarse part of the V-cycle

// One CTA (q threads, q = sd^3 * L_c) per cc element; thread i owns the
// element-local coarse dof i = child*L_c + a. 32-bit index math throughout.
struct ElemDofs {
  int brick;  // coarse cell (brick) of this dof
  int a;      // basis index within the coarse cell
};
__device__ __forceinline__ ElemDofs elem_dof(const GridParams& g, int e, int i) {
  const int ncx = (int)g.ncx, ncy = (int)g.ncy, sd = g.sd;
  const int ei = e % ncx, ej = (e / ncx) % ncy, ek = e / (ncx * ncy);
  const int ci = i / g.lc;
  const int di = ci % sd, dj = (ci / sd) % sd, dk = ci / (sd * sd);
  ElemDofs d;
  d.brick = (ei * sd + di) + (int)g.nbx * ((ej * sd + dj) + (int)g.nby * (ek * sd + dk));
  d.a = i % g.lc;
  return d;
}

// (A_c x)_(I,a) for a global coarse vector x (block 7-point, Ac[I][dir][a][:]).
__device__ __forceinline__ double coarse_apply_row(const GridParams& g, const double* __restrict__ Ac,
                                                   const double* __restrict__ x, int I, int a) {
  const int nbx = (int)g.nbx, nby = (int)g.nby, nbz = (int)g.nbz;
  const int bi = I % nbx, bj = (I / nbx) % nby, bk = I / (nbx * nby);
  const int nb[7] = {I, bi > 0 ? I - 1 : -1, bi + 1 < nbx ? I + 1 : -1,
                     bj > 0 ? I - nbx : -1, bj + 1 < nby ? I + nbx : -1,
                     bk > 0 ? I - nbx * nby : -1, bk + 1 < nbz ? I + nbx * nby : -1};
  double s = 0.0;
#pragma unroll
  for (int dir = 0; dir < 7; ++dir) {
    if (nb[dir] < 0) continue;
    const int lc = g.lc;
    const double* blk = Ac + ((size_t)I * 7 + dir) * lc * lc + a * lc;
    const double* xv = x + (size_t)nb[dir] * lc;
    if (lc == 4) {  // the default L_c, unrolled
#pragma unroll
      for (int b = 0; b < 4; ++b) s = fma(blk[b], xv[b], s);
    } else {
      for (int b = 0; b < lc; ++b) s = fma(blk[b], xv[b], s);
    }
  }
  return s;
}

// coarse_apply_row reading x through L2 only (x written by other CTAs of the
// same cooperative grid)
__device__ __forceinline__ double coarse_apply_row_cg(const GridParams& g,
                                                      const double* __restrict__ Ac,
                                                      const double* x, int I, int a) {
  const int nbx = (int)g.nbx, nby = (int)g.nby, nbz = (int)g.nbz;
  const int bi = I % nbx, bj = (I / nbx) % nby, bk = I / (nbx * nby);
  const int nb[7] = {I, bi > 0 ? I - 1 : -1, bi + 1 < nbx ? I + 1 : -1,
                     bj > 0 ? I - nbx : -1, bj + 1 < nby ? I + nbx : -1,
                     bk > 0 ? I - nbx * nby : -1, bk + 1 < nbz ? I + nbx * nby : -1};
  double s = 0.0;
#pragma unroll
  for (int dir = 0; dir < 7; ++dir) {
    if (nb[dir] < 0) continue;
    const int lc = g.lc;
    const double* blk = Ac + ((size_t)I * 7 + dir) * lc * lc + a * lc;
    const double* xv = x + (size_t)nb[dir] * lc;
    if (lc == 4) {  // the default L_c, unrolled
#pragma unroll
      for (int b = 0; b < 4; ++b) s = fma(blk[b], __ldcg(xv + b), s);
    } else {
      for (int b = 0; b < lc; ++b) s = fma(blk[b], __ldcg(xv + b), s);
    }
  }
  return s;
}

// out_E = add_E + Winv_E in_E  (coarse_blocks_by_cc smoother, one sweep from 0:
// solver.cpp:221-243). Winv is symmetric: column i read coalesced.
__global__ void k_coarse_smooth(GridParams g, const int* __restrict__ done,
                                const double* __restrict__ Winv, const double* __restrict__ in,
                                const double* __restrict__ add, double* out) {
  pdl_trigger();
  pdl_wait();
  if (*done) return;
  extern __shared__ double sm[];
  const int q = g.sd * g.sd * g.sd * g.lc, e = (int)(blockIdx.x + g.e0);
  double* xin = sm;
  for (int i = threadIdx.x; i < q; i += blockDim.x) {
    const ElemDofs d = elem_dof(g, e, i);
    xin[i] = in[(size_t)d.brick * g.lc + d.a];
  }
  __syncthreads();
  const double* W = Winv + (size_t)e * q * q;
  for (int i = threadIdx.x; i < q; i += blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
    int j = 0;
    for (; j + 1 < q; j += 2) {
      s0 = fma(W[(size_t)j * q + i], xin[j], s0);
      s1 = fma(W[(size_t)(j + 1) * q + i], xin[j + 1], s1);
    }
    if (j < q) s0 = fma(W[(size_t)j * q + i], xin[j], s0);
    const ElemDofs d = elem_dof(g, e, i);
    const size_t gi = (size_t)d.brick * g.lc + d.a;
    out[gi] = (add ? add[gi] : 0.0) + (s0 + s1);
  }
}

// wc = rc - A_c rc0 on the element's dofs; rcc_(E,b) = R_cc[E][b] . wc
// (solver.cpp:297-301).
__global__ void k_coarse_restrict(GridParams g, const int* __restrict__ done,
                                  const double* __restrict__ Ac, const double* __restrict__ Rcc,
                                  const double* __restrict__ rc, const double* __restrict__ rc0,
                                  double* rcc) {
  pdl_trigger();
  pdl_wait();
  if (*done) return;
  extern __shared__ double sm[];
  const int q = g.sd * g.sd * g.sd * g.lc, e = (int)(blockIdx.x + g.e0);
  double* wc = sm;
  for (int i = threadIdx.x; i < q; i += blockDim.x) {
    const ElemDofs d = elem_dof(g, e, i);
    wc[i] = rc[(size_t)d.brick * g.lc + d.a] - coarse_apply_row(g, Ac, rc0, d.brick, d.a);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < g.lcc; b += blockDim.x) {
    const double* R = Rcc + ((size_t)e * g.lcc + b) * q;
    double s = 0.0;
    for (int i = 0; i < q; ++i) s = fma(R[i], wc[i], s);
    rcc[(size_t)e * g.lcc + b] = s;
  }
}

// rc1 = rc0 + R_cc^T ecc on the element's dofs (solver.cpp:307-309).
__global__ void k_coarse_prolong(GridParams g, const int* __restrict__ done,
                                 const double* __restrict__ Rcc, const double* __restrict__ rc0,
                                 const double* __restrict__ ecc, double* rc1) {
  pdl_trigger();
  pdl_wait();
  if (*done) return;
  const int q = g.sd * g.sd * g.sd * g.lc, e = (int)(blockIdx.x + g.e0);
  for (int i = threadIdx.x; i < q; i += blockDim.x) {
    const ElemDofs d = elem_dof(g, e, i);
    double s = 0.0;
    for (int b = 0; b < g.lcc; ++b)
      s = fma(Rcc[((size_t)e * g.lcc + b) * q + i], ecc[(size_t)e * g.lcc + b], s);
    const size_t gi = (size_t)d.brick * g.lc + d.a;
    rc1[gi] = rc0[gi] + s;
  }
}

// tc = rc - A_c rc1 (any dof) — thread per coarse dof.
__global__ void k_coarse_resid(GridParams g, const int* __restrict__ done,
                               const double* __restrict__ Ac, const double* __restrict__ rc,
                               const double* __restrict__ x, double* out, int n) {
  pdl_trigger();
  pdl_wait();
  if (*done) return;
  const int64_t k = g.b0 * g.lc + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= g.b0 * g.lc + n) return;
  out[k] = rc[k] - coarse_apply_row(g, Ac, x, k / g.lc, k % g.lc);
}

// ---------------------------------------- fused coarse level (one kernel)
//
// The whole coarse part of one V-cycle for a single-slab context as one
// cooperative persistent kernel: one warp per cc element (q = sd^3 L_c <= 32
// dofs, lane i = dof i), four grid barriers between the phases that need
// other elements' results, and the symmetric tiled A_cc^-1 GEMV in the middle
// (its constant tiles start streaming at kernel entry). Replaces seven
// launch-latency-bound kernels (launch_coarse_cycle).
//   1  rc0 = W rc                      (solver.cpp:292-296)
//   2  rcc = R_cc (rc - A_c rc0)       (:297-301)
//   3  P   = tiles of A_cc^-1 . rcc    (:304)
//   4  ecc = sum_J P; rc1 = rc0 + R_cc^T ecc   (:307-309)
//   5  ec  = rc1 + W (rc - A_c rc1)    (:311-319)
// Grid-wide barrier for a co-resident (cooperative) grid: arrive on a global
// counter; the last CTA resets it and bumps the generation every other CTA
// waits on. Data other CTAs wrote before the barrier is read afterwards with
// L2-only loads (__ldcg), so no L1 invalidation is needed.
__device__ __forceinline__ void grid_barrier(unsigned int* bar) {
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
      while (*gen == my) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kFusedLc = 4;  // the fused coarse kernel is built for L_c = 4 (q = 32)

template <int Q, int LCC>
__global__ void __launch_bounds__(256, 2) k_coarse_fused(GridParams g, const int* __restrict__ done,
                                                        const double* __restrict__ Ac,
                                                        const double* __restrict__ Winv,
                                                        const double* __restrict__ Rcc,
                                                        const double* __restrict__ T, int64_t n,
                                                        double* P, const double* __restrict__ rc,
                                                        double* rc0, double* rcc, double* rc1,
                                                        double* ec, unsigned int* bar) {
  static_assert(Q == 32, "one lane per element dof");
  extern __shared__ __align__(128) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>(smraw);
  double* xs = ring + kSymvSlots * TS * TS;
  __shared__ SymvSmem ss;
  symv_begin(ss, ring, T, n);  // constant tiles stream while phases 1-2 run
  pdl_wait();
  if (*done) {  // same flag for every CTA: no barrier is left half-entered
    symv_drain(ss, n);
    return;
  }
  const int lane = threadIdx.x & 31;
  // element e -> warp (e / gridDim.x) of CTA (e % gridDim.x): spread over every SM
  const int64_t w0 = (int64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t e_end = g.e0 + g.neo;
  // every phase first issues all of its loads (one round trip), then computes
  // 1: rc0 = W rc
  for (int64_t e = g.e0 + w0; e < e_end; e += nw) {
    const ElemDofs d = elem_dof(g, (int)e, lane);
    const size_t gi = (size_t)d.brick * kFusedLc + d.a;
    const double* W = Winv + (size_t)e * Q * Q;
    double wcol[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) wcol[j] = W[(size_t)j * Q + lane];  // W symmetric: column = row
    const double xin = rc[gi];
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int j = 0; j < Q; j += 2) {
      s0 = fma(wcol[j], __shfl_sync(0xffffffffu, xin, j), s0);
      s1 = fma(wcol[j + 1], __shfl_sync(0xffffffffu, xin, j + 1), s1);
    }
    rc0[gi] = s0 + s1;
  }
  grid_barrier(bar);
  // 2: rcc = R_cc (rc - A_c rc0)
  for (int64_t e = g.e0 + w0; e < e_end; e += nw) {
    const ElemDofs d = elem_dof(g, (int)e, lane);
    double rr[LCC];
#pragma unroll
    for (int b = 0; b < LCC; ++b) rr[b] = Rcc[((size_t)e * LCC + b) * Q + lane];
    const double wc = rc[(size_t)d.brick * kFusedLc + d.a] - coarse_apply_row_cg(g, Ac, rc0, d.brick, d.a);
#pragma unroll
    for (int b = 0; b < LCC; ++b) {
      const double v = warp_sum(rr[b] * wc);
      if (lane == b) rcc[(size_t)e * LCC + b] = v;
    }
  }
  grid_barrier(bar);
  // 3: tile partials of A_cc^-1 rcc
  symv_run(ss, ring, xs, T, n, rcc, P);
  grid_barrier(bar);
  // 4: ecc rows of the element (fixed-order sums over the nt tile columns), rc1
  const int64_t nt = (n + TS - 1) / TS;
  for (int64_t e = g.e0 + w0; e < e_end; e += nw) {
    const ElemDofs d = elem_dof(g, (int)e, lane);
    const size_t gi = (size_t)d.brick * kFusedLc + d.a;
    double rr[LCC], pv[LCC][2];
#pragma unroll
    for (int b = 0; b < LCC; ++b) {
      rr[b] = Rcc[((size_t)e * LCC + b) * Q + lane];
      const int64_t row = e * LCC + b, I = row / TS, r = row % TS;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t J = lane + 32 * h;
        pv[b][h] = J < nt ? __ldcg(P + (I * nt + J) * TS + r) : 0.0;
      }
    }
    const double r0v = __ldcg(rc0 + gi);
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < LCC; ++b) s = fma(rr[b], warp_sum(pv[b][0] + pv[b][1]), s);
    rc1[gi] = r0v + s;
    if (nt > 64) __trap();  // two tile columns per lane (n_cc <= 4096)
  }
  grid_barrier(bar);
  // 5: ec = rc1 + W (rc - A_c rc1)
  for (int64_t e = g.e0 + w0; e < e_end; e += nw) {
    const ElemDofs d = elem_dof(g, (int)e, lane);
    const size_t gi = (size_t)d.brick * kFusedLc + d.a;
    const double* W = Winv + (size_t)e * Q * Q;
    double wcol[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) wcol[j] = W[(size_t)j * Q + lane];
    const double tcv = rc[gi] - coarse_apply_row_cg(g, Ac, rc1, d.brick, d.a);
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int j = 0; j < Q; j += 2) {
      s0 = fma(wcol[j], __shfl_sync(0xffffffffu, tcv, j), s0);
      s1 = fma(wcol[j + 1], __shfl_sync(0xffffffffu, tcv, j + 1), s1);
    }
    ec[gi] = __ldcg(rc1 + gi) + (s0 + s1);
  }
}

// true when launch_coarse_fused handles the hierarchy (q = 32, L_cc = 8, n_cc <= 4096)
bool coarse_fused_supported(const GridParams& g, int64_t n_cc) {
  return g.lc == kFusedLc && g.sd * g.sd * g.sd * g.lc == 32 && g.lcc == 8 && n_cc <= 64 * TS;
}

// ------------------------------------------------------------- launchers

void launch_coarse_fused(const GridParams& g, const int* done, const double* Ac,
                         const double* Winv, const double* Rcc, const double* Acc_tiles,
                         double* symv_partials, int64_t n_cc, const double* rc, double* rc0,
                         double* rcc, double* rc1, double* ec, unsigned int* bar,
                         cudaStream_t s) {
  const size_t smem = symv_dyn_smem(n_cc);
  // co-residency of the grid barriers: every CTA of the grid resident at
  // once, per device (device_occupancy also raises the smem limit there)
  const int grid = device_occupancy(k_coarse_fused<32, 8>, 256, smem) * device_sm_count();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  launch_check(cudaLaunchKernelEx(&cfg, k_coarse_fused<32, 8>, g, done, Ac, Winv, Rcc, Acc_tiles,
                                  n_cc, symv_partials, rc, rc0, rcc, rc1, ec, bar),
               "k_coarse_fused (cooperative) launch");
}

void launch_coarse_blocks(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                          const double* phi, double* Ac, double* Bc, cudaStream_t s) {
  auto go = [&](auto L) {
    constexpr int LM = decltype(L)::value;
    if (cb == 8)
      k_coarse_blocks<8, LM><<<(unsigned)g.nbo, 512, 0, s>>>(g, kappa, dmask, phi, Ac, Bc);
    else
      k_coarse_blocks<4, LM><<<(unsigned)g.nbo, 64, 0, s>>>(g, kappa, dmask, phi, Ac, Bc);
  };
  switch (g.lc) {
    case 1: go(std::integral_constant<int, 1>{}); break;
    case 2: go(std::integral_constant<int, 2>{}); break;
    case 3: go(std::integral_constant<int, 3>{}); break;
    case 4: go(std::integral_constant<int, 4>{}); break;
    case 5: go(std::integral_constant<int, 5>{}); break;
    default: go(std::integral_constant<int, 6>{}); break;
  }
}

void launch_cc_basis(const GridParams& g, const double* Ac, const double* Bc, double* Rcc,
                     double* cc_evals, cudaStream_t s) {
  const int q = g.sd * g.sd * g.sd * g.lc;
  const size_t smem = sizeof(double) * (size_t)(2 * q * q + q + 8);
  cudaFuncSetAttribute(k_cc_basis, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_cc_basis<<<(unsigned)g.neo, 64, smem, s>>>(g, Ac, Bc, Rcc, cc_evals);
}

// two_grid: R_cc = I (build_two_grid, solver.cpp:401-420), lcc = q: row
// (E, k) of R_cc is the unit vector of the element's k-th coarse dof.
__global__ void k_cc_identity(GridParams g, double* Rcc, double* cc_evals) {
  const int q = g.sd * g.sd * g.sd * g.lc;
  const int64_t e = blockIdx.x + g.e0;
  for (int i = threadIdx.x; i < q * q; i += blockDim.x)
    Rcc[e * q * q + i] = (i / q == i % q) ? 1.0 : 0.0;
  for (int k = threadIdx.x; k < q; k += blockDim.x) cc_evals[e * q + k] = 0.0;
}

void launch_cc_identity(const GridParams& g, double* Rcc, double* cc_evals, cudaStream_t s) {
  k_cc_identity<<<(unsigned)g.neo, 256, 0, s>>>(g, Rcc, cc_evals);
}

void launch_coarse_smoother(const GridParams& g, const double* Ac, double* Winv, int* status,
                            cudaStream_t s) {
  const int q = g.sd * g.sd * g.sd * g.lc;
  const size_t smem = sizeof(double) * (size_t)(q * q + 3 * q + 8);
  cudaFuncSetAttribute(k_coarse_smoother, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_coarse_smoother<<<(unsigned)g.neo, 256, smem, s>>>(g, Ac, Winv, status);
}

void launch_acc_assemble(const GridParams& g, const double* Ac, const double* Rcc, double* Acc,
                         cudaStream_t s) {
  const int64_t n = g.ncc * g.lcc;
  // this context's rows of the global n x n matrix
  cudaMemsetAsync(Acc + g.e0 * g.lcc * n, 0, sizeof(double) * (size_t)(g.neo * g.lcc * n), s);
  dim3 grid((unsigned)g.neo, 7);
  k_acc_assemble<<<grid, g.lcc * g.lcc < 256 ? g.lcc * g.lcc : 256, 0, s>>>(g, Ac, Rcc, Acc, n,
                                                                           nullptr, 0);
}

// plane blocks + z couplings of A_cc (single slab; acc_planes.cu)
// The blocks of the caller's elements (g.e0 .. g.e0 + g.neo: whole planes);
// zero = clear all planes first (single slab, or the first of several slabs).
void launch_acc_assemble_planes(const GridParams& g, const double* Ac, const double* Rcc,
                                double* Gd, double* C, cudaStream_t s, bool zero) {
  const int64_t P = g.ncx * g.ncy * g.lcc;
  if (zero) {
    cudaMemsetAsync(Gd, 0, sizeof(double) * (size_t)(g.ncz * P * P), s);
    cudaMemsetAsync(C, 0, sizeof(double) * (size_t)(g.ncc * g.lcc * g.lcc), s);
  }
  dim3 grid((unsigned)g.neo, 7);
  k_acc_assemble<<<grid, g.lcc * g.lcc < 256 ? g.lcc * g.lcc : 256, 0, s>>>(g, Ac, Rcc, Gd, P, C,
                                                                           1);
}

// Coarse part of one V-cycle (solver.cpp:292-319): rc -> ec.
//  rc0 = S_c(rc); rcc = R_cc (rc - A_c rc0); ecc = A_cc^-1 rcc;
//  rc1 = rc0 + R_cc^T ecc; ec = rc1 + S_c(rc - A_c rc1).
void launch_coarse_cycle(const GridParams& g, const int* done, const double* Ac,
                         const double* Winv, const double* Rcc, const double* Acc_tiles,
                         double* symv_partials, int64_t n_cc, const double* rc, double* rc0,
                         double* rcc, double* ecc, double* rc1, double* tc, double* ec,
                         const AccPlanesRef* planes, cudaStream_t s) {
  const int q = g.sd * g.sd * g.sd * g.lc;
  const int nt = (q < 256 ? (q + 31) / 32 * 32 : 256);
  const int nc = (int)(g.nbo * g.lc);
  const size_t sm = sizeof(double) * (size_t)q;
  const double* nul = nullptr;
  launch_pdl(k_coarse_smooth, dim3((unsigned)g.neo), dim3(nt), sm, s, g, done, Winv, rc, nul, rc0);
  launch_pdl(k_coarse_restrict, dim3((unsigned)g.neo), dim3(nt), sm, s, g, done, Ac, Rcc, rc, rc0,
             rcc);
  if (planes)
    launch_acc_planes_solve(g, done, planes->T, planes->C, rcc, ecc, planes->wv, symv_partials,
                            s);
  else
    launch_symv(done, Acc_tiles, n_cc, rcc, symv_partials, ecc, s);
  launch_pdl(k_coarse_prolong, dim3((unsigned)g.neo), dim3(nt), 0, s, g, done, Rcc, rc0, ecc, rc1);
  launch_pdl(k_coarse_resid, dim3((unsigned)((nc + 255) / 256)), dim3(256), 0, s, g, done, Ac, rc,
             rc1, tc, nc);
  launch_pdl(k_coarse_smooth, dim3((unsigned)g.neo), dim3(nt), sm, s, g, done, Winv, tc, rc1, ec);
}

// Phase launchers of the same cycle for partitioned solves (ghost exchanges
// and the A_cc row-block GEMV go between them).
void launch_coarse_smooth(const GridParams& g, const int* done, const double* Winv,
                          const double* in, const double* add, double* out, cudaStream_t s) {
  const int q = g.sd * g.sd * g.sd * g.lc, nt = (q < 256 ? (q + 31) / 32 * 32 : 256);
  launch_pdl(k_coarse_smooth, dim3((unsigned)g.neo), dim3(nt), sizeof(double) * (size_t)q, s, g,
             done, Winv, in, add, out);
}
void launch_coarse_restrict(const GridParams& g, const int* done, const double* Ac,
                            const double* Rcc, const double* rc, const double* rc0, double* rcc,
                            cudaStream_t s) {
  const int q = g.sd * g.sd * g.sd * g.lc, nt = (q < 256 ? (q + 31) / 32 * 32 : 256);
  launch_pdl(k_coarse_restrict, dim3((unsigned)g.neo), dim3(nt), sizeof(double) * (size_t)q, s, g,
             done, Ac, Rcc, rc, rc0, rcc);
}
void launch_coarse_prolong(const GridParams& g, const int* done, const double* Rcc,
                           const double* rc0, const double* ecc, double* rc1, cudaStream_t s) {
  const int q = g.sd * g.sd * g.sd * g.lc, nt = (q < 256 ? (q + 31) / 32 * 32 : 256);
  launch_pdl(k_coarse_prolong, dim3((unsigned)g.neo), dim3(nt), 0, s, g, done, Rcc, rc0, ecc, rc1);
}
void launch_coarse_resid(const GridParams& g, const int* done, const double* Ac, const double* rc,
                         const double* x, double* out, cudaStream_t s) {
  const int nc = (int)(g.nbo * g.lc);
  launch_pdl(k_coarse_resid, dim3((unsigned)((nc + 255) / 256)), dim3(256), 0, s, g, done, Ac, rc,
             x, out, nc);
}

int max_lc() { return kMaxLcCoarse; }

}  // namespace tmg
