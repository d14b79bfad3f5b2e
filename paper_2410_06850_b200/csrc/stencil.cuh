// Matrix-free TPFA operator on a brick tile (north_star item 1).
//
// The operator is the reference's cell-centred two-point flux approximation
// (proj/core/src/fvm.cpp:33-166): T_F = 2 k1 k2/(k1+k2) * area/h per interior
// face, 2 k_c * area/h per Dirichlet boundary face on the diagonal, nothing on
// Neumann faces. It is never materialised: each CTA stages the conductivity and
// the input vector of its brick plus a one-cell face halo in shared memory and
// computes every face transmissibility of the tile once (3 per cell) into
// shared face arrays. The diagonal is summed in the reference's face order
// (x-lo, x-hi, y-lo, y-hi, z-lo, z-hi, fvm.cpp:71-112) and the row product in
// its sorted-column order (z-lo, y-lo, x-lo, diag, x-hi, y-hi, z-hi;
// sparse.cpp:76-83) without FMA contraction, so y = A x is bitwise equal to
// SparseOperator::apply on the assembled CSR.
#pragma once
#include "common.cuh"

namespace tmg {

template <int CB>
struct Tile {
  static constexpr int E = CB + 2;
  static constexpr int N = E * E * E;
  static constexpr int C = CB * CB * CB;
  static constexpr int NF = (CB + 1) * CB * CB;  // faces per axis in a tile
  __device__ static __forceinline__ int idx(int i, int j, int k) {
    return (i + 1) + E * ((j + 1) + E * (k + 1));
  }
  // face between tile cells (i,j,k) and (i+1,j,k), i in [-1, CB-1]; likewise y, z
  __device__ static __forceinline__ int fxi(int i, int j, int k) { return (i + 1) + (CB + 1) * (j + CB * k); }
  __device__ static __forceinline__ int fyi(int i, int j, int k) { return (j + 1) + (CB + 1) * (i + CB * k); }
  __device__ static __forceinline__ int fzi(int i, int j, int k) { return (k + 1) + (CB + 1) * (i + CB * j); }
};

struct BrickCoord {
  int bi, bj, bk, b;
};

__device__ __forceinline__ BrickCoord brick_coord(const GridParams& g, int b) {
  BrickCoord c;
  const int nbx = (int)g.nbx, nby = (int)g.nby;
  c.b = b;
  c.bi = b % nbx;
  c.bj = (b / nbx) % nby;
  c.bk = b / (nbx * nby);
  return c;
}

__device__ __forceinline__ size_t bofs(int b, int C) { return (size_t)b * (size_t)C; }

// Neighbour brick across face f (0 x-lo .. 5 z-hi) or -1.
__device__ __forceinline__ int nbr_brick(const GridParams& g, const BrickCoord& bc, int f) {
  // selects, no branches: f differs between the lanes of a warp
  const int nbx = (int)g.nbx, nby = (int)g.nby, nbz = (int)g.nbz;
  const int ax = f >> 1;
  const int coord = ax == 0 ? bc.bi : ax == 1 ? bc.bj : bc.bk;
  const int n = ax == 0 ? nbx : ax == 1 ? nby : nbz;
  const int stride = ax == 0 ? 1 : ax == 1 ? nbx : nbx * nby;
  const bool inside = (f & 1) ? coord + 1 < n : coord > 0;
  return inside ? bc.b + ((f & 1) ? stride : -stride) : -1;
}

// Halo slot s in [0, 6*CB^2): face f = s / CB^2; returns the tile index and the
// neighbour-local cell index.
template <int CB>
__device__ __forceinline__ void halo_slot(int s, int& f, int& tidx, int& nl) {
  constexpr int F = CB * CB;
  f = s / F;
  const int q = s % F, u = q % CB, w = q / CB;
  switch (f) {
    case 0: tidx = Tile<CB>::idx(-1, u, w); nl = (CB - 1) + CB * (u + CB * w); break;
    case 1: tidx = Tile<CB>::idx(CB, u, w); nl = 0 + CB * (u + CB * w); break;
    case 2: tidx = Tile<CB>::idx(u, -1, w); nl = u + CB * ((CB - 1) + CB * w); break;
    case 3: tidx = Tile<CB>::idx(u, CB, w); nl = u + CB * (0 + CB * w); break;
    case 4: tidx = Tile<CB>::idx(u, w, -1); nl = u + CB * (w + CB * (CB - 1)); break;
    default: tidx = Tile<CB>::idx(u, w, CB); nl = u + CB * (w + CB * 0); break;
  }
}

// Load v's brick values into tile interior; if HALO, also the six face layers
// from the neighbouring bricks (0 outside the domain). Any CTA size (cells are
// strided by blockDim.x). Caller syncs.
template <int CB, bool HALO>
__device__ __forceinline__ void load_tile(const double* __restrict__ v, double* tile,
                                          const GridParams& g, const BrickCoord& bc) {
  constexpr int C = CB * CB * CB;
  for (int t = threadIdx.x; t < C; t += blockDim.x)
    tile[Tile<CB>::idx(t % CB, (t / CB) % CB, t / (CB * CB))] = __ldg(v + bofs(bc.b, C) + t);
  if (HALO) {
    for (int s = threadIdx.x; s < 6 * CB * CB; s += blockDim.x) {
      int f, ti, nl;
      halo_slot<CB>(s, f, ti, nl);
      const int nb = nbr_brick(g, bc, f);
      tile[ti] = nb >= 0 ? __ldg(v + bofs(nb, C) + nl) : 0.0;
    }
  }
}

// tile = z + beta * p_old (or z when `first`) over the brick and its face
// halo, loaded straight from the two vectors (solver.cpp:565-567).
template <int CB>
__device__ __forceinline__ void load_tile_axpy(const double* __restrict__ z,
                                               const double* __restrict__ p_old, double beta,
                                               bool first, double* tile, const GridParams& g,
                                               const BrickCoord& bc) {
  constexpr int C = CB * CB * CB;
  for (int t = threadIdx.x; t < C; t += blockDim.x) {
    const size_t s = bofs(bc.b, C) + t;
    const double zv = __ldg(z + s);
    tile[Tile<CB>::idx(t % CB, (t / CB) % CB, t / (CB * CB))] = first ? zv : zv + beta * __ldg(p_old + s);
  }
  for (int h = threadIdx.x; h < 6 * CB * CB; h += blockDim.x) {
    int f, ti, nl;
    halo_slot<CB>(h, f, ti, nl);
    const int nb = nbr_brick(g, bc, f);
    double v = 0.0;
    if (nb >= 0) {
      const size_t s = bofs(nb, C) + nl;
      const double zv = __ldg(z + s);
      v = first ? zv : zv + beta * __ldg(p_old + s);
    }
    tile[ti] = v;
  }
}

// All face transmissibilities of the tile (faces touching at least one
// interior cell); 0 where a face cell lies outside the domain.
template <int CB>
__device__ __forceinline__ void tile_faces(const double* kt, double* fx, double* fy, double* fz,
                                           const GridParams& g, const BrickCoord& bc) {
  constexpr int NF = Tile<CB>::NF;
  constexpr int C = CB * CB * CB;
  for (int s = threadIdx.x; s < 3 * NF; s += blockDim.x) {
    const int ax = s / NF, r = s % NF;
    const int a = r % (CB + 1) - 1, u = (r / (CB + 1)) % CB, w = r / ((CB + 1) * CB);
    int i0, j0, k0, i1, j1, k1, ga;
    int64_t n;
    if (ax == 0) { i0 = a; j0 = u; k0 = w; i1 = a + 1; j1 = u; k1 = w; ga = bc.bi * CB + a; n = g.nx; }
    else if (ax == 1) { i0 = u; j0 = a; k0 = w; i1 = u; j1 = a + 1; k1 = w; ga = bc.bj * CB + a; n = g.ny; }
    else { i0 = u; j0 = w; k0 = a; i1 = u; j1 = w; k1 = a + 1; ga = bc.bk * CB + a; n = g.nz; }
    double T = 0.0;
    if (ga >= 0 && ga + 1 < n) {
      // low cell first: face_transmissibility(k[low], k[high]) — both reference
      // call sites evaluate this product order (fvm.cpp:73-76, 91-94)
      T = __dmul_rn(face_t(kt[Tile<CB>::idx(i0, j0, k0)], kt[Tile<CB>::idx(i1, j1, k1)]),
                    g.cpl[ax]);
    }
    (ax == 0 ? fx : ax == 1 ? fy : fz)[r] = T;
  }
}

// Six face coefficients of one cell in the reference face order
// (x-lo, x-hi, y-lo, y-hi, z-lo, z-hi) plus presence bits of the neighbours.
struct FaceSet {
  double t[6];
  int nbmask;  // bit f: interior neighbour across face f exists
  double diag;
};

template <int CB>
__device__ __forceinline__ FaceSet cell_faces(const double* fx, const double* fy, const double* fz,
                                              double kc, int li, int lj, int lk,
                                              const GridParams& g, const BrickCoord& bc,
                                              unsigned dmask) {
  const int gi = bc.bi * CB + li, gj = bc.bj * CB + lj, gk = bc.bk * CB + lk;
  const bool has[6] = {gi > 0, gi < g.nx - 1, gj > 0, gj < g.ny - 1, gk > 0, gk < g.nz - 1};
  const double ft[6] = {fx[Tile<CB>::fxi(li - 1, lj, lk)], fx[Tile<CB>::fxi(li, lj, lk)],
                        fy[Tile<CB>::fyi(li, lj - 1, lk)], fy[Tile<CB>::fyi(li, lj, lk)],
                        fz[Tile<CB>::fzi(li, lj, lk - 1)], fz[Tile<CB>::fzi(li, lj, lk)]};
  FaceSet fs;
  fs.nbmask = 0;
  double diag = 0.0;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    double t = 0.0;
    if (has[f]) {
      t = ft[f];
      fs.nbmask |= 1 << f;
      diag = __dadd_rn(diag, t);
    } else if (dmask & (1u << f)) {
      t = __dmul_rn(__dmul_rn(2.0, kc), g.cpl[f >> 1]);
      diag = __dadd_rn(diag, t);
    }
    fs.t[f] = t;
  }
  fs.diag = diag;
  return fs;
}

// (A x)_c from a face set and an x tile, sorted-column order, no FMA.
template <int CB>
__device__ __forceinline__ double apply_row(const FaceSet& fs, const double* xt, int li, int lj,
                                            int lk) {
  constexpr int E = Tile<CB>::E;
  const int ti = Tile<CB>::idx(li, lj, lk);
  double s = 0.0;
  if (fs.nbmask & 16) s = __dadd_rn(s, __dmul_rn(-fs.t[4], xt[ti - E * E]));
  if (fs.nbmask & 4) s = __dadd_rn(s, __dmul_rn(-fs.t[2], xt[ti - E]));
  if (fs.nbmask & 1) s = __dadd_rn(s, __dmul_rn(-fs.t[0], xt[ti - 1]));
  s = __dadd_rn(s, __dmul_rn(fs.diag, xt[ti]));
  if (fs.nbmask & 2) s = __dadd_rn(s, __dmul_rn(-fs.t[1], xt[ti + 1]));
  if (fs.nbmask & 8) s = __dadd_rn(s, __dmul_rn(-fs.t[3], xt[ti + E]));
  if (fs.nbmask & 32) s = __dadd_rn(s, __dmul_rn(-fs.t[5], xt[ti + E * E]));
  return s;
}

__device__ __forceinline__ bool brick_on_boundary(const GridParams& g, const BrickCoord& bc) {
  return bc.bi == 0 || bc.bj == 0 || bc.bk == 0 || bc.bi == g.nbx - 1 || bc.bj == g.nby - 1 ||
         bc.bk == g.nbz - 1;
}

// Shared-memory scratch of one stencil tile: kappa tile + three face arrays.
template <int CB>
struct StencilSmem {
  double kt[Tile<CB>::N];
  double fx[Tile<CB>::NF], fy[Tile<CB>::NF], fz[Tile<CB>::NF];
};

// ------------------------------------------------ precomputed coefficients
//
// The solve phase applies A from four per-cell coefficient arrays computed
// once at set-up with the reference's exact expressions (k_coefficients):
//   coef[0] = T to the +x neighbour (0 if none), coef[1] = +y, coef[2] = +z,
//   coef[3] = diagonal (faces summed in reference order, Dirichlet included).
// A tile needs each axis' coefficients for its cells plus the low halo layer.
// Natural cell order (conflict-free stores and neighbour reads): cx/cy/cz[c]
// = T from cell c to its +axis neighbour, dg[c] = diagonal; hx/hy/hz = the
// low halo layer (the -axis neighbour brick's +axis T), indexed by the two
// in-face coordinates (x face: lj + CB*lk, y face: li + CB*lk, z face: li + CB*lj).
template <int CB>
struct CoefSmem {
  alignas(16) double cx[CB * CB * CB];
  alignas(16) double cy[CB * CB * CB];
  alignas(16) double cz[CB * CB * CB];
  alignas(16) double dg[CB * CB * CB];
  double hx[CB * CB], hy[CB * CB], hz[CB * CB];
};

// T to the cell one plane below (lk > 0)
template <int CB>
__device__ __forceinline__ double coef_tz_below(const CoefSmem<CB>& cs, int c) {
  return cs.cz[c - CB * CB];
}

template <int CB>
__device__ __forceinline__ void load_coefs(const double* __restrict__ coef, int64_t M, CoefSmem<CB>& cs,
                                           const GridParams& g, const BrickCoord& bc) {
  constexpr int C = CB * CB * CB;
  for (int t = threadIdx.x; t < C; t += blockDim.x) {
    const size_t s = bofs(bc.b, C) + t;
    cs.cx[t] = __ldg(coef + s);
    cs.cy[t] = __ldg(coef + M + s);
    cs.cz[t] = __ldg(coef + 2 * M + s);
    cs.dg[t] = __ldg(coef + 3 * M + s);
  }
  // low halo layers: the +axis coefficient of the neighbouring brick's top layer
  for (int h = threadIdx.x; h < 3 * CB * CB; h += blockDim.x) {
    const int ax = h / (CB * CB), q = h % (CB * CB), u = q % CB, w = q / CB;
    const int nb = nbr_brick(g, bc, 2 * ax);
    const int nl = ax == 0 ? (CB - 1) + CB * (u + CB * w)
                           : ax == 1 ? u + CB * ((CB - 1) + CB * w) : u + CB * (w + CB * (CB - 1));
    const double v = nb >= 0 ? __ldg(coef + (size_t)ax * M + bofs(nb, C) + nl) : 0.0;
    (ax == 0 ? cs.hx : ax == 1 ? cs.hy : cs.hz)[q] = v;
  }
}

// load_coefs + load_tile_axpy for a CTA of exactly NT threads, each owning
// pairs of x-adjacent cells (c = 2 pr, 2 pr + 1): the brick's own data moves
// as coalesced 128-bit loads, and every global load of a thread is issued
// before the first shared-memory store (~12 loads in flight per thread).
template <int CB, int NT>
__device__ __forceinline__ void load_coefs_tile_axpy(const double* __restrict__ coef, int64_t M,
                                                     CoefSmem<CB>& cs, const double* __restrict__ z,
                                                     const double* __restrict__ p_old, double beta,
                                                     bool first, double* tile,
                                                     const GridParams& g, const BrickCoord& bc,
                                                     bool with_dg = true) {
  // with_dg = false (CTA-uniform): the diagonal array is neither read nor
  // staged; apply_coef<CB, false> sums it from the six face coefficients
  constexpr int C = CB * CB * CB, F = CB * CB, NPAIR = C / 2;
  constexpr int KO = (NPAIR + NT - 1) / NT;      // own cell pairs per thread
  constexpr int KH = (6 * F + NT - 1) / NT;      // halo cells per thread
  constexpr int KC = (3 * F + NT - 1) / NT;      // coefficient halo entries per thread
  const int t = threadIdx.x;
  double2 cf[KO][4], zo[KO], po[KO];
  double zh[KH], ph[KH], ch[KC];
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int pr = t + k * NT;
    if (pr < NPAIR) {
      const size_t s = bofs(bc.b, C) + 2 * pr;
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (a < 3 || with_dg) cf[k][a] = __ldg(reinterpret_cast<const double2*>(coef + (size_t)a * M + s));
      zo[k] = __ldg(reinterpret_cast<const double2*>(z + s));
      po[k] = first ? make_double2(0.0, 0.0) : __ldg(reinterpret_cast<const double2*>(p_old + s));
    }
  }
#pragma unroll
  for (int k = 0; k < KH; ++k) {
    const int h = t + k * NT;
    zh[k] = 0.0;
    ph[k] = 0.0;
    if (h < 6 * F) {
      int f, ti, nl;
      halo_slot<CB>(h, f, ti, nl);
      const int nb = nbr_brick(g, bc, f);
      if (nb >= 0) {
        const size_t s = bofs(nb, C) + nl;
        zh[k] = __ldg(z + s);
        ph[k] = first ? 0.0 : __ldg(p_old + s);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int h = t + k * NT;
    ch[k] = 0.0;
    if (h < 3 * F) {
      const int ax = h / F, q = h % F, u = q % CB, w = q / CB;
      const int nb = nbr_brick(g, bc, 2 * ax);
      const int nl = ax == 0 ? (CB - 1) + CB * (u + CB * w)
                             : ax == 1 ? u + CB * ((CB - 1) + CB * w) : u + CB * (w + CB * (CB - 1));
      if (nb >= 0) ch[k] = __ldg(coef + (size_t)ax * M + bofs(nb, C) + nl);
    }
  }
  // stores
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int pr = t + k * NT;
    if (pr < NPAIR) {
      const int c = 2 * pr, li = c % CB, lj = (c / CB) % CB, lk = c / (CB * CB);
      *reinterpret_cast<double2*>(cs.cx + c) = cf[k][0];
      *reinterpret_cast<double2*>(cs.cy + c) = cf[k][1];
      *reinterpret_cast<double2*>(cs.cz + c) = cf[k][2];
      if (with_dg) *reinterpret_cast<double2*>(cs.dg + c) = cf[k][3];
      const int ti = Tile<CB>::idx(li, lj, lk);
      tile[ti] = first ? zo[k].x : zo[k].x + beta * po[k].x;
      tile[ti + 1] = first ? zo[k].y : zo[k].y + beta * po[k].y;
    }
  }
#pragma unroll
  for (int k = 0; k < KH; ++k) {
    const int h = t + k * NT;
    if (h < 6 * F) {
      int f, ti, nl;
      halo_slot<CB>(h, f, ti, nl);
      tile[ti] = first ? zh[k] : zh[k] + beta * ph[k];
    }
  }
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int h = t + k * NT;
    if (h < 3 * F) {
      const int ax = h / F, q = h % F;
      (ax == 0 ? cs.hx : ax == 1 ? cs.hy : cs.hz)[q] = ch[k];
    }
  }
}

// (A x)_c, branch-free: missing neighbours have T = 0 and a 0 halo value, so
// their -0 terms leave the sum bitwise unchanged; order and rounding are those
// of SparseOperator::apply on the assembled row (sparse.cpp:76-83).
// DG = false: the diagonal is summed from the six face coefficients in the
// assembly's face order (x-lo, x-hi, y-lo, y-hi, z-lo, z-hi; fvm.cpp:71-112,
// cell_faces) instead of read from cs.dg -- bitwise the stored diagonal of a
// cell without Dirichlet faces (a missing neighbour's T = 0 adds +0).
template <int CB, bool DG = true>
__device__ __forceinline__ double apply_coef(const CoefSmem<CB>& cs, const double* xt, int li, int lj,
                                             int lk) {
  constexpr int E = Tile<CB>::E;
  const int ti = Tile<CB>::idx(li, lj, lk);
  const int c = li + CB * (lj + CB * lk);
  const double* pz = lk > 0 ? cs.cz + (c - CB * CB) : cs.hz + (li + CB * lj);
  const double* py = lj > 0 ? cs.cy + (c - CB) : cs.hy + (li + CB * lk);
  const double* px = li > 0 ? cs.cx + (c - 1) : cs.hx + (lj + CB * lk);
  double s = __dadd_rn(0.0, __dmul_rn(-*pz, xt[ti - E * E]));
  s = __dadd_rn(s, __dmul_rn(-*py, xt[ti - E]));
  s = __dadd_rn(s, __dmul_rn(-*px, xt[ti - 1]));
  double dg;
  if constexpr (DG) dg = cs.dg[c];
  else
    dg = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(*px, cs.cx[c]), *py), cs.cy[c]), *pz), cs.cz[c]);
  s = __dadd_rn(s, __dmul_rn(dg, xt[ti]));
  s = __dadd_rn(s, __dmul_rn(-cs.cx[c], xt[ti + 1]));
  s = __dadd_rn(s, __dmul_rn(-cs.cy[c], xt[ti + E]));
  s = __dadd_rn(s, __dmul_rn(-cs.cz[c], xt[ti + E * E]));
  return s;
}

}  // namespace tmg
