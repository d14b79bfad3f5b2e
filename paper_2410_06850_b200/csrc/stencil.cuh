// Matrix-free TPFA operator on a brick tile (north_star item 1).
//
// The operator is the reference's cell-centred two-point flux approximation
// (proj/core/src/fvm.cpp:33-166): T_F = 2 k1 k2/(k1+k2) * area/h per interior
// face, 2 k_c * area/h per Dirichlet boundary face on the diagonal, nothing on
// Neumann faces. It is never materialised: each CTA stages the conductivity and
// the input vector of its brick plus a one-cell face halo in shared memory and
// recomputes the face transmissibilities in registers. The diagonal is summed
// in the reference's face order (x-lo, x-hi, y-lo, y-hi, z-lo, z-hi,
// fvm.cpp:71-112) and the row product in its sorted-column order
// (z-lo, y-lo, x-lo, diag, x-hi, y-hi, z-hi; sparse.cpp:76-83) without FMA
// contraction, so y = A x is bitwise equal to SparseOperator::apply on the
// assembled CSR.
#pragma once
#include "common.cuh"

namespace tmg {

template <int CB>
struct Tile {
  static constexpr int E = CB + 2;
  static constexpr int N = E * E * E;
  static constexpr int C = CB * CB * CB;
  __device__ static __forceinline__ int idx(int i, int j, int k) {
    return (i + 1) + E * ((j + 1) + E * (k + 1));
  }
};

struct BrickCoord {
  int64_t bi, bj, bk, b;
};

__device__ __forceinline__ BrickCoord brick_coord(const GridParams& g, int64_t b) {
  BrickCoord c;
  c.b = b;
  c.bi = b % g.nbx;
  c.bj = (b / g.nbx) % g.nby;
  c.bk = b / (g.nbx * g.nby);
  return c;
}

// Load v's brick values into tile interior; if HALO, also the six face layers
// from the neighbouring bricks (0 outside the domain). Caller syncs.
template <int CB, bool HALO>
__device__ __forceinline__ void load_tile(const double* __restrict__ v, double* tile,
                                          const GridParams& g, const BrickCoord& bc) {
  constexpr int C = CB * CB * CB;
  constexpr int F = CB * CB;
  const int t = threadIdx.x;
  {
    const int li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
    tile[Tile<CB>::idx(li, lj, lk)] = __ldg(v + bc.b * C + t);
  }
  if (HALO) {
    for (int s = t; s < 6 * F; s += C) {
      const int f = s / F, q = s % F;
      const int u = q % CB, w = q / CB;
      int64_t nbrick = -1;
      int li = 0, lj = 0, lk = 0, ti = 0, tj = 0, tk = 0;
      switch (f) {
        case 0:  // x-lo halo: neighbour bi-1, its li = CB-1
          if (bc.bi > 0) nbrick = bc.b - 1;
          li = CB - 1; lj = u; lk = w; ti = -1; tj = u; tk = w; break;
        case 1:
          if (bc.bi + 1 < g.nbx) nbrick = bc.b + 1;
          li = 0; lj = u; lk = w; ti = CB; tj = u; tk = w; break;
        case 2:
          if (bc.bj > 0) nbrick = bc.b - g.nbx;
          li = u; lj = CB - 1; lk = w; ti = u; tj = -1; tk = w; break;
        case 3:
          if (bc.bj + 1 < g.nby) nbrick = bc.b + g.nbx;
          li = u; lj = 0; lk = w; ti = u; tj = CB; tk = w; break;
        case 4:
          if (bc.bk > 0) nbrick = bc.b - g.nbx * g.nby;
          li = u; lj = w; lk = CB - 1; ti = u; tj = w; tk = -1; break;
        default:
          if (bc.bk + 1 < g.nbz) nbrick = bc.b + g.nbx * g.nby;
          li = u; lj = w; lk = 0; ti = u; tj = w; tk = CB; break;
      }
      tile[Tile<CB>::idx(ti, tj, tk)] =
          nbrick >= 0 ? __ldg(v + nbrick * C + (li + CB * (lj + CB * lk))) : 0.0;
    }
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
__device__ __forceinline__ FaceSet cell_faces(const double* kt, int li, int lj, int lk,
                                              const GridParams& g, const BrickCoord& bc,
                                              unsigned dmask) {
  constexpr int E = Tile<CB>::E;
  const int ti = Tile<CB>::idx(li, lj, lk);
  const double kc = kt[ti];
  const int64_t gi = bc.bi * CB + li, gj = bc.bj * CB + lj, gk = bc.bk * CB + lk;
  const bool has[6] = {gi > 0, gi < g.nx - 1, gj > 0, gj < g.ny - 1, gk > 0, gk < g.nz - 1};
  const int off[6] = {-1, 1, -E, E, -E * E, E * E};
  FaceSet fs;
  fs.nbmask = 0;
  double diag = 0.0;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const double cp = g.cpl[f >> 1];
    double t;
    if (has[f]) {
      const double kn = kt[ti + off[f]];
      // low side: face_transmissibility(k[nb], k[c]); high: (k[c], k[nb])
      t = (f & 1) ? __dmul_rn(face_t(kc, kn), cp) : __dmul_rn(face_t(kn, kc), cp);
      fs.nbmask |= 1 << f;
      diag = __dadd_rn(diag, t);
    } else if (dmask & (1u << f)) {
      t = __dmul_rn(__dmul_rn(2.0, kc), cp);
      diag = __dadd_rn(diag, t);
    } else {
      t = 0.0;
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

}  // namespace tmg
