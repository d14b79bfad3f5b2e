// Per-cc-element helpers shared by coarse.cu and coarse_large.cu: element
// coordinates, children (HierarchicalGrid::coarse_children, grid.cpp:183-194),
// the dense element matrix and the warp-parallel Jacobi eigensolver.
#pragma once
#include "kernels.h"

namespace tmg {

// L_c (basis vectors per coarse cell) is the runtime g.lc throughout the
// coarse level; kMaxLcCoarse bounds the register / shared arrays of
// k_coarse_blocks.
constexpr int kMaxLcCoarse = 6;

// ----------------------------------------------------- per-element helpers

struct ElemCoord {
  int64_t ei, ej, ek, e;
};
__device__ __forceinline__ ElemCoord elem_coord(const GridParams& g, int64_t e) {
  return {e % g.ncx, (e / g.ncx) % g.ncy, e / (g.ncx * g.ncy), e};
}
// coarse cell (brick) id of child c (di + sd*(dj + sd*dk)) of element E
// (HierarchicalGrid::coarse_children, grid.cpp:183-194)
__device__ __forceinline__ int64_t child_brick(const GridParams& g, const ElemCoord& ec, int c) {
  const int di = c % g.sd, dj = (c / g.sd) % g.sd, dk = c / (g.sd * g.sd);
  return (ec.ei * g.sd + di) + g.nbx * ((ec.ej * g.sd + dj) + g.nby * (ec.ek * g.sd + dk));
}
__device__ __forceinline__ int64_t brick_nbr(const GridParams& g, int64_t b, int dir /*0..5*/) {
  const int64_t bi = b % g.nbx, bj = (b / g.nbx) % g.nby, bk = b / (g.nbx * g.nby);
  switch (dir) {
    case 0: return bi > 0 ? b - 1 : -1;
    case 1: return bi + 1 < g.nbx ? b + 1 : -1;
    case 2: return bj > 0 ? b - g.nbx : -1;
    case 3: return bj + 1 < g.nby ? b + g.nbx : -1;
    case 4: return bk > 0 ? b - g.nbx * g.nby : -1;
    default: return bk + 1 < g.nbz ? b + g.nbx * g.nby : -1;
  }
}
// element-local child index of brick b, or -1 if b is not in element e
__device__ __forceinline__ int child_index(const GridParams& g, const ElemCoord& ec, int64_t b) {
  const int64_t bi = b % g.nbx, bj = (b / g.nbx) % g.nby, bk = b / (g.nbx * g.nby);
  const int64_t di = bi - ec.ei * g.sd, dj = bj - ec.ej * g.sd, dk = bk - ec.ek * g.sd;
  if (di < 0 || dj < 0 || dk < 0 || di >= g.sd || dj >= g.sd || dk >= g.sd) return -1;
  return (int)(di + g.sd * (dj + g.sd * dk));
}

// Element matrix (q x q, q = sd^3 * g.lc) into smem: A_c restricted to E's
// children, optionally minus Bc on diagonal blocks. Symmetrised.
__device__ inline void build_elem_matrix(const GridParams& g, const ElemCoord& ec, const double* Ac,
                                  const double* Bc, bool subtract_bc, double* M, int q) {
  const int nch = g.sd * g.sd * g.sd;
  for (int e = threadIdx.x; e < q * q; e += blockDim.x) M[e] = 0.0;
  __syncthreads();
  for (int e = threadIdx.x; e < nch * 7 * g.lc * g.lc; e += blockDim.x) {
    const int ci = e / (7 * g.lc * g.lc), rem = e % (7 * g.lc * g.lc);
    const int dir = rem / (g.lc * g.lc), ab = rem % (g.lc * g.lc), a = ab / g.lc, b = ab % g.lc;
    const int64_t I = child_brick(g, ec, ci);
    int cj;
    if (dir == 0) cj = ci;
    else {
      const int64_t J = brick_nbr(g, I, dir - 1);
      cj = J >= 0 ? child_index(g, ec, J) : -1;
    }
    if (cj < 0) continue;
    double v = Ac[(I * 7 + dir) * g.lc * g.lc + ab];
    if (dir == 0 && subtract_bc) v -= Bc[I * g.lc * g.lc + ab];
    M[(ci * g.lc + a) * q + cj * g.lc + b] = v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < q * q; e += blockDim.x) {
    const int i = e / q, j = e % q;
    if (i < j) {
      const double s = 0.5 * (M[i * q + j] + M[j * q + i]);
      M[i * q + j] = s;
      M[j * q + i] = s;
    }
  }
  __syncthreads();
}

// Warp-parallel Jacobi on q x q (q <= 64) symmetric M in smem; V (q x q)
// eigenvectors in columns. Lanes own rows r = lane, lane+32.
__device__ inline void warp_jacobi(double* M, double* V, int q) {
  // round-robin ("tournament") ordering: a sweep is Q-1 rounds of Q/2
  // disjoint rotations (Q = q rounded up to even: for odd q one player is a
  // bye, its pair is skipped); lane g computes rotation g of the round, then
  // every lane applies all of them to its rows / columns.
  __shared__ double rc[32], rs[32];
  __shared__ int rp[32], rq[32];
  const int lane = threadIdx.x & 31, Q = q + (q & 1), np = Q / 2;
  for (int r = lane; r < q; r += 32)
    for (int c = 0; c < q; ++c) V[r * q + c] = r == c ? 1.0 : 0.0;
  __syncwarp();
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int r = lane; r < q; r += 32)
      for (int c = 0; c < q; ++c) {
        const double v = M[r * q + c] * M[r * q + c];
        tot += v;
        if (r != c) off += v;
      }
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if (off <= 1e-26 * tot || off == 0.0) break;
    for (int round = 0; round < Q - 1; ++round) {
      if (lane < np) {  // circle method: player Q-1 fixed
        int p, qq;
        if (lane == 0) {
          p = round;
          qq = Q - 1;
        } else {
          p = (round + lane) % (Q - 1);
          qq = (round - lane + (Q - 1)) % (Q - 1);
        }
        if (p > qq) {
          const int tmp = p;
          p = qq;
          qq = tmp;
        }
        const bool bye = qq >= q;  // odd q: the pair with the bye player
        const double apq = bye ? 0.0 : M[p * q + qq];
        const double app = M[p * q + p], aqq = bye ? 0.0 : M[qq * q + qq];
        double c = 1.0, sn = 0.0;
        if (!bye && !(fabs(apq) <= 1e-300 || fabs(apq) <= 1e-18 * sqrt(fabs(app * aqq)))) {
          const double theta = (aqq - app) / (2.0 * apq);
          const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(tt * tt + 1.0);
          sn = tt * c;
        }
        rc[lane] = c;
        rs[lane] = sn;
        rp[lane] = p;
        rq[lane] = bye ? p : qq;  // a bye pair rotates p with itself by c = 1, s = 0
      }
      __syncwarp();
      for (int r = lane; r < q; r += 32)  // columns p, qq of row r (pairs disjoint)
        for (int g = 0; g < np; ++g) {
          const int p = rp[g], qq = rq[g];
          if (p == qq) continue;
          const double c = rc[g], sn = rs[g];
          const double akp = M[r * q + p], akq = M[r * q + qq];
          M[r * q + p] = c * akp - sn * akq;
          M[r * q + qq] = sn * akp + c * akq;
          const double vkp = V[r * q + p], vkq = V[r * q + qq];
          V[r * q + p] = c * vkp - sn * vkq;
          V[r * q + qq] = sn * vkp + c * vkq;
        }
      __syncwarp();
      for (int r = lane; r < q; r += 32)  // rows p, qq at column r
        for (int g = 0; g < np; ++g) {
          const int p = rp[g], qq = rq[g];
          if (p == qq) continue;
          const double c = rc[g], sn = rs[g];
          const double apk = M[p * q + r], aqk = M[qq * q + r];
          M[p * q + r] = c * apk - sn * aqk;
          M[qq * q + r] = sn * apk + c * aqk;
        }
      __syncwarp();
    }
  }
}

}  // namespace tmg
