// Set-up of the fine smoother factors (see smoother.cuh): per brick, the
// packed inverses G_k of the plane Schur complements of A_II.
#include "kernels.h"
#include "smoother.cuh"

namespace tmg {

// One CTA per brick, C = CB^3 threads. Dynamic smem: 2 full P x P matrices +
// kappa tile + C pivots + P scratch x2.
template <int CB>
__global__ void __launch_bounds__(CB * CB * CB) k_thomas_factor(GridParams g,
                                                               const double* __restrict__ kappa,
                                                               const uint8_t* __restrict__ dmask,
                                                               double* G, int* status) {
  constexpr int P = Thomas<CB>::P, C = CB * CB * CB;
  extern __shared__ double sm[];
  double* S = sm;                  // P*P  current Schur complement -> inverse
  double* Gprev = S + P * P;       // P*P  previous plane inverse
  double* kt = Gprev + P * P;      // tile
  double* fx = kt + Tile<CB>::N;   // 3 face arrays
  double* fy = fx + Tile<CB>::NF;
  double* fz = fy + Tile<CB>::NF;
  double* piv = fz + Tile<CB>::NF; // C
  double* col = piv + C;           // P
  double* rowp = col + P;          // P
  double* dg = rowp + P;           // C  diagonal of A
  double* tx = dg + C;             // C  T to +x neighbour in brick (0 if none)
  double* ty = tx + C;             // C
  double* tzb = ty + C;            // C  T to the cell one plane below (0 for lk=0)
  __shared__ double red[64];
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  load_tile<CB, true>(kappa, kt, g, bc);
  __syncthreads();
  tile_faces<CB>(kt, fx, fy, fz, g, bc);
  __syncthreads();
  const int t = threadIdx.x, li = t % CB, lj = (t / CB) % CB, lk = t / (CB * CB);
  {
    const unsigned dm = brick_on_boundary(g, bc) ? dmask[bofs(bc.b, C) + t] : 0u;
    const FaceSet fs = cell_faces<CB>(fx, fy, fz, kt[Tile<CB>::idx(li, lj, lk)], li, lj, lk, g, bc, dm);
    dg[t] = fs.diag;
    tx[t] = li + 1 < CB ? fs.t[1] : 0.0;
    ty[t] = lj + 1 < CB ? fs.t[3] : 0.0;
    tzb[t] = lk > 0 ? fs.t[4] : 0.0;
  }
  __syncthreads();
  double* Gout = G + (size_t)bc.b * Thomas<CB>::PER_BRICK;
  for (int k = 0; k < CB; ++k) {
    // S = A_k - B_k Gprev B_k, B_k = diag(-tz)
    for (int e = t; e < P * P; e += C) {
      const int i = e / P, j = e % P;
      const int ci = k * P + i, cj = k * P + j;
      double v = 0.0;
      if (i == j) v = dg[ci];
      else {
        const int ii = i % CB, ij = i / CB, ji = j % CB, jj = j / CB;
        if (ij == jj && ji == ii + 1) v = -tx[ci];
        else if (ij == jj && ii == ji + 1) v = -tx[cj];
        else if (ii == ji && jj == ij + 1) v = -ty[ci];
        else if (ii == ji && ij == jj + 1) v = -ty[cj];
      }
      if (k > 0) v -= tzb[ci] * Gprev[e] * tzb[cj];
      S[e] = v;
    }
    __syncthreads();
    // in-place Gauss-Jordan sweep inversion (SPD, no pivoting)
    for (int p = 0; p < P; ++p) {
      const double pv = S[p * P + p];
      if (t < P) {
        col[t] = S[t * P + p];
        rowp[t] = S[p * P + t];
      }
      if (t == 0) piv[k * P + p] = pv;
      __syncthreads();
      const double inv = 1.0 / pv;
      for (int e = t; e < P * P; e += C) {
        const int i = e / P, j = e % P;
        double v;
        if (i == p && j == p) v = inv;
        else if (i == p) v = rowp[j] * inv;
        else if (j == p) v = -col[i] * inv;
        else v = S[e] - col[i] * (rowp[j] * inv);
        S[e] = v;
      }
      __syncthreads();
    }
    // symmetrise, store packed, keep full copy for the next plane
    for (int e = t; e < P * P; e += C) {
      const int i = e / P, j = e % P;
      Gprev[e] = 0.5 * (S[e] + S[j * P + i]);
    }
    __syncthreads();
    // lower block-triangle of 8 x 8 blocks, block (I, J <= I) at I(I+1)/2 + J
    for (int e = t; e < Thomas<CB>::PLANE; e += C) {
      const int blk = e / 64, rr = (e % 64) / 8, cc = e % 8;
      int I, J;
      block_of<CB>(blk, I, J);
      Gout[(size_t)k * Thomas<CB>::PLANE + blk * 64 + swz(rr, cc)] = Gprev[(8 * I + rr) * P + 8 * J + cc];
    }
    __syncthreads();
  }
  // reference singular-pivot rule over the block's pivots (solver.cpp:86-92)
  double mx = fabs(piv[t]);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((t & 31) == 0) red[t >> 5] = mx;
  __syncthreads();
  if (t == 0) {
    double m = 0.0;
    for (int w = 0; w < C / 32 || w == 0; ++w) m = fmax(m, red[w]);
    red[32] = m;
  }
  __syncthreads();
  if (!(piv[t] > 1e-14 * red[32])) atomicExch(status, 1);
}

size_t thomas_smem_bytes(int cb) {
  const int P = cb * cb, C = cb * cb * cb, N = (cb + 2) * (cb + 2) * (cb + 2);
  const int NF = (cb + 1) * cb * cb;
  return sizeof(double) * (size_t)(2 * P * P + N + 3 * NF + C + 2 * P + 4 * C);
}

void launch_thomas_factor(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                          double* G, int* status, cudaStream_t s) {
  const size_t smem = thomas_smem_bytes(cb);
  if (cb == 8) {
    cudaFuncSetAttribute(k_thomas_factor<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_thomas_factor<8><<<(unsigned)g.nbo, 512, smem, s>>>(g, kappa, dmask, G, status);
  } else {
    cudaFuncSetAttribute(k_thomas_factor<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_thomas_factor<4><<<(unsigned)g.nbo, 64, smem, s>>>(g, kappa, dmask, G, status);
  }
}

int64_t thomas_doubles_per_brick(int cb) {
  return cb == 8 ? Thomas<8>::PER_BRICK : Thomas<4>::PER_BRICK;
}

}  // namespace tmg
