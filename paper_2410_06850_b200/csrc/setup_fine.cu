// Set-up of the fine smoother factors (see smoother.cuh): per brick, the
// packed inverses G_k of the plane Schur complements of A_II.
#include "kernels.h"
#include "smoother.cuh"
#include "gj.cuh"

namespace tmg {

// One CTA per brick, NTF threads (256 at CB = 8: three CTAs per SM). Dynamic
// smem: 2 full P x P matrices + kappa tile + C pivots + P scratch x2.
template <int CB>
constexpr int factor_threads() { return CB == 8 ? 256 : CB * CB * CB; }

template <int CB>
__global__ void __launch_bounds__(factor_threads<CB>()) k_thomas_factor(GridParams g,
                                                               const double* __restrict__ kappa,
                                                               const uint8_t* __restrict__ dmask,
                                                               const int64_t* __restrict__ list,
                                                               double* G, int* status) {
  constexpr int P = Thomas<CB>::P, C = CB * CB * CB, NTF = factor_threads<CB>();
  constexpr int GP = P + 1;        // padded row stride of Gprev (conflict-free transpose)
  extern __shared__ double sm[];
  double* Gprev = sm;              // P*GP  previous plane inverse
  double* kt = Gprev + P * GP;     // tile (prologue only)
  double* fx = kt + Tile<CB>::N;   // 3 face arrays (prologue only)
  double* fy = fx + Tile<CB>::NF;
  double* fz = fy + Tile<CB>::NF;
  double* dg = fz + Tile<CB>::NF;  // C  diagonal of A
  double* tx = dg + C;             // C  T to +x neighbour in brick (0 if none)
  double* ty = tx + C;             // C
  double* tzb = ty + C;            // C  T to the cell one plane below (0 for lk=0)
  __shared__ double red[64];
  const BrickCoord bc = brick_coord(g, (int)list[blockIdx.x]);  // factor slot blockIdx.x
  load_tile<CB, true>(kappa, kt, g, bc);
  __syncthreads();
  tile_faces<CB>(kt, fx, fy, fz, g, bc);
  __syncthreads();
  const int t = threadIdx.x;
  for (int c = t; c < C; c += NTF) {
    const int li = c % CB, lj = (c / CB) % CB, lk = c / (CB * CB);
    const unsigned dm = brick_on_boundary(g, bc) ? dmask[bofs(bc.b, C) + c] : 0u;
    const FaceSet fs = cell_faces<CB>(fx, fy, fz, kt[Tile<CB>::idx(li, lj, lk)], li, lj, lk, g, bc, dm);
    dg[c] = fs.diag;
    tx[c] = li + 1 < CB ? fs.t[1] : 0.0;
    ty[c] = lj + 1 < CB ? fs.t[3] : 0.0;
    tzb[c] = lk > 0 ? fs.t[4] : 0.0;
  }
  __syncthreads();
  double* Gout = G + (size_t)blockIdx.x * Thomas<CB>::PER_BRICK;
  // Register-resident Gauss-Jordan per plane (gj.cuh)
  using L = GjLayout<P, NTF>;
  constexpr int CW = L::CW, RH = L::RH;
  const int lane = t & 31, c0 = CW * (t >> 5);
  const bool lane_active = lane < P;  // P < 32 (CB = 4): lanes >= P idle
  double pmin = 1e300, pmax = 0.0;    // this thread's pivots
  __shared__ GjSmem<P> gjs;
  for (int k = 0; k < CB; ++k) {
    // S = A_k - B_k Gprev B_k, B_k = diag(-tz) (own entries, in registers)
    double v[RH][CW];
#pragma unroll
    for (int h = 0; h < RH; ++h) {
      const int ri = lane_active ? lane + 32 * h : 0;
      const int ci = k * P + ri;
#pragma unroll
      for (int q = 0; q < CW; ++q) {
        const int j = c0 + q, cj = k * P + j;
        double a = 0.0;
        if (ri == j) a = dg[ci];
        else {
          const int ii = ri % CB, ij = ri / CB, ji = j % CB, jj = j / CB;
          if (ij == jj && ji == ii + 1) a = -tx[ci];
          else if (ij == jj && ii == ji + 1) a = -tx[cj];
          else if (ii == ji && jj == ij + 1) a = -ty[ci];
          else if (ii == ji && ij == jj + 1) a = -ty[cj];
        }
        if (k > 0) a -= tzb[ci] * Gprev[ri * GP + j] * tzb[cj];
        v[h][q] = a;
      }
    }
    __syncthreads();  // every thread has read Gprev
    gj_invert<P, NTF>(v, gjs, pmin, pmax);  // the LDL^T pivots of A_II (natural order)
    // symmetrise in place, store packed, keep the full copy for the next plane
    if (lane_active) {
#pragma unroll
      for (int h = 0; h < RH; ++h)
#pragma unroll
        for (int q = 0; q < CW; ++q) Gprev[(lane + 32 * h) * GP + c0 + q] = v[h][q];
    }
    __syncthreads();
    for (int e = t; e < P * P; e += NTF) {
      const int i = e / P, j = e % P;
      if (i < j) {
        const double m = 0.5 * (Gprev[i * GP + j] + Gprev[j * GP + i]);
        Gprev[i * GP + j] = m;
        Gprev[j * GP + i] = m;
      }
    }
    __syncthreads();
    // stored blocks in smoother.cuh's order and swizzle (block_of / plane_off);
    // packed diagonals: the off-diagonal blocks, then 40 doubles per diagonal block
    constexpr int NWHOLE = kDiagPacked ? Thomas<CB>::NOFF : Thomas<CB>::NBLK;
    for (int e = t; e < NWHOLE * 64; e += NTF) {
      const int blk = e / 64, rr = (e % 64) / 8, cc = e % 8;
      int I, J;
      block_of<CB>(blk, I, J);
      Gout[(size_t)k * Thomas<CB>::PLANE + plane_off(blk, rr, cc)] = Gprev[(8 * I + rr) * GP + 8 * J + cc];
    }
    if constexpr (kDiagPacked) {
      for (int e = t; e < Thomas<CB>::NBK * kDiagBlock; e += NTF) {
        const int d = e / kDiagBlock;
        int row, col;
        const bool stored = diag_slot(e % kDiagBlock, row, col);
        Gout[(size_t)k * Thomas<CB>::PLANE + NWHOLE * 64 + e] =
            stored ? Gprev[(8 * d + row) * GP + 8 * d + col] : 0.0;
      }
    }
    __syncthreads();
  }
  // reference singular-pivot rule over the block's pivots (solver.cpp:86-92):
  // every d > 1e-14 max|d|  <=>  min d > 1e-14 max|d|
  double mx = pmax, mn = pmin;
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if ((t & 31) == 0) {
    red[t >> 5] = mx;
    red[32 + (t >> 5)] = mn;
  }
  __syncthreads();
  if (t == 0) {
    double m = 0.0, n = 1e300;
    for (int w = 0; w < NTF / 32 || w == 0; ++w) {
      m = fmax(m, red[w]);
      n = fmin(n, red[32 + w]);
    }
    if (!(n > 1e-14 * m)) atomicExch(status, 1);
  }
}

size_t thomas_smem_bytes(int cb) {
  const int P = cb * cb, C = cb * cb * cb, N = (cb + 2) * (cb + 2) * (cb + 2);
  const int NF = (cb + 1) * cb * cb;
  return sizeof(double) * (size_t)(P * (P + 1) + N + 3 * NF + 4 * C);
}

void launch_thomas_factor(const GridParams& g, int cb, const double* kappa, const uint8_t* dmask,
                          const int64_t* list, int64_t nslots, double* G, int* status,
                          cudaStream_t s) {
  const size_t smem = thomas_smem_bytes(cb);
  if (nslots < 1) return;
  if (cb == 8) {
    ensure_dyn_smem(k_thomas_factor<8>, smem);
    k_thomas_factor<8><<<(unsigned)nslots, factor_threads<8>(), smem, s>>>(g, kappa, dmask, list,
                                                                           G, status);
  } else {
    ensure_dyn_smem(k_thomas_factor<4>, smem);
    k_thomas_factor<4><<<(unsigned)nslots, factor_threads<4>(), smem, s>>>(g, kappa, dmask, list,
                                                                           G, status);
  }
}

// An interior brick (all six neighbours exist) whose cells and six face halo
// layers carry bitwise the same conductivity k: every face T is
// face_t(k, k) * area/h and A_II = face_t(k, k) A_hat with A_hat fixed.
template <int CB>
__global__ void __launch_bounds__(256) k_uniform_bricks(GridParams g,
                                                       const double* __restrict__ kappa,
                                                       int* flag) {
  constexpr int C = CB * CB * CB;
  const BrickCoord bc = brick_coord(g, (int)(blockIdx.x + g.b0));
  __shared__ int same;
  const bool interior = bc.bi > 0 && bc.bj > 0 && bc.bk > 0 && bc.bi + 1 < g.nbx &&
                        bc.bj + 1 < g.nby && bc.bk + 1 < g.nbz;
  if (threadIdx.x == 0) same = interior ? 1 : 0;
  __syncthreads();
  if (!interior) {
    if (threadIdx.x == 0) flag[blockIdx.x] = 0;
    return;
  }
  const double k0 = kappa[bofs(bc.b, C)];
  bool ok = true;
  for (int t = threadIdx.x; t < C; t += blockDim.x) ok = ok && kappa[bofs(bc.b, C) + t] == k0;
  for (int h = threadIdx.x; h < 6 * CB * CB; h += blockDim.x) {
    int f, ti, nl;
    halo_slot<CB>(h, f, ti, nl);
    ok = ok && kappa[bofs(nbr_brick(g, bc, f), C) + nl] == k0;
  }
  if (!ok) same = 0;  // benign race: every writer stores 0
  __syncthreads();
  if (threadIdx.x == 0) flag[blockIdx.x] = same;
}

void launch_uniform_bricks(const GridParams& g, int cb, const double* kappa, int* flag,
                           cudaStream_t s) {
  if (cb == 8) k_uniform_bricks<8><<<(unsigned)g.nbo, 256, 0, s>>>(g, kappa, flag);
  else k_uniform_bricks<4><<<(unsigned)g.nbo, 64, 0, s>>>(g, kappa, flag);
}

// uniform bricks: A_II = face_t(k, k) A_hat, solved by fast diagonalisation
// of A_hat with scale 1 / face_t(k, k) (smoother.cuh, brick_inverse)
template <int CB>
__global__ void k_factor_scales(GridParams g, const double* __restrict__ kappa,
                                const int* __restrict__ flag, GSlot* map) {
  constexpr int C = CB * CB * CB;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= g.nbo) return;
  const int64_t b = g.b0 + i;
  const double kb = kappa[b * C];
  map[b].scale = flag[i] ? 1.0 / face_t(kb, kb) : 1.0;
}

void launch_factor_scales(const GridParams& g, int cb, const double* kappa, const int* flag,
                          GSlot* map, cudaStream_t s) {
  const unsigned grid = (unsigned)((g.nbo + 255) / 256);
  if (cb == 8) k_factor_scales<8><<<grid, 256, 0, s>>>(g, kappa, flag, map);
  else k_factor_scales<4><<<grid, 256, 0, s>>>(g, kappa, flag, map);
}

int64_t thomas_doubles_per_brick(int cb) {
  return cb == 8 ? Thomas<8>::PER_BRICK : Thomas<4>::PER_BRICK;
}

}  // namespace tmg
