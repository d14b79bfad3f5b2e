// Fine-level smoother: exact block-Jacobi with one block per coarse cell
// (north_star item 2).
//
// Reference semantics: BlockJacobiSmoother (proj/core/src/solver.cpp:128-251)
// with the partition {cells_of_coarse(I)} — one sweep from z = 0 gives
// z_I = A_II^{-1} r_I, the exact solve of the coarse cell's diagonal block of A.
// The reference factorises each block with Eigen LDL^T (solver.cpp:69-109); here
// each brick's block is factorised as a block-tridiagonal matrix over its CB
// z-planes (CB^2 cells each): S_0 = A_0, S_k = A_k - B_k S_{k-1}^{-1} B_k with
// B_k = diag(-T_z) the plane coupling, and the Schur inverses G_k = S_k^{-1}
// are stored densely. One solve is 2*CB-1 dense CB^2 x CB^2 mat-vecs — the
// same arithmetic as the LDL^T solve, reorganised into wide parallel steps.
// The pivots of the Gauss-Jordan sweeps are the LDL^T pivots of A_II in natural
// order; the reference's singular-pivot rule (d_i > 1e-14 max|d|,
// solver.cpp:86-92) is applied to them.
//
// Storage of one plane: the lower block-triangle of 8 x 8 blocks (I, J <= I),
// block index I(I+1)/2 + J, rows swizzled in 16-byte chunks (swz); diagonal
// blocks are kept whole. 36 blocks = 2304 doubles (18 KiB) per plane at
// CB = 8. Planes stream global -> shared through a ring of kSlots TMA bulk
// copies (cp.async.bulk + mbarrier complete_tx) issued kSlots plane-steps
// ahead. Each mat-vec thread owns one row of one block: it applies the row to
// w (row product, y_I) and — for off-diagonal blocks — its transpose (column
// products, y_J, reduce-scattered across the block's 8 lanes with shuffles).
// Every output row then has exactly NBK partial sums, added in a fixed order.
#pragma once
#include "stencil.cuh"
#include "tma.cuh"

namespace tmg {

template <int CB>
struct Thomas {
  static constexpr int P = CB * CB;                 // cells per plane
  static constexpr int NBK = P / 8;                 // 8-row block rows per plane
  static constexpr int NBLK = NBK * (NBK + 1) / 2;  // stored blocks per plane
  static constexpr int PLANE = NBLK * 64;           // doubles per plane
  static constexpr int PER_BRICK = CB * PLANE;      // doubles per brick
  static constexpr int NL = 2 * CB - 1;             // plane mat-vecs per solve
  static constexpr int MV = NBLK * 8;               // mat-vec threads
  static constexpr int NT = (MV + 31) / 32 * 32;    // CTA size of the solve kernels
  __host__ __device__ static constexpr int plane_of(int n) { return n < CB ? n : 2 * CB - 2 - n; }
  // storage offset of element (i, j), i, j < P (any order: symmetric)
  __host__ __device__ static constexpr int off(int i, int j) {
    return (i / 8 >= j / 8) ? (((i / 8) * (i / 8 + 1) / 2 + j / 8) * 64 + (i % 8) * 8 + j % 8)
                            : (((j / 8) * (j / 8 + 1) / 2 + i / 8) * 64 + (j % 8) * 8 + i % 8);
  }
};

// Storage / thread order of the 36 stored 8x8 blocks (I, J <= I) of a CB = 8
// plane, encoded 8*I + J. Chosen (offline search) so that the 4 blocks of each
// warp touch w and part[][] with the fewest shared-memory wavefronts: at most
// two distinct J (and I) per 64-byte bank half, I+J parities balanced 2/2.
static __constant__ unsigned char kBlockOrder8[36] = {44, 33, 41, 36, 60, 51, 59, 52, 17, 18, 25, 9, 26, 50, 63, 58, 24, 27, 16, 0, 57, 62, 54, 49, 45, 8, 32, 40, 61, 56, 53, 48, 34, 43, 42, 35};

template <int CB>
__device__ __forceinline__ void block_of(int blk, int& I, int& J) {
  if constexpr (CB == 8) {
    const int v = kBlockOrder8[blk];
    I = v >> 3;
    J = v & 7;
  } else {  // row-major lower block triangle
    I = 0;
    while ((I + 1) * (I + 2) / 2 <= blk) ++I;
    J = blk - I * (I + 1) / 2;
  }
}

// Swizzle inside an 8 x 8 block row: 16-byte chunk q (columns 2q, 2q+1) of
// row r is stored at chunk position (q + r/2) mod 4, so the 8 rows of a block
// read by one quarter-warp hit 8 distinct 16-byte bank groups.
__host__ __device__ constexpr int swz(int r, int c) {
  return r * 8 + 2 * (((c >> 1) + (r >> 1)) & 3) + (c & 1);
}

#ifndef TMG_SLOTS
#define TMG_SLOTS 2
#endif
constexpr int kSlots = TMG_SLOTS;  // TMA ring depth (planes in flight per CTA)
#ifndef TMG_G_HINTS
#define TMG_G_HINTS 1
#endif
// Forward-sweep planes requested into L2 ahead of the TMA ring (bulk L2
// prefetch: bytes in flight that hold no shared memory). 0 = off.
#ifndef TMG_L2_AHEAD
#define TMG_L2_AHEAD 0
#endif

// Plane load n of a solve: forward loads of planes the backward sweep re-reads
// ask L2 to keep them (evict_last); the last forward plane and the backward
// re-reads are last uses (evict_first).
__device__ __forceinline__ void plane_load(void* dst, const double* src, uint32_t bytes, uint64_t* bar,
                                           int n, int cb) {
#if TMG_G_HINTS
  bulk_g2s_hint(dst, src, bytes, bar, l2_policy(n < cb - 1));
#else
  bulk_g2s(dst, src, bytes, bar);
#endif
}

template <int CB>
using PlaneSlots = double[kSlots][Thomas<CB>::PLANE];

// Per-solve scratch; the TMA plane slots live separately (16-byte aligned,
// caller-owned) so kernels can alias them with data dead before the solve.
template <int CB>
struct ThomasSmem {
  alignas(16) double w2[2][CB * CB];  // read as double2 broadcasts
  // part[s][row]: contribution of block column s to a row (8-double pad keeps
  // the stores of a warp's 4 blocks in distinct bank halves by I+J parity)
  double part[Thomas<CB>::NBK][CB * CB + 8];
  uint64_t bars[kSlots];
  double (*slots)[Thomas<CB>::PLANE];
  // fast diagonalisation of uniform bricks (brick_inverse): the orthonormal
  // DST-I matrix Q[i][j] = sqrt(2/(CB+1)) sin(pi (i+1)(j+1)/(CB+1)) and the
  // eigenvalues 2 - 2 cos(pi (j+1)/(CB+1)) of the 1-D Dirichlet Laplacian
  double fdq[CB * CB];
  double fdl[CB];
};

template <int CB>
struct MvRole {
  int I, J, r, blk;
  bool active;
};

template <int CB>
__device__ __forceinline__ MvRole<CB> mv_role() {
  MvRole<CB> m;
  const int tid = threadIdx.x;
  m.active = tid < Thomas<CB>::MV;
  m.blk = m.active ? tid / 8 : 0;
  m.r = tid % 8;
  block_of<CB>(m.blk, m.I, m.J);
  return m;
}

// 8-lane reduce-scatter: lane r (of an aligned group of 8) returns sum over the
// group's lanes of b[r].
__device__ __forceinline__ double reduce_scatter8(double (&b)[8], int r) {
  const bool h4 = r & 4, h2 = r & 2, h1 = r & 1;
  double c4[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double send = h4 ? b[k] : b[k + 4];
    const double keep = h4 ? b[k + 4] : b[k];
    c4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  double c2[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double send = h2 ? c4[k] : c4[k + 2];
    const double keep = h2 ? c4[k + 2] : c4[k];
    c2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  const double send = h1 ? c2[0] : c2[1];
  const double keep = h1 ? c2[1] : c2[0];
  return keep + __shfl_xor_sync(0xffffffffu, send, 1);
}

// One plane mat-vec step: partial products into part[][].
template <int CB>
__device__ __forceinline__ void mv_partials(ThomasSmem<CB>& sm, const double* Gp, const double* w,
                                            const MvRole<CB>& m) {
  // whole warps take part (the shuffles below need every lane)
  if ((int)(threadIdx.x >> 5) >= (Thomas<CB>::MV + 31) / 32) return;
  const bool off_diag = m.active && m.J < m.I;
  double gv[8];
  const uint32_t row = smem_u32(Gp + m.blk * 64);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double2 v;  // explicit ld.shared: the slot pointer is opaque to the compiler
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "r"(row + (uint32_t)(swz(m.r, 2 * q) * sizeof(double))));
    gv[2 * q] = v.x;
    gv[2 * q + 1] = v.y;
  }
  double a0 = 0.0, a1 = 0.0;  // two chains halve the dependent-FMA latency
#pragma unroll
  for (int c = 0; c < 8; c += 2) {
    const double2 wv = *reinterpret_cast<const double2*>(w + 8 * m.J + c);  // broadcast
    a0 = fma(gv[c], wv.x, a0);
    a1 = fma(gv[c + 1], wv.y, a1);
  }
  if (m.active) sm.part[m.J][8 * m.I + m.r] = a0 + a1;
  // transposed block; diagonal blocks (and idle lanes) contribute zeros
  const double wr = off_diag ? w[8 * m.I + m.r] : 0.0;
  double b[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) b[c] = gv[c] * wr;
  const double cs = reduce_scatter8(b, m.r);
  if (off_diag) sm.part[m.I][8 * m.J + m.r] = cs;
}

template <int CB>
__device__ __forceinline__ void thomas_init(ThomasSmem<CB>& sm) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < kSlots; ++s) mbar_init(&sm.bars[s], 1);
    fence_barrier_init();
  }
  for (int e = threadIdx.x; e < CB * CB; e += blockDim.x) {
    const int i = e / CB, j = e % CB;
    sm.fdq[e] = sqrt(2.0 / (CB + 1)) * sinpi((double)((i + 1) * (j + 1)) / (CB + 1));
    if (i == 0) sm.fdl[j] = 2.0 - 2.0 * cospi((double)(j + 1) / (CB + 1));
  }
}

// Issue the first kSlots plane loads of a solve (thread 0). Call after
// thomas_init + __syncthreads, as early as possible in the kernel.
template <int CB>
__device__ __forceinline__ void thomas_prefetch(ThomasSmem<CB>& sm, const double* __restrict__ G) {
  if (!G) return;  // uniform brick: no factor planes (brick_inverse)
  // resident mode (kSlots >= CB): all CB planes stay in shared memory and the
  // backward sweep reuses them; otherwise a ring refilled kSlots steps ahead.
  constexpr int NPRE = kSlots >= CB ? CB : kSlots;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int n = 0; n < NPRE && n < Thomas<CB>::NL; ++n) {
      mbar_arrive_expect_tx(&sm.bars[n], Thomas<CB>::PLANE * sizeof(double));
      plane_load(sm.slots[n], G + (size_t)Thomas<CB>::plane_of(n) * Thomas<CB>::PLANE,
                 Thomas<CB>::PLANE * sizeof(double), &sm.bars[n], n, CB);
    }
#if TMG_L2_AHEAD > 0
#pragma unroll
    for (int n = NPRE; n < NPRE + TMG_L2_AHEAD && n < CB; ++n)
      prefetch_l2(G + (size_t)n * Thomas<CB>::PLANE, Thomas<CB>::PLANE * sizeof(double));
#endif
  }
}

// Wait for the loads thomas_prefetch issued (a CTA that exits early must not
// leave bulk copies in flight into its shared memory).
template <int CB>
__device__ __forceinline__ void thomas_drain(ThomasSmem<CB>& sm, const double* G) {
  constexpr int NPRE = kSlots >= CB ? CB : kSlots;
  if (threadIdx.x == 0 && G)
    for (int n = 0; n < NPRE && n < Thomas<CB>::NL; ++n) mbar_wait(&sm.bars[n], 0);
}

// Exact block solve x = A_II^{-1} t for one brick (after thomas_prefetch).
//  t  : smem, C values (plane k = t[k*P .. k*P+P)); x must alias t (the
//       forward sweep keeps u_k in x, over the consumed t_k)
//  tz : smem, C values; tz[l] = T_z between cell l and the cell one plane below
// Thread i < P reads t[i] before the first __syncthreads: plane 0 of t must
// be complete (written by thread i itself, or published by a caller barrier).
// Ends with a __syncthreads.
// scale: every plane mat-vec result is multiplied by it (the shared factor
// of a uniform brick, FineFactors; 1.0 leaves the solve bitwise unchanged).
template <int CB>
__device__ __forceinline__ void thomas_solve(ThomasSmem<CB>& sm, const double* __restrict__ G,
                                             const double* t, const double* tz, double* x,
                                             double scale = 1.0) {
  constexpr int P = Thomas<CB>::P, NL = Thomas<CB>::NL, NBK = Thomas<CB>::NBK;
  const int tid = threadIdx.x;
  const MvRole<CB> m = mv_role<CB>();
  constexpr bool resident = kSlots >= CB;
  auto slot_of = [](int n) { return resident ? Thomas<CB>::plane_of(n) : n % kSlots; };
  auto parity_of = [](int n) { return resident ? 0u : (uint32_t)((n / kSlots) & 1); };
  // The last warp issues the TMA refills and waits for the next plane before
  // each step's closing barrier, which then publishes "plane ready" to all.
  const bool waiter = tid >= (int)blockDim.x - 32;
  const bool issuer = tid == (int)blockDim.x - 32;
  if (waiter) mbar_wait(&sm.bars[slot_of(0)], parity_of(0));
  if (tid < P) sm.w2[0][tid] = t[tid];
  __syncthreads();
#pragma unroll 1
  for (int n = 0; n < NL; ++n) {
    const int slot = slot_of(n);
    mv_partials<CB>(sm, sm.slots[slot], sm.w2[n & 1], m);
    __syncthreads();
    // slot consumed by every thread: refill it with the plane kSlots steps ahead
    if (!resident && issuer && n + kSlots < NL) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&sm.bars[slot], Thomas<CB>::PLANE * sizeof(double));
      plane_load(sm.slots[slot], G + (size_t)Thomas<CB>::plane_of(n + kSlots) * Thomas<CB>::PLANE,
                 Thomas<CB>::PLANE * sizeof(double), &sm.bars[slot], n + kSlots, CB);
#if TMG_L2_AHEAD > 0
      if (n + kSlots + TMG_L2_AHEAD < CB)
        prefetch_l2(G + (size_t)(n + kSlots + TMG_L2_AHEAD) * Thomas<CB>::PLANE,
                    Thomas<CB>::PLANE * sizeof(double));
#endif
    }
    if (tid < P) {
      double pr[NBK];
#pragma unroll
      for (int s = 0; s < NBK; ++s) pr[s] = sm.part[s][tid];
#pragma unroll
      for (int w = 1; w < NBK; w *= 2)  // fixed pairwise tree
#pragma unroll
        for (int s = 0; s + w < NBK; s += 2 * w) pr[s] += pr[s + w];
      const double acc = pr[0] * scale;
      double* wn = sm.w2[(n + 1) & 1];
      const int row = tid;
      if (n < CB) {  // forward: u_k = G_k w_k ; w_{k+1} = t_{k+1} + Tz_{k+1} u_k
        const int l = n * P + row;
        x[l] = acc;  // u_k overwrites t_k, dead since step k-1 formed w_k
        if (n + 1 < CB) {
          wn[row] = fma(tz[l + P], acc, t[l + P]);
        } else {  // x_{K-1} = u_{K-1};  first backward w = -Tz_{K-1} x_{K-1}
          wn[row] = -tz[l] * acc;
        }
      } else {  // backward plane k: x_k = u_k - G_k (B_{k+1} x_{k+1})
        const int k = Thomas<CB>::plane_of(n);
        const int l = k * P + row;
        const double xv = x[l] - acc;  // u_k - G_k B_{k+1} x_{k+1}
        x[l] = xv;
        if (k > 0) wn[row] = -tz[l] * xv;
      }
    }
    if (waiter && n + 1 < NL && (!resident || n + 1 < CB))
      mbar_wait(&sm.bars[slot_of(n + 1)], parity_of(n + 1));
    __syncthreads();
  }
}

// x = A_II^-1 t of an interior brick of one conductivity k (cells and face
// halo): A_II = face_t(k, k) sum_ax (area/h)_ax K_ax with K the 1-D Dirichlet
// Laplacian tridiag(-1, 2, -1) along each axis (every face of every cell,
// inside and to the neighbours, carries face_t(k, k) area/h), so
//   A_II^-1 = scale (Q x Q x Q) diag(1 / sum_ax (area/h)_ax lambda_ax) (Q x Q x Q),
// scale = 1 / face_t(k, k), Q the symmetric orthonormal DST-I: six 8-point
// transforms and a division instead of the 15 dependent plane mat-vecs. w:
// C doubles of scratch. Starts and ends with a __syncthreads; x aliases t.
template <int CB>
__device__ __forceinline__ void fastdiag_solve(const ThomasSmem<CB>& sm, double* t, double* w,
                                               double scale, const double* cpl) {
  constexpr int C = CB * CB * CB;
  const int tid = threadIdx.x, nt = blockDim.x;
  // one transform along axis ax (stride st) from src to dst
  auto transform = [&](const double* src, double* dst, int st) {
    __syncthreads();
    for (int o = tid; o < C; o += nt) {
      const int io = (o / st) % CB, base = o - io * st;
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < CB; ++i) v = fma(sm.fdq[i * CB + io], src[base + i * st], v);
      dst[o] = v;
    }
  };
  transform(t, w, 1);
  transform(w, t, CB);
  transform(t, w, CB * CB);
  __syncthreads();
  for (int o = tid; o < C; o += nt) {
    const int i = o % CB, j = (o / CB) % CB, k = o / (CB * CB);
    w[o] *= scale / (cpl[0] * sm.fdl[i] + cpl[1] * sm.fdl[j] + cpl[2] * sm.fdl[k]);
  }
  transform(w, t, CB * CB);
  transform(t, w, CB);
  transform(w, t, 1);
  __syncthreads();
}

// The exact block solve of one brick: the plane-factor block Thomas (G), or
// the fast diagonalisation of a uniform interior brick (G == nullptr, tz
// used as scratch).
template <int CB>
__device__ __forceinline__ void brick_inverse(ThomasSmem<CB>& sm, const double* G, double* t,
                                              double* tz, double scale, const GridParams& g) {
  if (G) thomas_solve<CB>(sm, G, t, tz, t, scale);
  else fastdiag_solve<CB>(sm, t, tz, scale, g.cpl);
}

}  // namespace tmg
