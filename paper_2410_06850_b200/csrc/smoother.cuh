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
// block order kBlockOrder8, rows swizzled in 16-byte chunks (plane_off); diagonal
// blocks are kept whole. 36 blocks = 2304 doubles (18 KiB) per plane at
// CB = 8. Planes stream global -> shared through a ring of kSlots TMA bulk
// copies (cp.async.bulk + mbarrier complete_tx) issued kSlots plane-steps
// ahead. Each mat-vec thread owns R rows of one block (TMG_MV_ROWS, default
// 2): it applies them to w (row products, y_I) and — for off-diagonal blocks
// — their transposes (column products, y_J, reduce-scattered across the
// block's 8/R lanes with shuffles). Every output row then has exactly NBK
// partial sums, added in a fixed order.
#pragma once
#include "stencil.cuh"
#include "tma.cuh"

namespace tmg {

// Rows of an 8 x 8 block owned by one mat-vec thread (1, 2 or 4). The solve is
// bound by shared-memory wavefronts (TMA plane write 144 + plane read 144 per
// step are fixed; the column-product shuffles, 14 per thread at one row per
// thread, are not): R rows per thread reduce-scatter over 8/R lanes only,
// 126 -> 54 (R = 2) -> 18 (R = 4) shuffle wavefronts per plane step, and the
// CTA shrinks to 160 / 96 threads.
#ifndef TMG_MV_ROWS
#define TMG_MV_ROWS 2
#endif
constexpr int kMvRows = TMG_MV_ROWS;
constexpr int kMvTpb = 8 / kMvRows;  // threads per 8 x 8 block
static_assert(kMvRows == 1 || kMvRows == 2 || kMvRows == 4, "TMG_MV_ROWS");
// Opt-in (TMG_DIAG_PACK=1): diagonal 8 x 8 blocks stored as their lower
// triangle (two rows per thread only): 40 instead of 64 doubles per block,
// 2112 instead of 2304 per CB = 8 plane (264 instead of 288 B/cell of factor
// traffic, 2.4 GB less at 512^3). The diagonal blocks get a warp of their own
// (mv_partials_diag). Measured at configs[3]: the same time per iteration
// (21.82 against 21.77 ms) -- a plane step is bound by its per-warp chain and
// shared-memory wavefronts (quarter-warp granular, so the predicated loads
// save none), not by the plane's bytes -- so the whole-block layout stays the
// default.
#ifndef TMG_DIAG_PACK
#define TMG_DIAG_PACK 0
#endif
constexpr bool kDiagPacked = TMG_DIAG_PACK && kMvRows == 2;
constexpr int kDiagBlock = kDiagPacked ? 40 : 64;  // stored doubles per diagonal block

template <int CB>
struct Thomas {
  static constexpr int P = CB * CB;                 // cells per plane
  static constexpr int NBK = P / 8;                 // 8-row block rows per plane
  static constexpr int NBLK = NBK * (NBK + 1) / 2;  // stored blocks per plane
  static constexpr int NOFF = NBK * (NBK - 1) / 2;  // of which off-diagonal
  // doubles per plane: the off-diagonal blocks first, then the diagonal ones
  static constexpr int PLANE = kDiagPacked ? NOFF * 64 + NBK * kDiagBlock : NBLK * 64;
  static constexpr int PER_BRICK = CB * PLANE;      // doubles per brick
  static constexpr int NL = 2 * CB - 1;             // plane mat-vecs per solve
  // mat-vec threads: packed diagonals start at a warp boundary (DW)
  static constexpr int DW = kDiagPacked ? (NOFF * kMvTpb + 31) / 32 * 32 : 0;
  static constexpr int MV = kDiagPacked ? DW + NBK * kMvTpb : NBLK * kMvTpb;
  static constexpr int NT = (MV + 31) / 32 * 32;    // CTA size of the solve kernels
  __host__ __device__ static constexpr int plane_of(int n) { return n < CB ? n : 2 * CB - 2 - n; }
};

// Storage / thread order of the 36 stored 8x8 blocks (I, J <= I) of a CB = 8
// plane, encoded 8*I + J.
// One row per thread (4 blocks per warp): chosen (offline search) so that the
// 4 blocks of each warp touch w and part[][] with the fewest shared-memory
// wavefronts: at most two distinct J (and I) per 64-byte bank half, I+J
// parities balanced 2/2.
// Two or four rows per thread (8 / 16 blocks per warp): block columns, so a
// warp's blocks share w_J (broadcast loads) and their row products land in
// one contiguous run of part[J][]: warp 0 = column 0, warp 1 = column 1 +
// (7,7), warp 2 = columns 2 + 6, warp 3 = columns 3 + 5, warp 4 = column 4.
// Packed diagonals: the 28 off-diagonal blocks only, block columns again:
// warp 0 = column 0 + (7,6), warp 1 = columns 1 + 5, warp 2 = columns 2 + 4,
// warp 3 = column 3; the diagonal blocks (I, I) follow in order of I.
static __constant__ unsigned char kBlockOrder8[36] =
#if TMG_MV_ROWS == 1
    {44, 33, 41, 36, 60, 51, 59, 52, 17, 18, 25, 9, 26, 50, 63, 58, 24, 27, 16, 0, 57, 62, 54, 49, 45, 8, 32, 40, 61, 56, 53, 48, 34, 43, 42, 35};
#elif TMG_DIAG_PACK && TMG_MV_ROWS == 2
    {8, 16, 24, 32, 40, 48, 56, 62, 17, 25, 33, 41, 49, 57, 53, 61, 26, 34, 42, 50, 58, 44, 52, 60,
     35, 43, 51, 59, 0, 9, 18, 27, 36, 45, 54, 63};
#else
    {0, 8, 16, 24, 32, 40, 48, 56, 9, 17, 25, 33, 41, 49, 57, 63, 18, 26, 34, 42, 50, 58, 54, 62,
     27, 35, 43, 51, 59, 45, 53, 61, 36, 44, 52, 60};
#endif

template <int CB>
__device__ __forceinline__ void block_of(int blk, int& I, int& J) {
  if constexpr (CB == 8) {
    const int v = kBlockOrder8[blk];
    I = v >> 3;
    J = v & 7;
  } else if constexpr (kDiagPacked) {  // strictly lower blocks row-major, then the diagonal
    constexpr int NOFF = Thomas<CB>::NOFF;
    if (blk >= NOFF) {
      I = J = blk - NOFF;
    } else {
      I = 1;
      while (I * (I + 1) / 2 <= blk) ++I;
      J = blk - I * (I - 1) / 2;
    }
  } else {  // row-major lower block triangle
    I = 0;
    while ((I + 1) * (I + 2) / 2 <= blk) ++I;
    J = blk - I * (I + 1) / 2;
  }
}

// Position (in 16-byte chunks) of a mat-vec thread's k-th 128-bit load inside
// its R-row region of a block (R * 64 bytes, R * 4 chunks; chunk k holds
// columns 2 (k % 4), +1 of the thread's row k / 4). `sub` is the thread's
// index inside the block, `tid` its mat-vec thread index (blk * 8/R + sub).
//  R = 1: chunk q of row r sits at (q + r/2) mod 4, so the 8 rows of a block
//         read by one quarter-warp hit 8 distinct 16-byte bank groups;
//  R >= 2: a region spans all 8 bank groups; load k of the thread at
//         quarter-warp position tid % 8 is rotated by that position.
__host__ __device__ constexpr int mv_chunk_pos(int k, int sub, int tid) {
  return kMvRows == 1 ? ((k + (sub >> 1)) & 3) : ((k & ~7) | ((k + (tid & 7)) & 7));
}

// Storage offset (doubles) of element (r, c) of stored block `blk` in a plane
// (whole blocks: every block, or the off-diagonal ones with packed diagonals).
__host__ __device__ constexpr int plane_off(int blk, int r, int c) {
  const int sub = r / kMvRows, k = (r % kMvRows) * 4 + (c >> 1);
  return blk * 64 + sub * 8 * kMvRows + 2 * mv_chunk_pos(k, sub, blk * kMvTpb + sub) + (c & 1);
}

// Packed diagonal block (40 doubles): thread `sub` of the block owns rows
// 2 sub and 2 sub + 1; its region starts at 2 sub (sub + 1) doubles and holds
// row 2 sub, columns 0 .. 2 sub + 1 (the last one, above the diagonal, stored
// as 0), then row 2 sub + 1, columns 0 .. 2 sub + 1.
// diag_slot: the element (row, col) stored at slot s of a packed block;
// returns false for the zero pads.
__host__ __device__ constexpr int diag_region(int sub) { return 2 * sub * (sub + 1); }
__host__ __device__ constexpr bool diag_slot(int s, int& row, int& col) {
  int sub = 0;
  while (sub < 3 && s >= diag_region(sub + 1)) ++sub;
  const int o = s - diag_region(sub), len = 2 * sub + 2;
  row = o < len ? 2 * sub : 2 * sub + 1;
  col = o < len ? o : o - len;
  return col <= row;
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
  if constexpr (kDiagPacked) {
    // off-diagonal blocks on threads [0, NOFF * TPB), the diagonal warp(s)
    // from DW: block NOFF + d on threads DW + d * TPB ...
    constexpr int NOFF = Thomas<CB>::NOFF, DW = Thomas<CB>::DW;
    const bool diag = tid >= DW;
    m.active = diag ? tid < Thomas<CB>::MV : tid < NOFF * kMvTpb;
    m.blk = !m.active ? (diag ? NOFF : 0) : diag ? NOFF + (tid - DW) / kMvTpb : tid / kMvTpb;
  } else {
    m.active = tid < Thomas<CB>::MV;
    m.blk = m.active ? tid / kMvTpb : 0;
  }
  m.r = tid % kMvTpb;  // index inside the block: rows R m.r .. R m.r + R - 1
  block_of<CB>(m.blk, m.I, m.J);
  return m;
}

// Reduce-scatter over the TPB = 8/R lanes of a block (aligned lane group):
// lane `sub` returns, for its R columns c = sub R + i, the sum over the
// group's lanes of b[c]. Fixed exchange order (deterministic sums).
template <int TPB>
__device__ __forceinline__ void reduce_scatter(double (&b)[8], int sub, double (&out)[8 / TPB]) {
  if constexpr (TPB == 8) {
    const bool h4 = sub & 4, h2 = sub & 2, h1 = sub & 1;
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
    out[0] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
  } else if constexpr (TPB == 4) {
    const bool h2 = sub & 2, h1 = sub & 1;
    double c4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double send = h2 ? b[k] : b[k + 4];
      const double keep = h2 ? b[k + 4] : b[k];
      c4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double send = h1 ? c4[k] : c4[k + 2];
      const double keep = h1 ? c4[k + 2] : c4[k];
      out[k] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
  } else {
    const bool h1 = sub & 1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double send = h1 ? b[k] : b[k + 4];
      const double keep = h1 ? b[k + 4] : b[k];
      out[k] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
  }
}

// R consecutive doubles to / from shared memory (16-byte accesses for R >= 2;
// every address used below is a multiple of R doubles from a 16-byte base).
template <int R>
__device__ __forceinline__ void st_run(double* p, const double (&v)[R]) {
  if constexpr (R == 1) p[0] = v[0];
  else
#pragma unroll
    for (int i = 0; i < R; i += 2) *reinterpret_cast<double2*>(p + i) = make_double2(v[i], v[i + 1]);
}
template <int R>
__device__ __forceinline__ void ld_run(const double* p, double (&v)[R]) {
  if constexpr (R == 1) v[0] = p[0];
  else
#pragma unroll
    for (int i = 0; i < R; i += 2) {
      const double2 t = *reinterpret_cast<const double2*>(p + i);
      v[i] = t.x;
      v[i + 1] = t.y;
    }
}

// Packed diagonal block (I, I) of a plane mat-vec step (two rows per thread,
// the diagonal warp): the stored lower triangle gives the row products over
// columns <= row and, transposed, the column products of the strictly lower
// part; both land on the thread's own rows 8 I + 2 sub, + 1 after the
// reduce-scatter, so the block contributes one partial per row (part[I][]).
template <int CB>
__device__ __forceinline__ void mv_partials_diag(ThomasSmem<CB>& sm, const double* Gp, const double* w,
                                                 const MvRole<CB>& m) {
  const int sub = m.r, d = m.blk - Thomas<CB>::NOFF;
  const uint32_t reg = smem_u32(Gp + Thomas<CB>::NOFF * 64 + d * kDiagBlock + diag_region(sub));
  double gv[2][8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // chunk q (columns 2q, 2q + 1) of both rows, stored for q <= sub
    double2 v0 = make_double2(0.0, 0.0), v1 = make_double2(0.0, 0.0);
    if (q <= sub) {
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v0.x), "=d"(v0.y) : "r"(reg + 16u * q));
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                   : "=d"(v1.x), "=d"(v1.y)
                   : "r"(reg + 16u * (sub + 1 + q)));
    }
    gv[0][2 * q] = v0.x;
    gv[0][2 * q + 1] = v0.y;
    gv[1][2 * q] = v1.x;
    gv[1][2 * q + 1] = v1.y;
  }
  double ro[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int c = 0; c < 8; c += 2) {
      const double2 wv = *reinterpret_cast<const double2*>(w + 8 * m.I + c);  // broadcast
      a0 = fma(gv[i][c], wv.x, a0);
      a1 = fma(gv[i][c + 1], wv.y, a1);
    }
    ro[i] = a0 + a1;
  }
  double wr[2];
  ld_run<2>(w + 8 * m.I + 2 * sub, wr);
  if (!m.active) wr[0] = wr[1] = 0.0;
  double b[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {  // strictly lower entries only: the diagonal belongs to the row products
    b[c] = (c == 2 * sub ? 0.0 : gv[0][c]) * wr[0];
    b[c] = fma(c == 2 * sub + 1 ? 0.0 : gv[1][c], wr[1], b[c]);
  }
  double cs[2];
  reduce_scatter<4>(b, sub, cs);
  ro[0] += cs[0];
  ro[1] += cs[1];
  if (m.active) st_run<2>(&sm.part[m.I][8 * m.I + 2 * sub], ro);
}

// One plane mat-vec step: partial products into part[][].
template <int CB>
__device__ __forceinline__ void mv_partials(ThomasSmem<CB>& sm, const double* Gp, const double* w,
                                            const MvRole<CB>& m) {
  constexpr int R = kMvRows, TPB = kMvTpb;
  // whole warps take part (the shuffles below need every lane)
  if ((int)(threadIdx.x >> 5) >= (Thomas<CB>::MV + 31) / 32) return;
  if constexpr (kDiagPacked) {
    if ((int)threadIdx.x >= Thomas<CB>::DW) return mv_partials_diag<CB>(sm, Gp, w, m);
  }
  const bool off_diag = m.active && m.J < m.I;
  double gv[R][8];
  const uint32_t reg = smem_u32(Gp + m.blk * 64 + m.r * 8 * R);  // the thread's R rows
#pragma unroll
  for (int k = 0; k < 4 * R; ++k) {
    double2 v;  // explicit ld.shared: the slot pointer is opaque to the compiler
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "r"(reg + (uint32_t)(16 * mv_chunk_pos(k, m.r, (int)threadIdx.x))));
    gv[k / 4][2 * (k % 4)] = v.x;
    gv[k / 4][2 * (k % 4) + 1] = v.y;
  }
  double ro[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    double a0 = 0.0, a1 = 0.0;  // two chains halve the dependent-FMA latency
#pragma unroll
    for (int c = 0; c < 8; c += 2) {
      const double2 wv = *reinterpret_cast<const double2*>(w + 8 * m.J + c);  // broadcast
      a0 = fma(gv[i][c], wv.x, a0);
      a1 = fma(gv[i][c + 1], wv.y, a1);
    }
    ro[i] = a0 + a1;
  }
  if (m.active) st_run<R>(&sm.part[m.J][8 * m.I + R * m.r], ro);
  // transposed block; diagonal blocks (and idle lanes) contribute zeros
  double wr[R];
  ld_run<R>(w + 8 * m.I + R * m.r, wr);
  double b[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    b[c] = gv[0][c] * (off_diag ? wr[0] : 0.0);
#pragma unroll
    for (int i = 1; i < R; ++i) b[c] = fma(gv[i][c], off_diag ? wr[i] : 0.0, b[c]);
  }
  double cs[R];
  reduce_scatter<TPB>(b, m.r, cs);
  if (off_diag) st_run<R>(&sm.part[m.I][8 * m.J + R * m.r], cs);
}

template <int CB>
__device__ __forceinline__ void thomas_init(ThomasSmem<CB>& sm) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < kSlots; ++s) mbar_init(&sm.bars[s], 1);
    fence_barrier_init();
  }
}

// Issue the first kSlots plane loads of a solve (thread 0). Call after
// thomas_init + __syncthreads, as early as possible in the kernel.
template <int CB>
__device__ __forceinline__ void thomas_prefetch(ThomasSmem<CB>& sm, const double* __restrict__ G,
                                                uint32_t m0 = 0) {
  if (!G) return;  // uniform brick: no factor planes (brick_inverse)
  // resident mode (kSlots >= CB): all CB planes stay in shared memory and the
  // backward sweep reuses them; otherwise a ring refilled kSlots steps ahead.
  constexpr int NPRE = kSlots >= CB ? CB : kSlots;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int n = 0; n < NPRE && n < Thomas<CB>::NL; ++n) {
      const int sl = kSlots >= CB ? n : (int)((m0 + n) % kSlots);
      mbar_arrive_expect_tx(&sm.bars[sl], Thomas<CB>::PLANE * sizeof(double));
      plane_load(sm.slots[sl], G + (size_t)Thomas<CB>::plane_of(n) * Thomas<CB>::PLANE,
                 Thomas<CB>::PLANE * sizeof(double), &sm.bars[sl], n, CB);
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
// Persistent callers (one CTA, a sequence of bricks): m0 = plane loads this CTA
// has issued before this brick's (the ring's slot and mbarrier phase continue
// across bricks; NL loads per factored brick), Gnext = the factor of the CTA's
// next brick when that brick follows immediately (its first kSlots planes are
// requested as this brick's last planes are consumed, so the ring never
// drains between bricks), else nullptr.
template <int CB>
__device__ __forceinline__ void thomas_solve(ThomasSmem<CB>& sm, const double* __restrict__ G,
                                             const double* t, const double* tz, double* x,
                                             double scale = 1.0, uint32_t m0 = 0,
                                             const double* __restrict__ Gnext = nullptr) {
  constexpr int P = Thomas<CB>::P, NL = Thomas<CB>::NL, NBK = Thomas<CB>::NBK;
  const int tid = threadIdx.x;
  const MvRole<CB> m = mv_role<CB>();
  constexpr bool resident = kSlots >= CB;
  auto slot_of = [m0](int n) { return resident ? Thomas<CB>::plane_of(n) : (int)((m0 + n) % kSlots); };
  auto parity_of = [m0](int n) { return resident ? 0u : (uint32_t)(((m0 + n) / kSlots) & 1); };
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
    if (!resident && issuer && (n + kSlots < NL || Gnext)) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&sm.bars[slot], Thomas<CB>::PLANE * sizeof(double));
      const bool own = n + kSlots < NL;
      const int nn = own ? n + kSlots : n + kSlots - NL;  // load index in its brick
      plane_load(sm.slots[slot], (own ? G : Gnext) + (size_t)Thomas<CB>::plane_of(nn) * Thomas<CB>::PLANE,
                 Thomas<CB>::PLANE * sizeof(double), &sm.bars[slot], nn, CB);
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

// Orthonormal DST-I matrices Q[a][b] = sqrt(2/(CB+1)) sin(pi (a+1)(b+1)/(CB+1))
// (symmetric; row a is even about the midpoint for even a, odd for odd a)
// and the eigenvalues 2 - 2 cos(pi (j+1)/(CB+1)) of the 1-D Dirichlet
// Laplacian tridiag(-1, 2, -1), CB = 8 and 4.
static __constant__ double kDstQ8[64] = {
    0.16122984176531682, 0.30301298511469577, 0.40824829046386296, 0.46424282688001262, 0.46424282688001262, 0.40824829046386296, 0.30301298511469577, 0.16122984176531682,
    0.30301298511469577, 0.46424282688001262, 0.40824829046386296, 0.16122984176531682, -0.16122984176531682, -0.40824829046386296, -0.46424282688001262, -0.30301298511469577,
    0.40824829046386296, 0.40824829046386296, 0, -0.40824829046386296, -0.40824829046386296, 0, 0.40824829046386296, 0.40824829046386296,
    0.46424282688001262, 0.16122984176531682, -0.40824829046386296, -0.30301298511469577, 0.30301298511469577, 0.40824829046386296, -0.16122984176531682, -0.46424282688001262,
    0.46424282688001262, -0.16122984176531682, -0.40824829046386296, 0.30301298511469577, 0.30301298511469577, -0.40824829046386296, -0.16122984176531682, 0.46424282688001262,
    0.40824829046386296, -0.40824829046386296, 0, 0.40824829046386296, -0.40824829046386296, 0, 0.40824829046386296, -0.40824829046386296,
    0.30301298511469577, -0.46424282688001262, 0.40824829046386296, -0.16122984176531682, -0.16122984176531682, 0.40824829046386296, -0.46424282688001262, 0.30301298511469577,
    0.16122984176531682, -0.30301298511469577, 0.40824829046386296, -0.46424282688001262, 0.46424282688001262, -0.40824829046386296, 0.30301298511469577, -0.16122984176531682,
};
static __constant__ double kDstL8[8] = {0.12061475842818314, 0.46791111376204397, 0.99999999999999978, 1.6527036446661392, 2.3472963553338606, 2.9999999999999996, 3.5320888862379558, 3.8793852415718169};
static __constant__ double kDstQ4[16] = {
    0.37174803446018451, 0.60150095500754563, 0.60150095500754563, 0.37174803446018451,
    0.60150095500754563, 0.37174803446018451, -0.37174803446018451, -0.60150095500754563,
    0.60150095500754563, -0.37174803446018451, -0.37174803446018451, 0.60150095500754563,
    0.37174803446018451, -0.60150095500754563, 0.60150095500754563, -0.37174803446018451,
};
static __constant__ double kDstL4[4] = {0.3819660112501051, 1.3819660112501051, 2.6180339887498949, 3.6180339887498949};

template <int CB>
__device__ __forceinline__ double dst_q(int a, int b) {
  if constexpr (CB == 8) return kDstQ8[a * 8 + b];
  else return kDstQ4[a * 4 + b];
}
template <int CB>
__device__ __forceinline__ double dst_l(int j) {
  if constexpr (CB == 8) return kDstL8[j];
  else return kDstL4[j];
}

// o = Q v for one line of CB points in registers: the even / odd halves of v
// about the midpoint feed the even / odd rows (CB^2/2 FMAs; Q comes from the
// constant bank with compile-time indices, no shared-memory traffic).
template <int CB>
__device__ __forceinline__ void dst_line(const double (&v)[CB], double (&o)[CB]) {
  double e[CB / 2], d[CB / 2];
#pragma unroll
  for (int n = 0; n < CB / 2; ++n) {
    e[n] = v[n] + v[CB - 1 - n];
    d[n] = v[n] - v[CB - 1 - n];
  }
#pragma unroll
  for (int m = 0; m < CB; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int n = 0; n < CB / 2; ++n) acc = fma(dst_q<CB>(m, n), (m & 1) ? d[n] : e[n], acc);
    o[m] = acc;
  }
}

// x = A_II^-1 t of an interior brick of one conductivity k (cells and face
// halo): A_II = face_t(k, k) sum_ax (area/h)_ax K_ax with K the 1-D Dirichlet
// Laplacian tridiag(-1, 2, -1) along each axis (every face of every cell,
// inside and to the neighbours, carries face_t(k, k) area/h), so
//   A_II^-1 = scale (Q x Q x Q) diag(1 / sum_ax (area/h)_ax lambda_ax) (Q x Q x Q),
// scale = 1 / face_t(k, k), Q the symmetric orthonormal DST-I: six CB-point
// transforms and a division instead of the 15 dependent plane mat-vecs.
// One thread per line of CB points (CB^2 threads; the line lives in
// registers), five shared-memory passes: z, y, then x + division + x on the
// thread's own line, y, z. The intermediate arrays sit in the two (unused)
// plane slots, padded so that every pass reads and writes without bank
// conflicts: A[i + CB j + (CB^2 + 8) k] between the z and y passes,
// B[i + (CB + 1) j + CB (CB + 1) k] around the x pass (x lines at an odd
// stride). Starts and ends with a __syncthreads; the result overwrites t.
template <int CB>
__device__ __forceinline__ void fastdiag_solve(const ThomasSmem<CB>& sm, double* t, double scale,
                                               const double* cpl) {
  static_assert(kSlots >= 2, "fastdiag_solve keeps its two scratch arrays in the plane slots");
  constexpr int P = CB * CB, SA = P + 8, LX = CB + 1, SB = CB * LX;
  static_assert(CB * SA <= Thomas<CB>::PLANE && CB * SB <= Thomas<CB>::PLANE, "scratch fits a slot");
  double* A = &sm.slots[0][0];
  double* B = &sm.slots[1][0];
  const int tid = threadIdx.x, a = tid % CB, b = tid / CB;
  const bool on = tid < P;
  double v[CB], o[CB];
  __syncthreads();  // t complete
  if (on) {  // z pass, thread (i, j) = (a, b): t -> A
#pragma unroll
    for (int k = 0; k < CB; ++k) v[k] = t[a + CB * b + P * k];
    dst_line<CB>(v, o);
#pragma unroll
    for (int k = 0; k < CB; ++k) A[a + CB * b + SA * k] = o[k];
  }
  __syncthreads();
  if (on) {  // y pass, thread (i, k) = (a, b): A -> B
#pragma unroll
    for (int j = 0; j < CB; ++j) v[j] = A[a + CB * j + SA * b];
    dst_line<CB>(v, o);
#pragma unroll
    for (int j = 0; j < CB; ++j) B[a + LX * j + SB * b] = o[j];
  }
  __syncthreads();
  if (on) {  // x pass, division, x pass on the thread's own line (j, k) = (a, b)
    double* line = B + LX * a + SB * b;
#pragma unroll
    for (int i = 0; i < CB; ++i) v[i] = line[i];
    dst_line<CB>(v, o);
    const double cjk = cpl[1] * dst_l<CB>(a) + cpl[2] * dst_l<CB>(b);
#pragma unroll
    for (int i = 0; i < CB; ++i) o[i] *= scale / (cpl[0] * dst_l<CB>(i) + cjk);
    dst_line<CB>(o, v);
#pragma unroll
    for (int i = 0; i < CB; ++i) line[i] = v[i];
  }
  __syncthreads();
  if (on) {  // y pass back, thread (i, k): B -> A
#pragma unroll
    for (int j = 0; j < CB; ++j) v[j] = B[a + LX * j + SB * b];
    dst_line<CB>(v, o);
#pragma unroll
    for (int j = 0; j < CB; ++j) A[a + CB * j + SA * b] = o[j];
  }
  __syncthreads();
  if (on) {  // z pass back, thread (i, j): A -> t
#pragma unroll
    for (int k = 0; k < CB; ++k) v[k] = A[a + CB * b + SA * k];
    dst_line<CB>(v, o);
#pragma unroll
    for (int k = 0; k < CB; ++k) t[a + CB * b + P * k] = o[k];
  }
  __syncthreads();
}

// The exact block solve of one brick: the plane-factor block Thomas (G), or
// the fast diagonalisation of a uniform interior brick (G == nullptr, tz
// used as scratch).
template <int CB>
__device__ __forceinline__ void brick_inverse(ThomasSmem<CB>& sm, const double* G, double* t,
                                              double* tz, double scale, const GridParams& g) {
  if (G) thomas_solve<CB>(sm, G, t, tz, t, scale);
  else fastdiag_solve<CB>(sm, t, scale, g.cpl);
}

}  // namespace tmg
