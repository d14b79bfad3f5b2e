// Host-side check of the fine factor plane layout (smoother.cuh): for the
// TMG_MV_ROWS / TMG_DIAG_PACK the file is compiled with, every stored slot of
// a plane is written exactly once (plane_off / diag_slot are a bijection onto
// [0, PLANE)), each 128-bit load of a quarter-warp covers eight distinct
// 16-byte bank groups, and the stored blocks are the lower block triangle.
// Built and run by tests/test_layout_cpu.py (no GPU needed).
#include <cstdio>
#include <vector>

#include "smoother.cuh"

using namespace tmg;

template <int CB>
int check() {
  using T = Thomas<CB>;
  int bad = 0;
  std::vector<int> hit(T::PLANE, 0);
  const int nwhole = kDiagPacked ? T::NOFF : T::NBLK;
  for (int blk = 0; blk < nwhole; ++blk)
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 8; ++c) {
        const int o = plane_off(blk, r, c);
        if (o < 0 || o >= nwhole * 64) { ++bad; continue; }
        ++hit[o];
      }
  if (kDiagPacked) {
    for (int d = 0; d < T::NBK; ++d) {
      int seen[8][8] = {};
      for (int s = 0; s < kDiagBlock; ++s) {
        int row = 0, col = 0;
        const bool stored = diag_slot(s, row, col);
        ++hit[nwhole * 64 + d * kDiagBlock + s];
        if (stored) {
          if (row < 0 || row > 7 || col < 0 || col > row) ++bad;
          else ++seen[row][col];
        }
      }
      for (int r = 0; r < 8; ++r)
        for (int c = 0; c <= r; ++c) bad += seen[r][c] != 1;
    }
  }
  for (int o = 0; o < T::PLANE; ++o) bad += hit[o] != 1;
  // bank groups of the whole-block loads: mat-vec thread tid = blk * TPB + sub
  const int nthr = nwhole * kMvTpb;
  for (int k = 0; k < 4 * kMvRows; ++k)
    for (int q0 = 0; q0 + 8 <= nthr; q0 += 8) {
      unsigned groups = 0;
      for (int tid = q0; tid < q0 + 8; ++tid) {
        const int blk = tid / kMvTpb, sub = tid % kMvTpb;
        const int byte = (blk * 64 + sub * 8 * kMvRows) * 8 + 16 * mv_chunk_pos(k, sub, tid);
        groups |= 1u << ((byte / 16) % 8);
      }
      bad += groups != 0xffu;
    }
  printf("CB=%d rows=%d packed=%d PLANE=%d MV=%d NT=%d bad=%d\n", CB, kMvRows, (int)kDiagPacked, T::PLANE,
         T::MV, T::NT, bad);
  return bad;
}

int main() {
  return (check<8>() + check<4>()) ? 1 : 0;
}
