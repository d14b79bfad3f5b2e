// Small dense symmetric eigensolvers and the seeded pseudo-random fill shared
// by the local spectral-basis kernels (spectral.cu: cubic bricks; generic.cu:
// any brick shape).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tmg {

__device__ __forceinline__ double hash_uniform(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t z = a * 0x9E3779B97F4A7C15ULL ^ (b + 0x632BE59BD9B4E019ULL) * 0xBF58476D1CE4E5B9ULL ^
               (c + 0x94D049BB133111EBULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return (double)(z >> 11) * 0x1.0p-53 - 0.5;
}

// Cyclic Jacobi eigen-decomposition of a K x K symmetric matrix (single thread).
// a: row-major, destroyed (diag -> eigenvalues). v: eigenvectors in columns.
template <int K>
__device__ void jacobi_eig_small(double* a, double* v) {
  for (int i = 0; i < K; ++i)
    for (int j = 0; j < K; ++j) v[i * K + j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < K; ++i)
      for (int j = 0; j < K; ++j) {
        tot += a[i * K + j] * a[i * K + j];
        if (i != j) off += a[i * K + j] * a[i * K + j];
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int p = 0; p < K - 1; ++p)
      for (int q = p + 1; q < K; ++q) {
        const double apq = a[p * K + q];
        if (apq == 0.0) continue;
        const double app = a[p * K + p], aqq = a[q * K + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < K; ++k) {
          const double akp = a[k * K + p], akq = a[k * K + q];
          a[k * K + p] = c * akp - s * akq;
          a[k * K + q] = s * akp + c * akq;
        }
        for (int k = 0; k < K; ++k) {
          const double apk = a[p * K + k], aqk = a[q * K + k];
          a[p * K + k] = c * apk - s * aqk;
          a[q * K + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < K; ++k) {
          const double vkp = v[k * K + p], vkq = v[k * K + q];
          v[k * K + p] = c * vkp - s * vkq;
          v[k * K + q] = s * vkp + c * vkq;
        }
      }
  }
}

// Warp-parallel Jacobi on a K x K symmetric matrix in shared memory (K even),
// round-robin ("tournament") ordering: a sweep is K-1 rounds of K/2 disjoint
// rotations; lane g < K/2 computes rotation g of a round, then lanes r < K
// apply all of them to row / column r. Eigenvectors accumulate in V
// (columns). Called by one full warp.
template <int K>
__device__ void warp_jacobi_small(double* a, double* v) {
  static_assert(K % 2 == 0 && K <= 32, "round-robin Jacobi");
  constexpr int NP = K / 2;
  __shared__ double rot_c[NP], rot_s[NP];
  __shared__ int rot_p[NP], rot_q[NP];
  const int lane = threadIdx.x & 31;
  if (lane < K)
    for (int c = 0; c < K; ++c) v[lane * K + c] = lane == c ? 1.0 : 0.0;
  __syncwarp();
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, tot = 0.0;
    if (lane < K)
      for (int c = 0; c < K; ++c) {
        const double x = a[lane * K + c] * a[lane * K + c];
        tot += x;
        if (c != lane) off += x;
      }
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    // off-diagonal mass below ~1e-13 of the total: the Ritz values and
    // vectors are converged far beyond what the subspace iteration needs
    if (off <= 1e-26 * tot || off == 0.0) break;
    for (int round = 0; round < K - 1; ++round) {
      if (lane < NP) {  // circle method: player K-1 fixed, the others rotate
        int p, q;
        if (lane == 0) {
          p = round;
          q = K - 1;
        } else {
          p = (round + lane) % (K - 1);
          q = (round - lane + (K - 1)) % (K - 1);
        }
        if (p > q) {
          const int tmp = p;
          p = q;
          q = tmp;
        }
        const double apq = a[p * K + q];
        const double app = a[p * K + p], aqq = a[q * K + q];
        double c = 1.0, sn = 0.0;
        if (!(fabs(apq) <= 1e-16 * sqrt(fabs(app * aqq)) || apq == 0.0)) {
          const double theta = (aqq - app) / (2.0 * apq);
          const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(tt * tt + 1.0);
          sn = tt * c;
        }
        rot_c[lane] = c;
        rot_s[lane] = sn;
        rot_p[lane] = p;
        rot_q[lane] = q;
      }
      __syncwarp();
      if (lane < K) {  // columns p, q of row `lane` (all pairs are disjoint)
#pragma unroll
        for (int g = 0; g < NP; ++g) {
          const int p = rot_p[g], q = rot_q[g];
          const double c = rot_c[g], sn = rot_s[g];
          const double akp = a[lane * K + p], akq = a[lane * K + q];
          a[lane * K + p] = c * akp - sn * akq;
          a[lane * K + q] = sn * akp + c * akq;
          const double vkp = v[lane * K + p], vkq = v[lane * K + q];
          v[lane * K + p] = c * vkp - sn * vkq;
          v[lane * K + q] = sn * vkp + c * vkq;
        }
      }
      __syncwarp();
      if (lane < K) {  // rows p, q at column `lane`
#pragma unroll
        for (int g = 0; g < NP; ++g) {
          const int p = rot_p[g], q = rot_q[g];
          const double c = rot_c[g], sn = rot_s[g];
          const double apk = a[p * K + lane], aqk = a[q * K + lane];
          a[p * K + lane] = c * apk - sn * aqk;
          a[q * K + lane] = sn * apk + c * aqk;
        }
      }
      __syncwarp();
    }
  }
}

}  // namespace tmg
