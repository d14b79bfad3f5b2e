/*
 * ORACLE — test infrastructure only. Dense linear algebra used by the CPU
 * restatement (oracle/topmg_oracle.c) and by the Eigen-subset shim that lets
 * the reference's own solver.cpp / coarse_space.cpp compile (oracle/eigen_shim).
 * Nothing in the product path links this file.
 *
 * What it stands in for (third-party boundary):
 *   Eigen::SelfAdjointEigenSolver<MatrixXd>  (ascending eigenvalues, orthonormal
 *     eigenvector columns)  — called at proj/core/src/coarse_space.cpp:46,140,395
 *   Eigen::LDLT<MatrixXd> / SimplicialLDLT   — proj/core/src/solver.cpp:63-64,81,94
 * Eigen itself (>=3.3, unpinned, not vendored under /root/reference) is absent,
 * so these are textbook restatements of the published algorithms:
 *   - Householder reduction to tridiagonal form + implicit-shift QL
 *     (the classical EISPACK tred2/tql2 pair), all eigenpairs;
 *   - for "k smallest of n": Householder reduction, Sturm-sequence bisection
 *     for the k smallest eigenvalues, inverse iteration on the tridiagonal with
 *     cluster re-orthogonalisation (the LAPACK dstebz/dstein strategy) and
 *     back-transformation by the stored reflectors;
 *   - envelope (profile) LDL^T without pivoting for SPD matrices.
 * Eigenvector signs / rotations inside degenerate clusters differ from Eigen's;
 * every consumer on the path depends only on the spanned subspaces
 * (SURVEY.md §8(c) "Known deviation").
 */
#include "dense_la.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- tridiag */

/* Householder reduction of the symmetric n x n row-major matrix `a` to
 * tridiagonal form T = Q^T A Q. On return d[0..n) is diag(T), e[1..n) the
 * sub-diagonal (e[0] = 0). If `accumulate` is nonzero, `a` is overwritten with
 * Q (row-major, columns are the basis); otherwise `a` keeps the reflectors
 * (row i, columns [0, i) hold u_i scaled, and hh[i] = h_i) for
 * dla_tridiag_backtransform. */
static void tridiagonalize(int n, double* a, double* d, double* e, double* hh,
                           int accumulate) {
#define A(i, j) a[(size_t)(i) * (size_t)n + (size_t)(j)]
  for (int i = n - 1; i > 0; --i) {
    const int l = i - 1;
    double h = 0.0;
    if (l > 0) {
      double scale = 0.0;
      for (int k = 0; k <= l; ++k) scale += fabs(A(i, k));
      if (scale == 0.0) {
        e[i] = A(i, l);
      } else {
        for (int k = 0; k <= l; ++k) {
          A(i, k) /= scale;
          h += A(i, k) * A(i, k);
        }
        double f = A(i, l);
        const double g = f >= 0.0 ? -sqrt(h) : sqrt(h);
        e[i] = scale * g;
        h -= f * g;
        A(i, l) = f - g;
        f = 0.0;
        for (int j = 0; j <= l; ++j) {
          if (accumulate) A(j, i) = A(i, j) / h;
          double gg = 0.0;
          for (int k = 0; k <= j; ++k) gg += A(j, k) * A(i, k);
          for (int k = j + 1; k <= l; ++k) gg += A(k, j) * A(i, k);
          e[j] = gg / h;
          f += e[j] * A(i, j);
        }
        const double hh2 = f / (h + h);
        for (int j = 0; j <= l; ++j) {
          const double ff = A(i, j);
          const double gg = e[j] - hh2 * ff;
          e[j] = gg;
          for (int k = 0; k <= j; ++k) A(j, k) -= (ff * e[k] + gg * A(i, k));
        }
        /* A(i, 0..l) now holds u (unscaled by `scale`, which cancels in the
         * reflector u u^T / h because both u and h carry scale^2 ... ) */
      }
    } else {
      e[i] = A(i, l);
    }
    d[i] = h;
    if (hh) hh[i] = h;
  }
  d[0] = 0.0;
  e[0] = 0.0;
  if (hh) hh[0] = 0.0;
  if (accumulate) {
    for (int i = 0; i < n; ++i) {
      const int l = i - 1;
      if (d[i] != 0.0) {
        for (int j = 0; j <= l; ++j) {
          double g = 0.0;
          for (int k = 0; k <= l; ++k) g += A(i, k) * A(k, j);
          for (int k = 0; k <= l; ++k) A(k, j) -= g * A(k, i);
        }
      }
      d[i] = A(i, i);
      A(i, i) = 1.0;
      for (int j = 0; j <= l; ++j) A(j, i) = A(i, j) = 0.0;
    }
  } else {
    for (int i = 0; i < n; ++i) d[i] = A(i, i);
  }
#undef A
}

/* Implicit-shift QL on the tridiagonal (d, e with e[1..n) sub-diagonal).
 * zt is n x n row-major holding Q^T (row r = basis vector r); rotations act on
 * pairs of rows so the inner loop is contiguous. Returns 0 or -1 on failure. */
static int tql_rows(int n, double* d, double* e, double* zt) {
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  if (n > 0) e[n - 1] = 0.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = fabs(d[m]) + fabs(d[m + 1]);
        if (fabs(e[m]) <= 2.220446049250313e-16 * dd) break;
      }
      if (m != l) {
        if (iter++ == 200) return -1;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? fabs(r) : -fabs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          if (zt) {
            double* zi = zt + (size_t)i * (size_t)n;
            double* zi1 = zt + (size_t)(i + 1) * (size_t)n;
            for (int k = 0; k < n; ++k) {
              f = zi1[k];
              zi1[k] = s * zi[k] + c * f;
              zi[k] = c * zi[k] - s * f;
            }
          }
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  return 0;
}

int dla_syev_all(int n, double* a, double* w, double* v) {
  if (n <= 0) return 0;
  double* e = (double*)malloc(sizeof(double) * (size_t)n);
  double* zt = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  if (!e || !zt) {
    free(e);
    free(zt);
    return -2;
  }
  tridiagonalize(n, a, w, e, NULL, 1);
  /* zt = Q^T */
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      zt[(size_t)j * n + i] = a[(size_t)i * n + j];
  int rc = tql_rows(n, w, e, zt);
  if (rc == 0) {
    /* selection sort ascending (stable for equal keys by index) */
    int* order = (int*)malloc(sizeof(int) * (size_t)n);
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int i = 0; i < n; ++i) {
      int best = i;
      for (int j = i + 1; j < n; ++j)
        if (w[order[j]] < w[order[best]]) best = j;
      const int t = order[i];
      order[i] = order[best];
      order[best] = t;
    }
    double* ws = (double*)malloc(sizeof(double) * (size_t)n);
    for (int c = 0; c < n; ++c) {
      ws[c] = w[order[c]];
      const double* row = zt + (size_t)order[c] * n;
      for (int i = 0; i < n; ++i) v[(size_t)i * n + c] = row[i];
    }
    memcpy(w, ws, sizeof(double) * (size_t)n);
    free(ws);
    free(order);
  }
  free(e);
  free(zt);
  return rc;
}

/* Number of eigenvalues of the tridiagonal (d, e[1..n)) strictly below x. */
static int sturm_count(int n, const double* d, const double* e2, double x,
                       double pivmin) {
  int count = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0.0) ++count;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e2[i] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0.0) ++count;
  }
  return count;
}

/* Solve (T - lambda I) y = b for tridiagonal T by Gaussian elimination with
 * partial pivoting (LAPACK dlagtf/dlagts style, restated). b overwritten. */
static void tri_shift_solve(int n, const double* d, const double* e,
                            double lambda, double tiny, double* b, double* w1,
                            double* w2, double* w3, int* piv) {
  /* rows: sub = e[i] (i>=1), diag = d[i]-lambda, sup = e[i+1] */
  double* dd = w1; /* diagonal of U */
  double* du = w2; /* first super */
  double* du2 = w3; /* second super (from pivoting) */
  /* l multipliers stored in piv-independent array: reuse b? keep separate */
  double* lm = (double*)malloc(sizeof(double) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    dd[i] = d[i] - lambda;
    du[i] = (i + 1 < n) ? e[i + 1] : 0.0;
    du2[i] = 0.0;
    piv[i] = 0;
    lm[i] = 0.0;
  }
  for (int i = 0; i + 1 < n; ++i) {
    const double sub = e[i + 1];
    if (fabs(dd[i]) >= fabs(sub)) {
      if (dd[i] == 0.0) dd[i] = tiny;
      const double m = sub / dd[i];
      lm[i] = m;
      dd[i + 1] -= m * du[i];
      piv[i] = 0;
    } else {
      /* swap rows i and i+1 */
      const double m = dd[i] / sub;
      lm[i] = m;
      dd[i] = sub;
      const double t = du[i];
      du[i] = dd[i + 1];
      dd[i + 1] = t - m * du[i];
      du2[i] = (i + 2 < n) ? du[i + 1] : 0.0;
      if (i + 2 < n) du[i + 1] = -m * du2[i];
      piv[i] = 1;
    }
  }
  if (dd[n - 1] == 0.0) dd[n - 1] = tiny;
  /* forward: apply L^-1 P */
  for (int i = 0; i + 1 < n; ++i) {
    if (piv[i]) {
      const double t = b[i];
      b[i] = b[i + 1];
      b[i + 1] = t - lm[i] * b[i];
    } else {
      b[i + 1] -= lm[i] * b[i];
    }
  }
  /* back substitution with U (dd, du, du2) */
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    if (i + 1 < n) s -= du[i] * b[i + 1];
    if (i + 2 < n) s -= du2[i] * b[i + 2];
    double piv_v = dd[i];
    if (fabs(piv_v) < tiny) piv_v = piv_v < 0 ? -tiny : tiny;
    b[i] = s / piv_v;
  }
  free(lm);
}

/* Deterministic pseudo-random start vectors (splitmix64). */
static double det_uniform(unsigned long long* s) {
  unsigned long long z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

int dla_syev_smallest(int n, int k, double* a, double* w, double* v) {
  if (k <= 0 || n <= 0) return 0;
  if (k > n) return -3;
  if (n <= 64 || 4 * k >= n) {
    /* small problems: full solver, keep the first k */
    double* wall = (double*)malloc(sizeof(double) * (size_t)n);
    double* vall = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
    const int rc = dla_syev_all(n, a, wall, vall);
    if (rc == 0) {
      for (int c = 0; c < k; ++c) {
        w[c] = wall[c];
        for (int i = 0; i < n; ++i) v[(size_t)i * k + c] = vall[(size_t)i * n + c];
      }
    }
    free(wall);
    free(vall);
    return rc;
  }
  double* d = (double*)malloc(sizeof(double) * (size_t)n);
  double* e = (double*)malloc(sizeof(double) * (size_t)n);
  double* e2 = (double*)malloc(sizeof(double) * (size_t)n);
  double* hh = (double*)malloc(sizeof(double) * (size_t)n);
  double* y = (double*)malloc(sizeof(double) * (size_t)n * (size_t)k);
  double* w1 = (double*)malloc(sizeof(double) * (size_t)n);
  double* w2 = (double*)malloc(sizeof(double) * (size_t)n);
  double* w3 = (double*)malloc(sizeof(double) * (size_t)n);
  int* piv = (int*)malloc(sizeof(int) * (size_t)n);
  tridiagonalize(n, a, d, e, hh, 0);
  double tnorm = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = fabs(d[i]) + (i > 0 ? fabs(e[i]) : 0.0) +
                     (i + 1 < n ? fabs(e[i + 1]) : 0.0);
    if (r > tnorm) tnorm = r;
    e2[i] = e[i] * e[i];
  }
  if (tnorm == 0.0) tnorm = 1.0;
  const double eps = 2.220446049250313e-16;
  double maxe2 = 1.0;
  for (int i = 0; i < n; ++i)
    if (e2[i] > maxe2) maxe2 = e2[i];
  const double pivmin = 2.2250738585072014e-308 * maxe2;
  /* bisection for eigenvalues 0..k-1 */
  for (int j = 0; j < k; ++j) {
    double lo = -tnorm * 1.0000001 - 1e-300, hi = tnorm * 1.0000001 + 1e-300;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (mid == lo || mid == hi) break;
      if (sturm_count(n, d, e2, mid, pivmin) > j)
        hi = mid;
      else
        lo = mid;
      if (hi - lo <= 2.0 * eps * (fabs(lo) + fabs(hi)) + 1e-3 * pivmin) break;
    }
    w[j] = 0.5 * (lo + hi);
  }
  /* inverse iteration with reorthogonalisation inside clusters */
  unsigned long long seed = 0x5eedULL;
  const double cluster_tol = 1e-3 * tnorm;
  const double tiny = eps * tnorm;
  int cluster_start = 0;
  for (int j = 0; j < k; ++j) {
    if (j > 0 && fabs(w[j] - w[j - 1]) > cluster_tol) cluster_start = j;
    double* yj = y + (size_t)j * n;
    for (int i = 0; i < n; ++i) yj[i] = det_uniform(&seed) - 0.5;
    /* perturb the shift slightly away from exact to avoid a zero pivot */
    double shift = w[j];
    for (int it = 0; it < 5; ++it) {
      tri_shift_solve(n, d, e, shift, tiny, yj, w1, w2, w3, piv);
      for (int pass = 0; pass < 2; ++pass)
        for (int c = cluster_start; c < j; ++c) {
          const double* yc = y + (size_t)c * n;
          double dot = 0.0;
          for (int i = 0; i < n; ++i) dot += yc[i] * yj[i];
          for (int i = 0; i < n; ++i) yj[i] -= dot * yc[i];
        }
      double nrm = 0.0;
      for (int i = 0; i < n; ++i) nrm += yj[i] * yj[i];
      nrm = sqrt(nrm);
      if (!(nrm > 0.0)) {
        for (int i = 0; i < n; ++i) yj[i] = det_uniform(&seed) - 0.5;
        continue;
      }
      for (int i = 0; i < n; ++i) yj[i] /= nrm;
    }
  }
  /* back-transform: x = Q y, Q = H_{n-1}...H_1 applied as H_1 ... ;
   * reflector i (i = 1..n-1, when hh[i] != 0) acts on coordinates [0, i)
   * with vector u = a[i][0..i), scale h: H = I - u u^T / h. Q = H_{n-1} H_{n-2} ... H_1
   * in the order the reduction applied them; x = Q y means apply H_1 first? The
   * reduction computes T = H_1 ... H_{n-1} A H_{n-1} ... H_1, so
   * A = Q T Q^T with Q = H_{n-1} ... H_1, and x = Q y applies H_1 first. */
#define A(i, j) a[(size_t)(i) * (size_t)n + (size_t)(j)]
  for (int j = 0; j < k; ++j) {
    double* yj = y + (size_t)j * n;
    for (int i = 1; i < n; ++i) {
      if (hh[i] == 0.0 || i - 1 == 0) continue; /* l = 0 -> no reflector */
      const int l = i - 1;
      double dot = 0.0;
      for (int c = 0; c <= l; ++c) dot += A(i, c) * yj[c];
      const double f = dot / hh[i];
      for (int c = 0; c <= l; ++c) yj[c] -= f * A(i, c);
    }
    /* final normalisation */
    double nrm = 0.0;
    for (int i = 0; i < n; ++i) nrm += yj[i] * yj[i];
    nrm = sqrt(nrm);
    for (int i = 0; i < n; ++i) v[(size_t)i * k + j] = yj[i] / nrm;
  }
#undef A
  free(d);
  free(e);
  free(e2);
  free(hh);
  free(y);
  free(w1);
  free(w2);
  free(w3);
  free(piv);
  return 0;
}

/* ---------------------------------------------------------------- LDL^T */

int dla_env_ldlt_factor(int64_t n, const int64_t* first, const int64_t* rowptr,
                        double* vals, double* dout, double* max_pivot_out,
                        int64_t* bad_index_out) {
  /* Row i stores columns [first[i], i] at vals[rowptr[i] .. rowptr[i+1]).
   * On exit, vals holds L (unit lower, diagonal slot holds D). */
  double maxp = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double* ri = vals + rowptr[i];
    const int64_t fi = first[i];
    for (int64_t j = fi; j < i; ++j) {
      const double* rj = vals + rowptr[j];
      const int64_t fj = first[j];
      const int64_t k0 = fi > fj ? fi : fj;
      double s = ri[j - fi];
      for (int64_t kk = k0; kk < j; ++kk)
        s -= ri[kk - fi] * dout[kk] * rj[kk - fj];
      ri[j - fi] = s / dout[j];
    }
    double di = ri[i - fi];
    for (int64_t kk = fi; kk < i; ++kk) di -= ri[kk - fi] * ri[kk - fi] * dout[kk];
    dout[i] = di;
    ri[i - fi] = di;
    if (fabs(di) > maxp) maxp = fabs(di);
    if (!(di > 0.0) && !(di < 0.0)) {
      /* exact zero / NaN pivot: stop, caller reports */
      if (bad_index_out) *bad_index_out = i;
      if (max_pivot_out) *max_pivot_out = maxp;
      return -1;
    }
  }
  if (max_pivot_out) *max_pivot_out = maxp;
  if (bad_index_out) *bad_index_out = -1;
  for (int64_t i = 0; i < n; ++i)
    if (!(dout[i] > 1e-14 * maxp)) {
      if (bad_index_out) *bad_index_out = i;
      return -1;
    }
  return 0;
}

void dla_env_ldlt_solve(int64_t n, const int64_t* first, const int64_t* rowptr,
                        const double* vals, const double* d, double* x) {
  for (int64_t i = 0; i < n; ++i) {
    const double* ri = vals + rowptr[i];
    double s = x[i];
    for (int64_t kk = first[i]; kk < i; ++kk) s -= ri[kk - first[i]] * x[kk];
    x[i] = s;
  }
  for (int64_t i = 0; i < n; ++i) x[i] /= d[i];
  for (int64_t i = n - 1; i >= 0; --i) {
    const double* ri = vals + rowptr[i];
    const double xi = x[i];
    for (int64_t kk = first[i]; kk < i; ++kk) x[kk] -= ri[kk - first[i]] * xi;
  }
}

/* All eigenvalues (ascending) of the symmetric n x n row-major `a` (destroyed)
 * plus eigenvectors for the k smallest (v: n x k row-major). Used by the
 * Eigen shim: the reference reads only leading eigenvector columns. */
int dla_syev_partial(int n, int k, double* a, double* w_all, double* v) {
  if (n <= 0) return 0;
  if (k > n) k = n;
  double* acopy = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  memcpy(acopy, a, sizeof(double) * (size_t)n * (size_t)n);
  double* d = (double*)malloc(sizeof(double) * (size_t)n);
  double* e = (double*)malloc(sizeof(double) * (size_t)n);
  tridiagonalize(n, acopy, d, e, NULL, 0);
  int rc = tql_rows(n, d, e, NULL);
  if (rc == 0) {
    /* ascending insertion sort of the eigenvalues */
    for (int i = 1; i < n; ++i) {
      const double x = d[i];
      int j = i - 1;
      while (j >= 0 && d[j] > x) {
        d[j + 1] = d[j];
        --j;
      }
      d[j + 1] = x;
    }
    memcpy(w_all, d, sizeof(double) * (size_t)n);
    if (k > 0) {
      double* wk = (double*)malloc(sizeof(double) * (size_t)k);
      rc = dla_syev_smallest(n, k, a, wk, v);
      free(wk);
    }
  }
  free(acopy);
  free(d);
  free(e);
  return rc;
}
