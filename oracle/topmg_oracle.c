/*
 * ORACLE — test infrastructure only. CPU restatement of the reference's
 * linear-solve hot path; see topmg_oracle.h. Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library.
 */
#include "topmg_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "dense_la.h"

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_last_error(void) { return g_err; }

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

#define XMALLOC(T, n) ((T*)malloc(sizeof(T) * (size_t)((n) > 0 ? (n) : 1)))
#define XCALLOC(T, n) ((T*)calloc((size_t)((n) > 0 ? (n) : 1), sizeof(T)))

/* ================================================================= grid */

static inline double g_hx(const orc_grid* g) { return g->lx / (double)g->nx; }
static inline double g_hy(const orc_grid* g) { return g->ly / (double)g->ny; }
static inline double g_hz(const orc_grid* g) { return g->lz / (double)g->nz; }
static inline orc_index g_cell(const orc_grid* g, orc_index i, orc_index j,
                               orc_index k) {
  return i + g->nx * (j + g->ny * k); /* grid.hpp:44-46 */
}

/* grid.cpp:196-218 */
int orc_build_hierarchy(const orc_grid* g, const orc_index ncc[3], orc_index sd,
                        orc_hgrid* h) {
  if (ncc[0] <= 0 || ncc[1] <= 0 || ncc[2] <= 0 || sd <= 0)
    return fail(ORC_ECONFIG, "build_hierarchy: ncc and sd must be positive");
  const orc_index n[3] = {g->nx, g->ny, g->nz};
  h->spec = *g;
  h->sd = sd;
  for (int a = 0; a < 3; ++a) {
    h->ncc[a] = ncc[a];
    const orc_index div = ncc[a] * sd;
    if (n[a] % div != 0)
      return fail(ORC_ECONFIG,
                  "build_hierarchy: axis %d has %lld cells, not divisible by "
                  "ncc*sd = %lld",
                  a, (long long)n[a], (long long)div);
    h->nc[a] = div;
    h->cpc[a] = n[a] / div;
  }
  return ORC_OK;
}

static inline orc_index h_num_coarse(const orc_hgrid* h) {
  return h->nc[0] * h->nc[1] * h->nc[2];
}
static inline orc_index h_num_cc(const orc_hgrid* h) {
  return h->ncc[0] * h->ncc[1] * h->ncc[2];
}
static inline orc_index h_cells_in_coarse(const orc_hgrid* h) {
  return h->cpc[0] * h->cpc[1] * h->cpc[2];
}

/* grid.cpp:135-140 */
static void h_coarse_origin(const orc_hgrid* h, orc_index id, orc_index o[3]) {
  const orc_index ci = id % h->nc[0];
  const orc_index cj = (id / h->nc[0]) % h->nc[1];
  const orc_index ck = id / (h->nc[0] * h->nc[1]);
  o[0] = ci * h->cpc[0];
  o[1] = cj * h->cpc[1];
  o[2] = ck * h->cpc[2];
}

/* grid.cpp:146-153 */
static void h_cc_origin(const orc_hgrid* h, orc_index id, orc_index o[3]) {
  const orc_index ci = id % h->ncc[0];
  const orc_index cj = (id / h->ncc[0]) % h->ncc[1];
  const orc_index ck = id / (h->ncc[0] * h->ncc[1]);
  o[0] = ci * h->cpc[0] * h->sd;
  o[1] = cj * h->cpc[1] * h->sd;
  o[2] = ck * h->cpc[2] * h->sd;
}

/* grid.cpp:157-167: box cells, x-fastest */
static void box_cells(const orc_grid* g, const orc_index o[3],
                      const orc_index n[3], orc_index* out) {
  orc_index t = 0;
  for (orc_index k = 0; k < n[2]; ++k)
    for (orc_index j = 0; j < n[1]; ++j)
      for (orc_index i = 0; i < n[0]; ++i)
        out[t++] = g_cell(g, o[0] + i, o[1] + j, o[2] + k);
}

/* grid.cpp:183-194 */
static void h_coarse_children(const orc_hgrid* h, orc_index cc,
                              orc_index* out) {
  const orc_index ci = cc % h->ncc[0];
  const orc_index cj = (cc / h->ncc[0]) % h->ncc[1];
  const orc_index ck = cc / (h->ncc[0] * h->ncc[1]);
  orc_index t = 0;
  const orc_index sd = h->sd;
  for (orc_index dk = 0; dk < sd; ++dk)
    for (orc_index dj = 0; dj < sd; ++dj)
      for (orc_index di = 0; di < sd; ++di)
        out[t++] = (ci * sd + di) +
                   h->nc[0] * ((cj * sd + dj) + h->nc[1] * (ck * sd + dk));
}

/* grid.cpp:61-75 (face_center :21-34, on_boundary :36-46) */
int orc_dirichlet_value(const orc_grid* g, const orc_patch* p, int np,
                        orc_index i, orc_index j, orc_index k, int face,
                        double* value) {
  int on = 0;
  switch (face) {
    case 0: on = i == 0; break;
    case 1: on = i == g->nx - 1; break;
    case 2: on = j == 0; break;
    case 3: on = j == g->ny - 1; break;
    case 4: on = k == 0; break;
    case 5: on = k == g->nz - 1; break;
  }
  if (!on) return 0;
  const double cx = ((double)i + 0.5) * g_hx(g);
  const double cy = ((double)j + 0.5) * g_hy(g);
  const double cz = ((double)k + 0.5) * g_hz(g);
  double u, v;
  if (face <= 1) {
    u = cy;
    v = cz;
  } else if (face <= 3) {
    u = cx;
    v = cz;
  } else {
    u = cx;
    v = cy;
  }
  for (int q = 0; q < np; ++q) {
    if (p[q].face != face) continue;
    if (u >= p[q].u0 && u <= p[q].u1 && v >= p[q].v0 && v <= p[q].v1) {
      if (value) *value = p[q].value;
      return 1;
    }
  }
  return 0;
}

/* grid.cpp:77-93 */
static int validate_boundary(const orc_grid* g, const orc_patch* p, int np) {
  for (int a = 0; a < np; ++a) {
    if (p[a].u1 < p[a].u0 || p[a].v1 < p[a].v0)
      return fail(ORC_ECONFIG, "BoundarySpec: patch with negative extent");
    double lu, lv;
    if (p[a].face <= 1) {
      lu = g->ly;
      lv = g->lz;
    } else if (p[a].face <= 3) {
      lu = g->lx;
      lv = g->lz;
    } else {
      lu = g->lx;
      lv = g->ly;
    }
    if (p[a].u0 < 0.0 || p[a].v0 < 0.0 || p[a].u1 > lu || p[a].v1 > lv)
      return fail(ORC_ECONFIG, "BoundarySpec: patch outside the domain face");
    for (int b = a + 1; b < np; ++b) {
      if (p[a].face != p[b].face) continue;
      if (p[a].u0 < p[b].u1 && p[b].u0 < p[a].u1 && p[a].v0 < p[b].v1 &&
          p[b].v0 < p[a].v1)
        return fail(ORC_ECONFIG, "BoundarySpec: overlapping patches");
    }
  }
  return ORC_OK;
}

/* grid.cpp:95-105 */
orc_index orc_count_dirichlet_faces(const orc_grid* g, const orc_patch* p,
                                    int np) {
  orc_index count = 0;
  double tmp;
  for (orc_index k = 0; k < g->nz; ++k)
    for (orc_index j = 0; j < g->ny; ++j)
      for (orc_index i = 0; i < g->nx; ++i)
        for (int f = 0; f < 6; ++f)
          if (orc_dirichlet_value(g, p, np, i, j, k, f, &tmp)) ++count;
  return count;
}

/* grid.cpp:220-241 */
int orc_interpolate_design(const double* lo, const orc_grid* glo,
                           const orc_grid* ghi, double* hi) {
  const orc_index nlo[3] = {glo->nx, glo->ny, glo->nz};
  const orc_index nhi[3] = {ghi->nx, ghi->ny, ghi->nz};
  orc_index f[3];
  for (int a = 0; a < 3; ++a) {
    if (nhi[a] % nlo[a] != 0)
      return fail(ORC_ECONFIG, "interpolate_design: non-integer refinement factor");
    f[a] = nhi[a] / nlo[a];
  }
  for (orc_index k = 0; k < ghi->nz; ++k)
    for (orc_index j = 0; j < ghi->ny; ++j)
      for (orc_index i = 0; i < ghi->nx; ++i)
        hi[g_cell(ghi, i, j, k)] = lo[g_cell(glo, i / f[0], j / f[1], k / f[2])];
  return ORC_OK;
}

/* ============================================================= material */

/* material.cpp:8-15 (ctor checks), :45-59 (int_pow + conductivity) */
int orc_conductivity(orc_index n, const double* x, double kappa_lo,
                     double kappa_hi, int p, double* kappa) {
  if (!(kappa_lo > 0.0) || !(kappa_hi > kappa_lo))
    return fail(ORC_ECONFIG, "MaterialModel: requires 0 < kappa_lo < kappa_hi");
  if (p < 1) return fail(ORC_ECONFIG, "MaterialModel: penalization p must be >= 1");
  const double dk = kappa_hi - kappa_lo;
  for (orc_index c = 0; c < n; ++c) {
    double r = 1.0;
    for (int i = 0; i < p; ++i) r *= x[c];
    kappa[c] = kappa_lo + r * dk;
  }
  return ORC_OK;
}

/* ================================================================ inputs */

typedef struct {
  uint64_t s;
} lcg64;
/* rng.hpp:13-29 */
static inline double lcg_uniform(lcg64* r) {
  r->s = 6364136223846793005ULL * r->s + 1442695040888963407ULL;
  return (double)(r->s >> 11) * 0x1.0p-53;
}

typedef struct {
  double v;
  orc_index i;
} vi_pair;
static int cmp_desc_then_index(const void* a, const void* b) {
  const vi_pair* x = (const vi_pair*)a;
  const vi_pair* y = (const vi_pair*)b;
  if (x->v != y->v) return x->v > y->v ? -1 : 1;
  return x->i < y->i ? -1 : (x->i > y->i);
}

/* rng.cpp:39-51: ceil(vstar*M) largest -> 1, ties by lower index */
static void binarize_top(orc_index m, const double* field, double vstar,
                         double* rho) {
  orc_index solid = (orc_index)ceil(vstar * (double)m);
  if (solid > m) solid = m;
  vi_pair* order = XMALLOC(vi_pair, m);
  for (orc_index c = 0; c < m; ++c) {
    order[c].v = field[c];
    order[c].i = c;
  }
  qsort(order, (size_t)m, sizeof(vi_pair), cmp_desc_then_index);
  for (orc_index c = 0; c < m; ++c) rho[c] = 0.0;
  for (orc_index r = 0; r < solid; ++r) rho[order[r].i] = 1.0;
  free(order);
}

/* rng.cpp:16-53 */
void orc_frozen_bench_design(const orc_grid* g, double vstar, uint64_t seed,
                             int passes, double* rho) {
  const orc_index m = g->nx * g->ny * g->nz;
  double* field = XMALLOC(double, m);
  double* next = XMALLOC(double, m);
  lcg64 r = {seed};
  for (orc_index c = 0; c < m; ++c) field[c] = lcg_uniform(&r);
  for (int pass = 0; pass < passes; ++pass) {
    for (orc_index k = 0; k < g->nz; ++k)
      for (orc_index j = 0; j < g->ny; ++j)
        for (orc_index i = 0; i < g->nx; ++i) {
          double sum = field[g_cell(g, i, j, k)];
          int n = 1;
          if (i > 0) { sum += field[g_cell(g, i - 1, j, k)]; ++n; }
          if (i < g->nx - 1) { sum += field[g_cell(g, i + 1, j, k)]; ++n; }
          if (j > 0) { sum += field[g_cell(g, i, j - 1, k)]; ++n; }
          if (j < g->ny - 1) { sum += field[g_cell(g, i, j + 1, k)]; ++n; }
          if (k > 0) { sum += field[g_cell(g, i, j, k - 1)]; ++n; }
          if (k < g->nz - 1) { sum += field[g_cell(g, i, j, k + 1)]; ++n; }
          next[g_cell(g, i, j, k)] = sum / n;
        }
    double* t = field;
    field = next;
    next = t;
  }
  binarize_top(m, field, vstar, rho);
  free(field);
  free(next);
}

/* BASELINE.json configs[0] generator: LCG uniforms in cell
 * order; `passes` box means of radius r over the domain-clipped (2r+1)^3
 * window, computed separably (x, then y, then z window sums, each summed in
 * increasing index order) and divided by count_x*count_y*count_z; then the
 * rng.cpp:39-51 top-k binarisation. The product-side generator
 * (paper_2410_06850_b200/inputs.py) follows the same operation order. */
void orc_box_filter_design(const orc_grid* g, double vf, uint64_t seed,
                           int passes, int radius, double* rho) {
  const orc_index nx = g->nx, ny = g->ny, nz = g->nz, m = nx * ny * nz;
  double* f = XMALLOC(double, m);
  double* t = XMALLOC(double, m);
  lcg64 r = {seed};
  for (orc_index c = 0; c < m; ++c) f[c] = lcg_uniform(&r);
  const orc_index R = radius;
  for (int pass = 0; pass < passes; ++pass) {
    /* x sums: f -> t */
    for (orc_index k = 0; k < nz; ++k)
      for (orc_index j = 0; j < ny; ++j)
        for (orc_index i = 0; i < nx; ++i) {
          double s = 0.0;
          for (orc_index d = -R; d <= R; ++d) {
            const orc_index ii = i + d;
            if (ii >= 0 && ii < nx) s += f[g_cell(g, ii, j, k)];
          }
          t[g_cell(g, i, j, k)] = s;
        }
    /* y sums: t -> f */
    for (orc_index k = 0; k < nz; ++k)
      for (orc_index j = 0; j < ny; ++j)
        for (orc_index i = 0; i < nx; ++i) {
          double s = 0.0;
          for (orc_index d = -R; d <= R; ++d) {
            const orc_index jj = j + d;
            if (jj >= 0 && jj < ny) s += t[g_cell(g, i, jj, k)];
          }
          f[g_cell(g, i, j, k)] = s;
        }
    /* z sums + normalisation: f -> t, then swap */
    for (orc_index k = 0; k < nz; ++k)
      for (orc_index j = 0; j < ny; ++j)
        for (orc_index i = 0; i < nx; ++i) {
          double s = 0.0;
          for (orc_index d = -R; d <= R; ++d) {
            const orc_index kk = k + d;
            if (kk >= 0 && kk < nz) s += f[g_cell(g, i, j, kk)];
          }
          const orc_index cx = (i + R < nx - 1 ? i + R : nx - 1) - (i - R > 0 ? i - R : 0) + 1;
          const orc_index cy = (j + R < ny - 1 ? j + R : ny - 1) - (j - R > 0 ? j - R : 0) + 1;
          const orc_index cz = (k + R < nz - 1 ? k + R : nz - 1) - (k - R > 0 ? k - R : 0) + 1;
          t[g_cell(g, i, j, k)] = s / ((double)cx * (double)cy * (double)cz);
        }
    double* tmp = f;
    f = t;
    t = tmp;
  }
  binarize_top(m, f, vf, rho);
  free(f);
  free(t);
}

/* ================================================================ sparse */

typedef struct {
  orc_index row, col;
  double value;
  orc_index seq;
} trip;

static int cmp_trip(const void* a, const void* b) {
  const trip* x = (const trip*)a;
  const trip* y = (const trip*)b;
  if (x->row != y->row) return x->row < y->row ? -1 : 1;
  if (x->col != y->col) return x->col < y->col ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

void orc_csr_free(orc_csr* a) {
  if (!a) return;
  free(a->off);
  free(a->col);
  free(a->val);
  a->off = NULL;
  a->col = NULL;
  a->val = NULL;
  a->rows = a->cols = 0;
}

/* sparse.cpp:28-59 — sort by (row, col), sum duplicates. The reference uses
 * std::sort (unstable); here duplicates are summed in insertion order. */
static void csr_from_triplets(orc_index rows, orc_index cols, trip* t,
                              orc_index nt, orc_csr* out) {
  for (orc_index i = 0; i < nt; ++i) t[i].seq = i;
  qsort(t, (size_t)nt, sizeof(trip), cmp_trip);
  out->rows = rows;
  out->cols = cols;
  out->off = XCALLOC(orc_index, rows + 1);
  out->col = XMALLOC(orc_index, nt);
  out->val = XMALLOC(double, nt);
  orc_index i = 0, nnz = 0;
  while (i < nt) {
    const orc_index r = t[i].row, c = t[i].col;
    double sum = 0.0;
    while (i < nt && t[i].row == r && t[i].col == c) sum += t[i++].value;
    out->col[nnz] = c;
    out->val[nnz] = sum;
    ++nnz;
    ++out->off[r + 1];
  }
  for (orc_index r = 0; r < rows; ++r) out->off[r + 1] += out->off[r];
}

static void csr_identity(orc_index n, orc_csr* out) {
  out->rows = out->cols = n;
  out->off = XMALLOC(orc_index, n + 1);
  out->col = XMALLOC(orc_index, n);
  out->val = XMALLOC(double, n);
  for (orc_index i = 0; i <= n; ++i) out->off[i] = i;
  for (orc_index i = 0; i < n; ++i) {
    out->col[i] = i;
    out->val[i] = 1.0;
  }
}

/* sparse.cpp:71-84 — per-row sum in column order */
void orc_spmv(const orc_csr* a, const double* x, double* y) {
  for (orc_index r = 0; r < a->rows; ++r) {
    double sum = 0.0;
    for (orc_index p = a->off[r]; p < a->off[r + 1]; ++p)
      sum += a->val[p] * x[a->col[p]];
    y[r] = sum;
  }
}

/* sparse.cpp:108-123 — y = A^T x, serial scatter, skipping zero x_r */
static void csr_apply_transpose(const orc_csr* a, const double* x, double* y) {
  for (orc_index c = 0; c < a->cols; ++c) y[c] = 0.0;
  for (orc_index r = 0; r < a->rows; ++r) {
    const double xr = x[r];
    if (xr == 0.0) continue;
    for (orc_index p = a->off[r]; p < a->off[r + 1]; ++p)
      y[a->col[p]] += a->val[p] * xr;
  }
}

/* sparse.cpp:125-144 */
static void csr_transposed(const orc_csr* a, orc_csr* out) {
  const orc_index nnz = a->off[a->rows];
  orc_index* offs = XCALLOC(orc_index, a->cols + 2);
  for (orc_index p = 0; p < nnz; ++p) ++offs[a->col[p] + 2];
  for (orc_index i = 2; i < a->cols + 2; ++i) offs[i] += offs[i - 1];
  out->col = XMALLOC(orc_index, nnz);
  out->val = XMALLOC(double, nnz);
  for (orc_index r = 0; r < a->rows; ++r)
    for (orc_index p = a->off[r]; p < a->off[r + 1]; ++p) {
      const orc_index c = a->col[p];
      const orc_index slot = offs[c + 1]++;
      out->col[slot] = r;
      out->val[slot] = a->val[p];
    }
  out->rows = a->cols;
  out->cols = a->rows;
  out->off = offs; /* first cols+1 entries are the offsets */
}

static int cmp_index(const void* a, const void* b) {
  const orc_index x = *(const orc_index*)a, y = *(const orc_index*)b;
  return x < y ? -1 : (x > y);
}

/* sparse.cpp:146-229 — Gustavson row merge, fixed per-row accumulation order */
static void csr_multiply(const orc_csr* a, const orc_csr* b, orc_csr* out) {
  const orc_index ncol = b->cols;
  orc_index* marker = XMALLOC(orc_index, ncol);
  double* accum = XMALLOC(double, ncol);
  orc_index* nz = XMALLOC(orc_index, ncol);
  for (orc_index c = 0; c < ncol; ++c) marker[c] = -1;
  orc_index* offs = XCALLOC(orc_index, a->rows + 1);
  for (orc_index r = 0; r < a->rows; ++r) {
    orc_index count = 0;
    for (orc_index p = a->off[r]; p < a->off[r + 1]; ++p) {
      const orc_index k = a->col[p];
      for (orc_index q = b->off[k]; q < b->off[k + 1]; ++q) {
        const orc_index c = b->col[q];
        if (marker[c] != r) {
          marker[c] = r;
          ++count;
        }
      }
    }
    offs[r + 1] = count;
  }
  for (orc_index r = 0; r < a->rows; ++r) offs[r + 1] += offs[r];
  out->rows = a->rows;
  out->cols = ncol;
  out->off = offs;
  out->col = XMALLOC(orc_index, offs[a->rows]);
  out->val = XMALLOC(double, offs[a->rows]);
  for (orc_index c = 0; c < ncol; ++c) marker[c] = -1;
  for (orc_index r = 0; r < a->rows; ++r) {
    orc_index nnz = 0;
    for (orc_index p = a->off[r]; p < a->off[r + 1]; ++p) {
      const orc_index k = a->col[p];
      const double av = a->val[p];
      for (orc_index q = b->off[k]; q < b->off[k + 1]; ++q) {
        const orc_index c = b->col[q];
        if (marker[c] != r) {
          marker[c] = r;
          accum[c] = 0.0;
          nz[nnz++] = c;
        }
        accum[c] += av * b->val[q];
      }
    }
    qsort(nz, (size_t)nnz, sizeof(orc_index), cmp_index);
    orc_index slot = offs[r];
    for (orc_index t = 0; t < nnz; ++t) {
      out->col[slot] = nz[t];
      out->val[slot] = accum[nz[t]];
      ++slot;
    }
  }
  free(marker);
  free(accum);
  free(nz);
}

/* sparse.cpp:261-270 */
int orc_galerkin(const orc_csr* r, const orc_csr* a, orc_csr* out) {
  if (r->cols != a->rows) return fail(ORC_EARG, "galerkin: dimension mismatch");
  orc_csr ra, rt;
  csr_multiply(r, a, &ra);
  csr_transposed(r, &rt);
  csr_multiply(&ra, &rt, out);
  orc_csr_free(&ra);
  orc_csr_free(&rt);
  return ORC_OK;
}

static double csr_coeff(const orc_csr* a, orc_index r, orc_index c) {
  for (orc_index p = a->off[r]; p < a->off[r + 1]; ++p)
    if (a->col[p] == c) return a->val[p];
  return 0.0;
}

/* ============================================================= assembly */

/* fvm.cpp:9-14 */
static inline double face_t(double kl, double kr) {
  return 2.0 * kl * kr / (kl + kr);
}

/* fvm.cpp:33-166 */
int orc_assemble(const orc_grid* g, const double* kappa, const double* source,
                 const orc_patch* p, int np, orc_csr* a, double* rhs) {
  const orc_index m = g->nx * g->ny * g->nz;
  for (orc_index c = 0; c < m; ++c)
    if (!(kappa[c] > 0.0))
      return fail(ORC_ECONFIG, "assemble_system: conductivity must be positive");
  int rc = validate_boundary(g, p, np);
  if (rc) return rc;
  if (orc_count_dirichlet_faces(g, p, np) == 0)
    return fail(ORC_ECONFIG,
                "assemble_system: no Dirichlet face on the boundary, the "
                "system would be singular");
  const double hx = g_hx(g), hy = g_hy(g), hz = g_hz(g);
  const double coupling[3] = {hy * hz / hx, hx * hz / hy, hx * hy / hz};
  const double volume = hx * hy * hz;
  const orc_index n_axis[3] = {g->nx, g->ny, g->nz};
  const orc_index stride[3] = {1, g->nx, g->nx * g->ny};
  a->rows = a->cols = m;
  a->off = XMALLOC(orc_index, m + 1);
  a->col = XMALLOC(orc_index, 7 * m);
  a->val = XMALLOC(double, 7 * m);
  orc_index nnz = 0;
  a->off[0] = 0;
  for (orc_index c = 0; c < m; ++c) {
    const orc_index ijk[3] = {c % g->nx, (c / g->nx) % g->ny, c / (g->nx * g->ny)};
    double diag = 0.0;
    double b = source[c] * volume;
    orc_index rcols[7];
    double rvals[7];
    int nn = 0;
    for (int ax = 0; ax < 3; ++ax) {
      if (ijk[ax] > 0) {
        const orc_index nb = c - stride[ax];
        const double t = face_t(kappa[nb], kappa[c]) * coupling[ax];
        diag += t;
        rcols[nn] = nb;
        rvals[nn] = -t;
        ++nn;
      } else {
        double td = 0.0;
        if (orc_dirichlet_value(g, p, np, ijk[0], ijk[1], ijk[2], 2 * ax, &td)) {
          const double t = 2.0 * kappa[c] * coupling[ax];
          diag += t;
          b += t * td;
        }
      }
      if (ijk[ax] < n_axis[ax] - 1) {
        const orc_index nb = c + stride[ax];
        const double t = face_t(kappa[c], kappa[nb]) * coupling[ax];
        diag += t;
        rcols[nn] = nb;
        rvals[nn] = -t;
        ++nn;
      } else {
        double td = 0.0;
        if (orc_dirichlet_value(g, p, np, ijk[0], ijk[1], ijk[2], 2 * ax + 1, &td)) {
          const double t = 2.0 * kappa[c] * coupling[ax];
          diag += t;
          b += t * td;
        }
      }
    }
    rcols[nn] = c;
    rvals[nn] = diag;
    ++nn;
    for (int i = 1; i < nn; ++i) { /* insertion sort by column */
      const orc_index ci = rcols[i];
      const double vi = rvals[i];
      int j = i - 1;
      while (j >= 0 && rcols[j] > ci) {
        rcols[j + 1] = rcols[j];
        rvals[j + 1] = rvals[j];
        --j;
      }
      rcols[j + 1] = ci;
      rvals[j + 1] = vi;
    }
    for (int i = 0; i < nn; ++i) {
      a->col[nnz] = rcols[i];
      a->val[nnz] = rvals[i];
      ++nnz;
    }
    a->off[c + 1] = nnz;
    rhs[c] = b;
  }
  return ORC_OK;
}

/* ========================================================= coarse spaces */

/* coarse_space.cpp:238-277 as triplets (local box order) */
static orc_index box_stiffness_trips(const orc_grid* g, const double* kappa,
                                     const orc_index o[3], const orc_index e[3],
                                     trip* t) {
  const double hx = g_hx(g), hy = g_hy(g), hz = g_hz(g);
  const double coupling[3] = {hy * hz / hx, hx * hz / hy, hx * hy / hz};
  orc_index nt = 0;
#define LOC(i, j, k) ((i) + e[0] * ((j) + e[1] * (k)))
  for (orc_index k = 0; k < e[2]; ++k)
    for (orc_index j = 0; j < e[1]; ++j)
      for (orc_index i = 0; i < e[0]; ++i) {
        const orc_index gid = g_cell(g, o[0] + i, o[1] + j, o[2] + k);
        const orc_index l = LOC(i, j, k);
        const orc_index nbl[3] = {LOC(i + 1, j, k), LOC(i, j + 1, k), LOC(i, j, k + 1)};
        const orc_index nbg[3] = {g_cell(g, o[0] + i + 1, o[1] + j, o[2] + k),
                                  g_cell(g, o[0] + i, o[1] + j + 1, o[2] + k),
                                  g_cell(g, o[0] + i, o[1] + j, o[2] + k + 1)};
        const int has[3] = {i + 1 < e[0], j + 1 < e[1], k + 1 < e[2]};
        for (int ax = 0; ax < 3; ++ax) {
          if (!has[ax]) continue;
          const double tt = face_t(kappa[gid], kappa[nbg[ax]]) * coupling[ax];
          t[nt++] = (trip){l, l, tt, 0};
          t[nt++] = (trip){nbl[ax], nbl[ax], tt, 0};
          t[nt++] = (trip){l, nbl[ax], -tt, 0};
          t[nt++] = (trip){nbl[ax], l, -tt, 0};
        }
      }
#undef LOC
  return nt;
}

static void box_stiffness(const orc_grid* g, const double* kappa,
                          const orc_index o[3], const orc_index e[3],
                          orc_csr* s) {
  const orc_index n = e[0] * e[1] * e[2];
  trip* t = XMALLOC(trip, 12 * n);
  const orc_index nt = box_stiffness_trips(g, kappa, o, e, t);
  csr_from_triplets(n, n, t, nt, s);
  free(t);
}

/* lanczos_smallest (coarse_space.cpp:61-198): Lanczos with full (two-pass)
 * reorthogonalisation on sigma I - B (sigma = max(Gershgorin row bound, 1)),
 * random unit starts from Lcg64(0x5eedbeef) drawn as next_uniform() - 0.5 and
 * Gram-Schmidt'ed against the basis, Ritz pairs of the tridiagonal T checked
 * every step once m >= count (residual nb |last component| <= 1e-10 sigma),
 * deflated restart on an invariant subspace (nb < 1e-14 sigma). The j-th
 * largest Ritz value goes to slot count - 1 - j (descending in lambda); the
 * returned block is re-orthonormalised in order. b: dense n x n (row-major). */
static int lanczos_smallest(orc_index n, const double* b, orc_index count, double* values,
                            double* vecs /* count x n */) {
  double sigma = 0.0;
  for (orc_index r = 0; r < n; ++r) {
    double row = 0.0;
    for (orc_index c = 0; c < n; ++c) {
      const double v = b[r * n + c];
      if (v != 0.0 || c == r) row += (c == r) ? v : fabs(v);
    }
    if (row > sigma) sigma = row;
  }
  if (sigma < 1.0) sigma = 1.0;
  lcg64 rng = {0x5eedbeefULL};
  double* basis = XMALLOC(double, (n + 1) * n);
  double* alpha = XMALLOC(double, n + 1);
  double* beta = XMALLOC(double, n + 1);
  double* w = XMALLOC(double, n);
  orc_index m = 0;
  const double conv_tol = 1e-10 * sigma;
#define FRESH(dst)                                                                   \
  do {                                                                               \
    for (orc_index i_ = 0; i_ < n; ++i_) (dst)[i_] = lcg_uniform(&rng) - 0.5;         \
    for (orc_index q_ = 0; q_ < m; ++q_) {                                           \
      double d_ = 0.0;                                                               \
      for (orc_index i_ = 0; i_ < n; ++i_) d_ += basis[q_ * n + i_] * (dst)[i_];      \
      for (orc_index i_ = 0; i_ < n; ++i_) (dst)[i_] -= d_ * basis[q_ * n + i_];      \
    }                                                                                \
    double nn_ = 0.0;                                                                \
    for (orc_index i_ = 0; i_ < n; ++i_) nn_ += (dst)[i_] * (dst)[i_];               \
    nn_ = sqrt(nn_);                                                                 \
    for (orc_index i_ = 0; i_ < n; ++i_) (dst)[i_] /= nn_;                           \
  } while (0)
  FRESH(basis);
  orc_index nbasis = 1;
  int rc = ORC_ESOLVER;
  for (orc_index step = 0; step < n; ++step) {
    const double* q = basis + (nbasis - 1) * n;
    for (orc_index r = 0; r < n; ++r) {  /* w = sigma q - B q */
      double y = 0.0;
      for (orc_index c = 0; c < n; ++c) y += b[r * n + c] * q[c];
      w[r] = sigma * q[r] - y;
    }
    double a = 0.0;
    for (orc_index i = 0; i < n; ++i) a += q[i] * w[i];
    alpha[m++] = a;
    for (int pass = 0; pass < 2; ++pass)
      for (orc_index k = 0; k < nbasis; ++k) {
        double d = 0.0;
        for (orc_index i = 0; i < n; ++i) d += basis[k * n + i] * w[i];
        for (orc_index i = 0; i < n; ++i) w[i] -= d * basis[k * n + i];
      }
    double nb = 0.0;
    for (orc_index i = 0; i < n; ++i) nb += w[i] * w[i];
    nb = sqrt(nb);
    if (m >= count) {
      double* t = XCALLOC(double, m * m);
      double* tw = XMALLOC(double, m);
      double* tv = XMALLOC(double, m * m);
      for (orc_index i = 0; i < m; ++i) {
        t[i * m + i] = alpha[i];
        if (i + 1 < m) t[i * m + i + 1] = t[(i + 1) * m + i] = beta[i];
      }
      if (dla_syev_all((int)m, t, tw, tv)) {
        free(t), free(tw), free(tv);
        break;
      }
      int converged = 1;
      for (orc_index j = 0; j < count; ++j)
        if (nb * fabs(tv[(m - 1) * m + (m - 1 - j)]) > conv_tol) converged = 0;
      if (converged || m == n || nb < 1e-14 * sigma) {
        for (orc_index j = 0; j < count; ++j) {
          const orc_index col = m - 1 - j, dst = count - 1 - j;
          values[dst] = sigma - tw[col];
          double* v = vecs + dst * n;
          for (orc_index i = 0; i < n; ++i) v[i] = 0.0;
          for (orc_index s2 = 0; s2 < m; ++s2)
            for (orc_index i = 0; i < n; ++i) v[i] += tv[s2 * m + col] * basis[s2 * n + i];
        }
        rc = ORC_OK;
        for (orc_index j = 0; j < count && rc == ORC_OK; ++j) {
          double* vj = vecs + j * n;
          for (orc_index k2 = 0; k2 < j; ++k2) {
            double d = 0.0;
            for (orc_index i = 0; i < n; ++i) d += vecs[k2 * n + i] * vj[i];
            for (orc_index i = 0; i < n; ++i) vj[i] -= d * vecs[k2 * n + i];
          }
          double nn = 0.0;
          for (orc_index i = 0; i < n; ++i) nn += vj[i] * vj[i];
          nn = sqrt(nn);
          if (nn < 1e-14) rc = ORC_ESOLVER;
          for (orc_index i = 0; i < n; ++i) vj[i] /= nn;
        }
        free(t), free(tw), free(tv);
        break;
      }
      free(t), free(tw), free(tv);
    }
    if (m == n) break;
    if (nb < 1e-14 * sigma) {
      beta[m - 1] = 0.0;
      FRESH(basis + nbasis * n);
    } else {
      beta[m - 1] = nb;
      for (orc_index i = 0; i < n; ++i) basis[nbasis * n + i] = w[i] / nb;
    }
    ++nbasis;
  }
#undef FRESH
  free(basis), free(alpha), free(beta), free(w);
  return rc;
}

/* coarse_space.cpp:279-304 with generalized_smallest :203-234: the dense path
 * dense_smallest :38-56 up to SpectralOptions::dense_threshold = 4096 cells
 * (coarse_space.hpp:37-42), lanczos_smallest :61-198 above. */
int orc_local_basis(const orc_hgrid* h, const double* kappa, orc_index cid,
                    orc_index count, double* values, double* vectors) {
  const orc_index n = h_cells_in_coarse(h);
  if (count > n)
    return fail(ORC_EARG, "local_spectral_basis: more eigenvectors than cells requested");
  orc_index o[3];
  h_coarse_origin(h, cid, o);
  orc_csr s;
  box_stiffness(&h->spec, kappa, o, h->cpc, &s);
  orc_index* cells = XMALLOC(orc_index, n);
  box_cells(&h->spec, o, h->cpc, cells);
  const double volume = g_hx(&h->spec) * g_hy(&h->spec) * g_hz(&h->spec);
  double* inv_sqrt = XMALLOC(double, n);
  for (orc_index i = 0; i < n; ++i) {
    const double m = kappa[cells[i]] * volume;
    if (!(m > 0.0)) {
      free(inv_sqrt);
      free(cells);
      orc_csr_free(&s);
      return fail(ORC_ESOLVER, "eigensolver: nonpositive mass entry (kappa <= 0?)");
    }
    inv_sqrt[i] = 1.0 / sqrt(m);
  }
  double* dense = XCALLOC(double, n * n);
  for (orc_index r = 0; r < n; ++r)
    for (orc_index p = s.off[r]; p < s.off[r + 1]; ++p)
      dense[r * n + s.col[p]] = s.val[p] * (inv_sqrt[r] * inv_sqrt[s.col[p]]);
  double* v = XMALLOC(double, n * count);
  int rc;
  if (n <= 4096) {
    rc = dla_syev_smallest((int)n, (int)count, dense, values, v);
    if (rc == 0)
      for (orc_index c = 0; c < count; ++c)
        for (orc_index i = 0; i < n; ++i)
          vectors[c * n + i] = v[i * count + c] * inv_sqrt[i];
  } else {  /* v: count x n */
    rc = lanczos_smallest(n, dense, count, values, v);
    if (rc == 0)
      for (orc_index c = 0; c < count; ++c)
        for (orc_index i = 0; i < n; ++i) vectors[c * n + i] = v[c * n + i] * inv_sqrt[i];
  }
  free(v);
  free(dense);
  free(inv_sqrt);
  free(cells);
  orc_csr_free(&s);
  if (rc) return fail(ORC_ESOLVER, "local eigensolver failed to converge");
  return ORC_OK;
}

/* coarse_space.cpp:306-341 */
static void assemble_restriction(const orc_hgrid* h, orc_index lc,
                                 const double* vecs /* m_c x (n x lc) */,
                                 orc_csr* rc) {
  const orc_index mc = h_num_coarse(h), n = h_cells_in_coarse(h);
  const orc_index rows = lc * mc;
  rc->rows = rows;
  rc->cols = h->spec.nx * h->spec.ny * h->spec.nz;
  rc->off = XMALLOC(orc_index, rows + 1);
  rc->col = XMALLOC(orc_index, rows * n);
  rc->val = XMALLOC(double, rows * n);
  orc_index* cells = XMALLOC(orc_index, n);
  orc_index nnz = 0;
  rc->off[0] = 0;
  for (orc_index e = 0; e < mc; ++e) {
    orc_index o[3];
    h_coarse_origin(h, e, o);
    box_cells(&h->spec, o, h->cpc, cells);
    for (orc_index j = 0; j < lc; ++j) {
      for (orc_index i = 0; i < n; ++i) {
        rc->col[nnz] = cells[i];
        rc->val[nnz] = vecs[e * n * lc + j * n + i];
        ++nnz;
      }
      rc->off[e * lc + j + 1] = nnz;
    }
  }
  free(cells);
}

/* coarse_space.cpp:343-406 */
int orc_cc_basis(const orc_hgrid* h, const double* kappa, const orc_csr* rc,
                 orc_index cc_id, orc_index count, double* values,
                 double* vectors) {
  const orc_index mc = h_num_coarse(h);
  if (rc->rows % mc != 0)
    return fail(ORC_EARG, "coarse_coarse_basis: restriction rows not uniform per element");
  const orc_index per = rc->rows / mc;
  const orc_index sd3 = h->sd * h->sd * h->sd;
  orc_index* children = XMALLOC(orc_index, sd3);
  h_coarse_children(h, cc_id, children);
  const orc_index q = sd3 * per;
  if (count > q) {
    free(children);
    return fail(ORC_EARG, "coarse_coarse_basis: more eigenvectors than coarse basis functions");
  }
  orc_index* rows = XMALLOC(orc_index, q);
  for (orc_index c = 0; c < sd3; ++c)
    for (orc_index j = 0; j < per; ++j) rows[c * per + j] = children[c] * per + j;
  orc_index o[3], e[3];
  h_cc_origin(h, cc_id, o);
  for (int a = 0; a < 3; ++a) e[a] = h->cpc[a] * h->sd;
  orc_csr s;
  box_stiffness(&h->spec, kappa, o, e, &s);
  const orc_index nloc = e[0] * e[1] * e[2];
  double* P = XCALLOC(double, q * nloc);
  for (orc_index r = 0; r < q; ++r)
    for (orc_index ptr = rc->off[rows[r]]; ptr < rc->off[rows[r] + 1]; ++ptr) {
      const orc_index g = rc->col[ptr];
      const orc_index gx = g % h->spec.nx, gy = (g / h->spec.nx) % h->spec.ny,
                      gz = g / (h->spec.nx * h->spec.ny);
      const orc_index loc = (gx - o[0]) + e[0] * ((gy - o[1]) + e[1] * (gz - o[2]));
      P[r * nloc + loc] = rc->val[ptr];
    }
  /* SP = S * P^T  (nloc x q), then projected = P * SP (q x q) */
  double* SP = XCALLOC(double, nloc * q);
  for (orc_index r = 0; r < nloc; ++r)
    for (orc_index p = s.off[r]; p < s.off[r + 1]; ++p) {
      const double v = s.val[p];
      const orc_index c = s.col[p];
      for (orc_index t = 0; t < q; ++t) SP[r * q + t] += v * P[t * nloc + c];
    }
  double* proj = XCALLOC(double, q * q);
  for (orc_index a = 0; a < q; ++a)
    for (orc_index r = 0; r < nloc; ++r) {
      const double pa = P[a * nloc + r];
      if (pa == 0.0) continue;
      for (orc_index b = 0; b < q; ++b) proj[a * q + b] += pa * SP[r * q + b];
    }
  double* sym = XMALLOC(double, q * q);
  for (orc_index a = 0; a < q; ++a)
    for (orc_index b = 0; b < q; ++b)
      sym[a * q + b] = 0.5 * (proj[a * q + b] + proj[b * q + a]);
  double* v = XMALLOC(double, q * count);
  const int rc2 = dla_syev_smallest((int)q, (int)count, sym, values, v);
  if (rc2 == 0)
    for (orc_index c = 0; c < count; ++c)
      for (orc_index i = 0; i < q; ++i) vectors[c * q + i] = v[i * count + c];
  free(v);
  free(sym);
  free(proj);
  free(SP);
  free(P);
  orc_csr_free(&s);
  free(rows);
  free(children);
  if (rc2) return fail(ORC_ESOLVER, "coarse-coarse eigensolver failed to converge");
  return ORC_OK;
}

/* coarse_space.cpp:408-426 */
static void assemble_cc_restriction(const orc_hgrid* h, orc_index lc,
                                    orc_index lcc, const double* ccvecs,
                                    orc_csr* rcc) {
  const orc_index mcc = h_num_cc(h), sd3 = h->sd * h->sd * h->sd;
  const orc_index q = sd3 * lc;
  trip* t = XMALLOC(trip, mcc * lcc * q);
  orc_index* children = XMALLOC(orc_index, sd3);
  orc_index nt = 0, row = 0;
  for (orc_index e = 0; e < mcc; ++e) {
    h_coarse_children(h, e, children);
    for (orc_index j = 0; j < lcc; ++j, ++row)
      for (orc_index i = 0; i < q; ++i) {
        const orc_index crow = children[i / lc] * lc + (i % lc);
        t[nt++] = (trip){row, crow, ccvecs[e * q * lcc + j * q + i], 0};
      }
  }
  csr_from_triplets(row, lc * h_num_coarse(h), t, nt, rcc);
  free(children);
  free(t);
}

static int local_bases_all(const orc_hgrid* h, const double* kappa,
                           orc_index lc, double* vecs) {
  const orc_index mc = h_num_coarse(h), n = h_cells_in_coarse(h);
  int err = 0;
  char msg[512] = {0};
#pragma omp parallel for schedule(dynamic, 1)
  for (orc_index e = 0; e < mc; ++e) {
    double vals[4096];
    if (err) continue;
    const int rc = orc_local_basis(h, kappa, e, lc, vals, vecs + e * n * lc);
    if (rc) {
#pragma omp critical
      {
        if (!err) {
          err = rc;
          snprintf(msg, sizeof msg, "%s", orc_last_error());
        }
      }
    }
  }
  if (err) return fail(err, "%s", msg);
  return ORC_OK;
}

/* coarse_space.cpp:428-457 */
int orc_build_coarse_spaces(const orc_hgrid* h, const double* kappa,
                            orc_index lc, orc_index lcc, orc_csr* rc,
                            orc_csr* rcc) {
  const orc_index mc = h_num_coarse(h), n = h_cells_in_coarse(h);
  const orc_index mcc = h_num_cc(h), q = h->sd * h->sd * h->sd * lc;
  double* vecs = XMALLOC(double, mc * n * lc);
  int rcode = local_bases_all(h, kappa, lc, vecs);
  if (rcode) {
    free(vecs);
    return rcode;
  }
  assemble_restriction(h, lc, vecs, rc);
  free(vecs);
  double* ccv = XMALLOC(double, mcc * q * lcc);
  int err = 0;
  char msg[512] = {0};
#pragma omp parallel for schedule(dynamic, 1)
  for (orc_index e = 0; e < mcc; ++e) {
    if (err) continue;
    double* vals = XMALLOC(double, lcc);
    const int r2 = orc_cc_basis(h, kappa, rc, e, lcc, vals, ccv + e * q * lcc);
    free(vals);
    if (r2) {
#pragma omp critical
      {
        if (!err) {
          err = r2;
          snprintf(msg, sizeof msg, "%s", orc_last_error());
        }
      }
    }
  }
  if (err) {
    free(ccv);
    orc_csr_free(rc);
    return fail(err, "%s", msg);
  }
  assemble_cc_restriction(h, lc, lcc, ccv, rcc);
  free(ccv);
  return ORC_OK;
}

/* ======================================================== direct solver */

/* DirectSolver (solver.cpp:60-126): symmetric LDL^T with the singular-pivot
 * rule d_i > 1e-14 max|d|. Both the reference's dense (n < 4096) and sparse
 * (SimplicialLDLT) branches are restated by one envelope LDL^T in natural
 * order (same factorisation in exact arithmetic). */
typedef struct {
  orc_index n;
  orc_index* first;
  orc_index* rowptr;
  double* vals;
  double* d;
} direct_solver;

static void direct_free(direct_solver* s) {
  free(s->first);
  free(s->rowptr);
  free(s->vals);
  free(s->d);
  memset(s, 0, sizeof *s);
}

static int direct_factor(const orc_csr* a, direct_solver* s) {
  if (a->rows != a->cols) return fail(ORC_EARG, "DirectSolver: matrix must be square");
  const orc_index n = a->rows;
  s->n = n;
  s->first = XMALLOC(orc_index, n);
  s->rowptr = XMALLOC(orc_index, n + 1);
  s->d = XMALLOC(double, n);
  for (orc_index i = 0; i < n; ++i) {
    orc_index f = i;
    for (orc_index p = a->off[i]; p < a->off[i + 1]; ++p)
      if (a->col[p] < f) f = a->col[p];
    s->first[i] = f;
  }
  /* symmetric envelope: first[j] also covers column entries above */
  for (orc_index i = 0; i < n; ++i)
    for (orc_index p = a->off[i]; p < a->off[i + 1]; ++p) {
      const orc_index c = a->col[p];
      if (c > i && s->first[c] > i) s->first[c] = i;
    }
  s->rowptr[0] = 0;
  for (orc_index i = 0; i < n; ++i) s->rowptr[i + 1] = s->rowptr[i] + (i - s->first[i] + 1);
  s->vals = XCALLOC(double, s->rowptr[n]);
  for (orc_index i = 0; i < n; ++i)
    for (orc_index p = a->off[i]; p < a->off[i + 1]; ++p) {
      const orc_index c = a->col[p];
      if (c <= i) s->vals[s->rowptr[i] + (c - s->first[i])] = a->val[p];
    }
  double maxp = 0.0;
  orc_index bad = -1;
  const int rc = dla_env_ldlt_factor(n, s->first, s->rowptr, s->vals, s->d, &maxp, &bad);
  if (rc) {
    const double piv = bad >= 0 ? s->d[bad] : 0.0;
    direct_free(s);
    return fail(ORC_ESOLVER, "DirectSolver: matrix numerically singular, pivot %g at index %lld",
                piv, (long long)bad);
  }
  return ORC_OK;
}

static void direct_solve(const direct_solver* s, double* x) {
  dla_env_ldlt_solve(s->n, s->first, s->rowptr, s->vals, s->d, x);
}

/* ============================================== block Jacobi smoother */

typedef struct {
  orc_index nblocks;
  orc_index* bptr; /* block b ids at ids[bptr[b] .. bptr[b+1]) */
  orc_index* ids;
  direct_solver* solvers;
  int sweeps;
  orc_index n;
} bj_smoother;

static void bj_free(bj_smoother* s) {
  if (s->solvers)
    for (orc_index b = 0; b < s->nblocks; ++b) direct_free(&s->solvers[b]);
  free(s->solvers);
  free(s->bptr);
  free(s->ids);
  memset(s, 0, sizeof *s);
}

/* solver.cpp:140-204 (partition check, block extraction, factorisation) */
static int bj_build(const orc_csr* a, orc_index nblocks, orc_index* bptr,
                    orc_index* ids, int sweeps, bj_smoother* s) {
  memset(s, 0, sizeof *s);
  if (sweeps < 0) return fail(ORC_EARG, "BlockJacobiSmoother: negative sweep count");
  s->sweeps = sweeps;
  s->n = a->rows;
  s->nblocks = nblocks;
  s->bptr = bptr;
  s->ids = ids;
  char* seen = XCALLOC(char, a->rows);
  orc_index covered = 0;
  for (orc_index t = 0; t < bptr[nblocks]; ++t) {
    const orc_index id = ids[t];
    if (id < 0 || id >= a->rows || seen[id]) {
      free(seen);
      return fail(ORC_EARG, "BlockJacobiSmoother: blocks must partition the index set");
    }
    seen[id] = 1;
    ++covered;
  }
  free(seen);
  if (covered != a->rows)
    return fail(ORC_EARG, "BlockJacobiSmoother: blocks must cover every index");
  s->solvers = XCALLOC(direct_solver, nblocks);
  orc_index* local_of = XMALLOC(orc_index, a->rows);
  for (orc_index i = 0; i < a->rows; ++i) local_of[i] = -1;
  int err = 0;
  for (orc_index b = 0; b < nblocks && !err; ++b) {
    const orc_index nb = bptr[b + 1] - bptr[b];
    const orc_index* bid = ids + bptr[b];
    for (orc_index i = 0; i < nb; ++i) local_of[bid[i]] = i;
    orc_index cap = 0;
    for (orc_index i = 0; i < nb; ++i) cap += a->off[bid[i] + 1] - a->off[bid[i]];
    trip* t = XMALLOC(trip, cap);
    orc_index nt = 0;
    for (orc_index i = 0; i < nb; ++i)
      for (orc_index p = a->off[bid[i]]; p < a->off[bid[i] + 1]; ++p) {
        const orc_index lc = local_of[a->col[p]];
        if (lc >= 0) t[nt++] = (trip){i, lc, a->val[p], 0};
      }
    orc_csr sub;
    csr_from_triplets(nb, nb, t, nt, &sub);
    free(t);
    for (orc_index i = 0; i < nb; ++i) local_of[bid[i]] = -1;
    const int rc = direct_factor(&sub, &s->solvers[b]);
    orc_csr_free(&sub);
    if (rc) {
      char m2[512];
      snprintf(m2, sizeof m2, "%s", orc_last_error());
      err = fail(ORC_ESOLVER, "BlockJacobiSmoother: singular block: %s", m2);
    }
  }
  free(local_of);
  return err;
}

/* solver.cpp:215-244 */
static void bj_apply(const bj_smoother* s, const orc_csr* a, const double* r,
                     double* z) {
  const orc_index n = s->n;
  for (orc_index i = 0; i < n; ++i) z[i] = 0.0;
  if (s->sweeps == 0) return;
  double* resid = XMALLOC(double, n);
  memcpy(resid, r, sizeof(double) * (size_t)n);
  double* local = NULL;
  orc_index lcap = 0;
  for (int sweep = 0; sweep < s->sweeps; ++sweep) {
    if (sweep > 0) {
      orc_spmv(a, z, resid);
      for (orc_index i = 0; i < n; ++i) resid[i] = r[i] - resid[i];
    }
    for (orc_index b = 0; b < s->nblocks; ++b) {
      const orc_index nb = s->bptr[b + 1] - s->bptr[b];
      const orc_index* bid = s->ids + s->bptr[b];
      if (nb > lcap) {
        free(local);
        lcap = nb;
        local = XMALLOC(double, lcap);
      }
      for (orc_index i = 0; i < nb; ++i) local[i] = resid[bid[i]];
      direct_solve(&s->solvers[b], local);
      for (orc_index i = 0; i < nb; ++i) z[bid[i]] += local[i];
    }
  }
  free(local);
  free(resid);
}

/* ========================================================= preconditioners */

struct orc_precond {
  int kind;
  orc_index n;
  double* inv_diag; /* Jacobi */
  orc_csr a, rc, rcc, ac, acc;
  bj_smoother fine, coarse;
  direct_solver acc_solver;
  int sweeps;
};

/* solver.cpp:353-360: one block per cc element (all its fine cells) */
static void fine_blocks_by_cc(const orc_hgrid* h, orc_index* nb, orc_index** bptr,
                              orc_index** ids) {
  const orc_index mcc = h_num_cc(h);
  orc_index e3[3];
  for (int a = 0; a < 3; ++a) e3[a] = h->cpc[a] * h->sd;
  const orc_index per = e3[0] * e3[1] * e3[2];
  *nb = mcc;
  *bptr = XMALLOC(orc_index, mcc + 1);
  *ids = XMALLOC(orc_index, mcc * per);
  for (orc_index e = 0; e < mcc; ++e) {
    (*bptr)[e] = e * per;
    orc_index o[3];
    h_cc_origin(h, e, o);
    box_cells(&h->spec, o, e3, *ids + e * per);
  }
  (*bptr)[mcc] = mcc * per;
}

/* one fine block per coarse cell: cells_of_coarse(I) (grid.cpp:169-173) */
static void fine_blocks_by_cell(const orc_hgrid* h, orc_index* nb,
                                orc_index** bptr, orc_index** ids) {
  const orc_index mc = h_num_coarse(h), per = h_cells_in_coarse(h);
  *nb = mc;
  *bptr = XMALLOC(orc_index, mc + 1);
  *ids = XMALLOC(orc_index, mc * per);
  for (orc_index e = 0; e < mc; ++e) {
    (*bptr)[e] = e * per;
    orc_index o[3];
    h_coarse_origin(h, e, o);
    box_cells(&h->spec, o, h->cpc, *ids + e * per);
  }
  (*bptr)[mc] = mc * per;
}

/* fine blocks = boxes of b x b x b cells (b divides the grid), box order */
static void fine_blocks_by_box(const orc_grid* g, orc_index b, orc_index* nb,
                               orc_index** bptr, orc_index** ids) {
  const orc_index bx = g->nx / b, by = g->ny / b, bz = g->nz / b;
  const orc_index m = bx * by * bz, per = b * b * b;
  const orc_index e3[3] = {b, b, b};
  *nb = m;
  *bptr = XMALLOC(orc_index, m + 1);
  *ids = XMALLOC(orc_index, m * per);
  for (orc_index e = 0; e < m; ++e) {
    (*bptr)[e] = e * per;
    const orc_index o[3] = {(e % bx) * b, ((e / bx) % by) * b, (e / (bx * by)) * b};
    box_cells(g, o, e3, *ids + e * per);
  }
  (*bptr)[m] = m * per;
}

static void point_blocks(orc_index n, orc_index* nb, orc_index** bptr,
                         orc_index** ids) {
  *nb = n;
  *bptr = XMALLOC(orc_index, n + 1);
  *ids = XMALLOC(orc_index, n);
  for (orc_index i = 0; i <= n; ++i) (*bptr)[i] = i;
  for (orc_index i = 0; i < n; ++i) (*ids)[i] = i;
}

/* solver.cpp:362-374 */
static void coarse_blocks_by_cc(const orc_hgrid* h, orc_index lc, orc_index* nb,
                                orc_index** bptr, orc_index** ids) {
  const orc_index mcc = h_num_cc(h), sd3 = h->sd * h->sd * h->sd;
  const orc_index per = sd3 * lc;
  orc_index* children = XMALLOC(orc_index, sd3);
  *nb = mcc;
  *bptr = XMALLOC(orc_index, mcc + 1);
  *ids = XMALLOC(orc_index, mcc * per);
  for (orc_index e = 0; e < mcc; ++e) {
    (*bptr)[e] = e * per;
    h_coarse_children(h, e, children);
    for (orc_index c = 0; c < sd3; ++c)
      for (orc_index j = 0; j < lc; ++j) (*ids)[e * per + c * lc + j] = children[c] * lc + j;
  }
  (*bptr)[mcc] = mcc * per;
  free(children);
}

/* one L_c x L_c block per coarse cell: rows {I*L_c .. I*L_c+L_c-1} */
static void coarse_blocks_by_cell(const orc_hgrid* h, orc_index lc,
                                  orc_index* nb, orc_index** bptr,
                                  orc_index** ids) {
  const orc_index mc = h_num_coarse(h);
  *nb = mc;
  *bptr = XMALLOC(orc_index, mc + 1);
  *ids = XMALLOC(orc_index, mc * lc);
  for (orc_index i = 0; i <= mc; ++i) (*bptr)[i] = i * lc;
  for (orc_index i = 0; i < mc * lc; ++i) (*ids)[i] = i;
}

static void csr_copy(const orc_csr* a, orc_csr* out) {
  const orc_index nnz = a->off[a->rows];
  out->rows = a->rows;
  out->cols = a->cols;
  out->off = XMALLOC(orc_index, a->rows + 1);
  out->col = XMALLOC(orc_index, nnz);
  out->val = XMALLOC(double, nnz);
  memcpy(out->off, a->off, sizeof(orc_index) * (size_t)(a->rows + 1));
  memcpy(out->col, a->col, sizeof(orc_index) * (size_t)nnz);
  memcpy(out->val, a->val, sizeof(double) * (size_t)nnz);
}

void orc_precond_free(orc_precond* m) {
  if (!m) return;
  free(m->inv_diag);
  orc_csr_free(&m->a);
  orc_csr_free(&m->rc);
  orc_csr_free(&m->rcc);
  orc_csr_free(&m->ac);
  orc_csr_free(&m->acc);
  bj_free(&m->fine);
  bj_free(&m->coarse);
  direct_free(&m->acc_solver);
  free(m);
}

const orc_csr* orc_precond_op(const orc_precond* m, int which) {
  if (m->kind != ORC_MMG && m->kind != ORC_TWO_GRID) return NULL;
  switch (which) {
    case 0: return &m->a;
    case 1: return &m->rc;
    case 2: return &m->rcc;
    case 3: return &m->ac;
    case 4: return &m->acc;
  }
  return NULL;
}

/* solver.cpp:253-270 + build_mmg :387-399 / build_two_grid :401-420 /
 * make_preconditioner :462-481 / JacobiPreconditioner :21-29 */
int orc_make_preconditioner(int kind, const orc_csr* a, const orc_hgrid* h,
                            const double* kappa, orc_index lc, orc_index lcc,
                            int sweeps, int fine_blocks, int coarse_blocks,
                            orc_precond** out) {
  orc_precond* m = XCALLOC(orc_precond, 1);
  m->kind = kind;
  m->n = a->rows;
  m->sweeps = sweeps;
  int rc = ORC_OK;
  if (kind == ORC_NONE) {
    *out = m;
    return ORC_OK;
  }
  if (kind == ORC_JACOBI) {
    m->inv_diag = XMALLOC(double, a->rows);
    for (orc_index i = 0; i < a->rows; ++i) {
      const double d = csr_coeff(a, i, i);
      if (!(d > 0.0)) {
        orc_precond_free(m);
        return fail(ORC_ESOLVER, "JacobiPreconditioner: nonpositive diagonal entry");
      }
      m->inv_diag[i] = 1.0 / d;
    }
    *out = m;
    return ORC_OK;
  }
  orc_index nb, *bptr, *ids;
  if (kind == ORC_BLOCK_JACOBI) {
    csr_copy(a, &m->a);
    if (fine_blocks == ORC_BLOCKS_POINT)
      point_blocks(a->rows, &nb, &bptr, &ids);
    else
      fine_blocks_by_cc(h, &nb, &bptr, &ids);
    rc = bj_build(&m->a, nb, bptr, ids, 1, &m->fine);
    if (rc) {
      orc_precond_free(m);
      return rc;
    }
    *out = m;
    return ORC_OK;
  }
  /* MMG / two-grid */
  csr_copy(a, &m->a);
  if (kind == ORC_MMG) {
    rc = orc_build_coarse_spaces(h, kappa, lc, lcc, &m->rc, &m->rcc);
  } else {
    const orc_index mc = h_num_coarse(h), n = h_cells_in_coarse(h);
    double* vecs = XMALLOC(double, mc * n * lc);
    rc = local_bases_all(h, kappa, lc, vecs);
    if (!rc) {
      assemble_restriction(h, lc, vecs, &m->rc);
      csr_identity(m->rc.rows, &m->rcc);
    }
    free(vecs);
  }
  if (rc) {
    orc_precond_free(m);
    return rc;
  }
  if (m->rc.cols != m->a.rows || m->rcc.cols != m->rc.rows) {
    orc_precond_free(m);
    return fail(ORC_EARG, "MultiscaleHierarchy: dimension mismatch");
  }
  orc_galerkin(&m->rc, &m->a, &m->ac);
  orc_galerkin(&m->rcc, &m->ac, &m->acc);
  if (fine_blocks == ORC_BLOCKS_POINT)
    point_blocks(m->a.rows, &nb, &bptr, &ids);
  else if (fine_blocks == ORC_BLOCKS_CELL)
    fine_blocks_by_cell(h, &nb, &bptr, &ids);
  else if (fine_blocks >= ORC_BLOCKS_BOX0)
    fine_blocks_by_box(&h->spec, fine_blocks - ORC_BLOCKS_BOX0, &nb, &bptr, &ids);
  else
    fine_blocks_by_cc(h, &nb, &bptr, &ids);
  rc = bj_build(&m->a, nb, bptr, ids, sweeps, &m->fine);
  if (!rc) {
    if (coarse_blocks == ORC_BLOCKS_CELL)
      coarse_blocks_by_cell(h, lc, &nb, &bptr, &ids);
    else
      coarse_blocks_by_cc(h, lc, &nb, &bptr, &ids);
    rc = bj_build(&m->ac, nb, bptr, ids, sweeps, &m->coarse);
  }
  if (!rc) rc = direct_factor(&m->acc, &m->acc_solver);
  if (rc) {
    orc_precond_free(m);
    return rc;
  }
  *out = m;
  return ORC_OK;
}

/* solver.cpp:272-334 */
static void mmg_apply(const orc_precond* m, const double* r, double* z) {
  const orc_index n = m->a.rows, nc = m->ac.rows, ncc = m->acc.rows;
  double* r1 = XMALLOC(double, n);
  double* work = XMALLOC(double, n);
  double* rc = XMALLOC(double, nc);
  double* rc0 = XMALLOC(double, nc);
  double* workc = XMALLOC(double, nc);
  double* rcc = XMALLOC(double, ncc);
  double* rc1 = XMALLOC(double, nc);
  double* ec = XMALLOC(double, nc);
  double* r2 = XMALLOC(double, n);
  bj_apply(&m->fine, &m->a, r, r1);
  orc_spmv(&m->a, r1, work);
  for (orc_index i = 0; i < n; ++i) work[i] = r[i] - work[i];
  orc_spmv(&m->rc, work, rc);
  bj_apply(&m->coarse, &m->ac, rc, rc0);
  orc_spmv(&m->ac, rc0, workc);
  for (orc_index i = 0; i < nc; ++i) workc[i] = rc[i] - workc[i];
  orc_spmv(&m->rcc, workc, rcc);
  direct_solve(&m->acc_solver, rcc); /* ecc in place */
  csr_apply_transpose(&m->rcc, rcc, rc1);
  for (orc_index i = 0; i < nc; ++i) rc1[i] += rc0[i];
  orc_spmv(&m->ac, rc1, workc);
  for (orc_index i = 0; i < nc; ++i) workc[i] = rc[i] - workc[i];
  bj_apply(&m->coarse, &m->ac, workc, ec);
  for (orc_index i = 0; i < nc; ++i) ec[i] += rc1[i];
  csr_apply_transpose(&m->rc, ec, r2);
  for (orc_index i = 0; i < n; ++i) r2[i] += r1[i];
  orc_spmv(&m->a, r2, work);
  for (orc_index i = 0; i < n; ++i) work[i] = r[i] - work[i];
  bj_apply(&m->fine, &m->a, work, z);
  for (orc_index i = 0; i < n; ++i) z[i] += r2[i];
  free(r1);
  free(work);
  free(rc);
  free(rc0);
  free(workc);
  free(rcc);
  free(rc1);
  free(ec);
  free(r2);
}

int orc_precond_apply(const orc_precond* m, const double* r, double* z) {
  switch (m->kind) {
    case ORC_NONE: /* solver.cpp:14-19 */
      memcpy(z, r, sizeof(double) * (size_t)m->n);
      return ORC_OK;
    case ORC_JACOBI: /* solver.cpp:31-36 */
      for (orc_index i = 0; i < m->n; ++i) z[i] = r[i] * m->inv_diag[i];
      return ORC_OK;
    case ORC_BLOCK_JACOBI: /* solver.cpp:450-452 */
      bj_apply(&m->fine, &m->a, r, z);
      return ORC_OK;
    default:
      mmg_apply(m, r, z);
      return ORC_OK;
  }
}

/* ================================================================== PCG */

/* solver.cpp:483-575 */
int orc_pcg(const orc_csr* a, const double* b, const orc_precond* m,
            double rtol, int max_iterations, const double* x0, double* x,
            double* history, orc_report* rep) {
  const orc_index n = a->rows;
  if (a->cols != n) return fail(ORC_EARG, "pcg: operator must be square");
  const double t0 = now_s();
  rep->iterations = 0;
  rep->converged = 0;
  double bb = 0.0;
  for (orc_index i = 0; i < n; ++i) bb += b[i] * b[i];
  const double bnorm = sqrt(bb);
  if (bnorm == 0.0) {
    for (orc_index i = 0; i < n; ++i) x[i] = 0.0;
    rep->converged = 1;
    rep->solve_seconds = now_s() - t0;
    return ORC_OK;
  }
  for (orc_index i = 0; i < n; ++i) x[i] = x0 ? x0[i] : 0.0;
  double* r = XMALLOC(double, n);
  double* z = XMALLOC(double, n);
  double* p = XMALLOC(double, n);
  double* q = XMALLOC(double, n);
  orc_spmv(a, x, r);
  for (orc_index i = 0; i < n; ++i) r[i] = b[i] - r[i];
  double rr = 0.0;
  for (orc_index i = 0; i < n; ++i) rr += r[i] * r[i];
  double rnorm = sqrt(rr);
  int status = ORC_OK;
  if (rnorm / bnorm <= rtol) {
    rep->converged = 1;
    goto done;
  }
  orc_precond_apply(m, r, z);
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rho = 0.0;
  for (orc_index i = 0; i < n; ++i) rho += r[i] * z[i];
  for (int it = 1; it <= max_iterations; ++it) {
    orc_spmv(a, p, q);
    double pq = 0.0;
    for (orc_index i = 0; i < n; ++i) pq += p[i] * q[i];
    if (!(pq > 0.0)) {
      status = fail(ORC_ESOLVER,
                    "pcg: operator or preconditioner not positive definite "
                    "(p^T A p = %g at iteration %d)",
                    pq, it);
      goto done;
    }
    const double alpha = rho / pq;
    for (orc_index i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
    }
    rr = 0.0;
    for (orc_index i = 0; i < n; ++i) rr += r[i] * r[i];
    rnorm = sqrt(rr);
    if (history) history[it - 1] = rnorm / bnorm;
    rep->iterations = it;
    if (rnorm / bnorm <= rtol) {
      rep->converged = 1;
      break;
    }
    orc_precond_apply(m, r, z);
    double rho_next = 0.0;
    for (orc_index i = 0; i < n; ++i) rho_next += r[i] * z[i];
    const double beta = rho_next / rho;
    rho = rho_next;
    for (orc_index i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
done:
  free(r);
  free(z);
  free(p);
  free(q);
  rep->solve_seconds = now_s() - t0;
  return status;
}
