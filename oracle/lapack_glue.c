/* ORACLE — test infrastructure only.
 * LAPACK backend for the Eigen-API shim's SelfAdjointEigenSolver (the analogue
 * of building Eigen with EIGEN_USE_LAPACKE): dsyevr for the k smallest
 * eigenpairs, from the OpenBLAS that numpy bundles (ILP64, "scipy_"-prefixed
 * symbols). Falls back to oracle/dense_la.c when that library is absent. Only
 * the reference build (oracle/_ref) links this file; the oracle restatement
 * keeps its own eigensolver so the two stay independent. */
#define _GNU_SOURCE
#include <dlfcn.h>
#include <glob.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "dense_la.h"

typedef int64_t (*dsyevr_fn)(int, char, char, char, int64_t, double*, int64_t, double, double,
                             int64_t, int64_t, double, int64_t*, double*, double*, int64_t,
                             int64_t*);
typedef void (*set_threads_fn)(int);

static dsyevr_fn g_dsyevr = NULL;
static int g_tried = 0;

static void load(void) {
  if (g_tried) return;
  g_tried = 1;
  const char* env = getenv("TOPMG_LAPACK");
  void* h = NULL;
  if (env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    glob_t gl;
    if (glob("/opt/prime-rl/.venv/lib/python3*/site-packages/numpy.libs/libscipy_openblas64_*.so",
             0, NULL, &gl) == 0 && gl.gl_pathc > 0)
      h = dlopen(gl.gl_pathv[0], RTLD_NOW | RTLD_LOCAL);
    globfree(&gl);
  }
  if (!h) return;
  g_dsyevr = (dsyevr_fn)dlsym(h, "scipy_LAPACKE_dsyevr64_");
  set_threads_fn st = (set_threads_fn)dlsym(h, "scipy_openblas_set_num_threads64_");
  if (st) st(1); /* parallelism comes from the reference's parallel_for */
}

int dla_lapack_available(void) {
  load();
  return g_dsyevr != NULL;
}

/* k smallest eigenpairs of the symmetric n x n row-major a (destroyed).
 * w: k ascending, v: n x k row-major. */
int dla_syev_smallest_lapack(int n, int k, double* a, double* w, double* v) {
  load();
  if (!g_dsyevr) return dla_syev_smallest(n, k, a, w, v);
  int64_t m = 0;
  int64_t* isuppz = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(k > 0 ? k : 1));
  double* wall = (double*)malloc(sizeof(double) * (size_t)n);
  /* row-major layout 101, jobz V, range I (il..iu 1-based), uplo L */
  const int64_t info = g_dsyevr(101, 'V', 'I', 'L', n, a, n, 0.0, 0.0, 1, k, 0.0, &m, wall, v, k,
                                isuppz);
  if (info == 0) memcpy(w, wall, sizeof(double) * (size_t)k);
  free(isuppz);
  free(wall);
  return info == 0 && m == k ? 0 : -1;
}
