/* ORACLE — test infrastructure only (see dense_la.c header). */
#ifndef TOPMG_ORACLE_DENSE_LA_H
#define TOPMG_ORACLE_DENSE_LA_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* All eigenpairs of the symmetric n x n row-major matrix a (destroyed).
 * w: n eigenvalues ascending; v: n x n row-major, column c = eigenvector c. */
int dla_syev_all(int n, double* a, double* w, double* v);

/* The k smallest eigenpairs. w: k ascending; v: n x k row-major. */
int dla_syev_smallest(int n, int k, double* a, double* w, double* v);

/* All eigenvalues ascending + the k smallest eigenvectors (v: n x k). */
int dla_syev_partial(int n, int k, double* a, double* w_all, double* v);

/* Envelope LDL^T (no pivoting) of an SPD matrix; row i holds columns
 * [first[i], i] at vals[rowptr[i]..]. Returns -1 (bad_index set) when a pivot
 * fails d_i > 1e-14 * max|d| (the rule of proj/core/src/solver.cpp:86-92). */
int dla_env_ldlt_factor(int64_t n, const int64_t* first, const int64_t* rowptr,
                        double* vals, double* d, double* max_pivot_out,
                        int64_t* bad_index_out);
void dla_env_ldlt_solve(int64_t n, const int64_t* first, const int64_t* rowptr,
                        const double* vals, const double* d, double* x);

#ifdef __cplusplus
}
#endif
#endif
