// Scalar logic of pcg() (solver.cpp:483-575) shared by the last-block
// reductions of the iteration kernels (pcg.cu, block_jacobi.cu) and
// k_finalize.
#pragma once
#include "kernels.h"

namespace tmg {

__device__ __forceinline__ bool is_finite(double v) { return isfinite(v); }

__device__ __forceinline__ void fin_init(PcgState* st, double bb, double rr) {
  const double bnorm = sqrt(bb), rnorm = sqrt(rr);
  st->bnorm = bnorm;
  st->rnorm = rnorm;
  st->it = 0;
  st->first = 0;
  if (bnorm == 0.0) {  // solver.cpp:506-513
    st->status = kStatusZeroRhs;
    st->done = 1;
  } else if (rnorm / bnorm <= st->rtol) {  // :523-531
    st->status = kStatusConverged;
    st->done = 1;
  } else {
    st->status = kStatusRunning;
    st->done = 0;
  }
}

__device__ __forceinline__ void fin_search(PcgState* st, double pqt) {
  st->pq = pqt;
  st->first = 0;
  if (!(pqt > 0.0)) {  // solver.cpp:541-548
    st->status = kStatusIndefinite;
    st->done = 1;
  } else {
    st->alpha = st->rho / pqt;  // :549
  }
}

__device__ __forceinline__ void finish_rr(PcgState* st, double rr, double* history) {
  const int it = st->it + 1;
  const double rel = sqrt(rr) / st->bnorm;
  st->it = it;
  st->rnorm = sqrt(rr);
  if (it - 1 < st->hist_cap) history[it - 1] = rel;  // solver.cpp:555
  if (!is_finite(rel)) {
    st->status = kStatusNonFinite;
    st->done = 1;
  } else if (rel <= st->rtol) {  // solver.cpp:557-560
    st->status = kStatusConverged;
    st->done = 1;
  } else if (it >= st->maxit) {
    st->status = kStatusMaxIt;
    st->done = 1;
  }
}

__device__ __forceinline__ void fin_post(PcgState* st, double rz, int init) {
  if (init) {
    st->rho = rz;  // solver.cpp:537
    st->beta = 0.0;
    st->first = 1;
  } else {
    st->beta = rz / st->rho;  // :562-564
    st->rho = rz;
  }
}

__device__ __forceinline__ void fin_jacobi(PcgState* st, double rr, double rz, int init,
                                           double* history) {
  if (init) {
    st->rho = rz;
    st->beta = 0.0;
    st->first = 1;
  } else {
    finish_rr(st, rr, history);
    if (!st->done) {
      st->beta = rz / st->rho;
      st->rho = rz;
    }
  }
}

}  // namespace tmg
