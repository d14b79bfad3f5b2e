// C-ABI implementation: context, set-up orchestration and the PCG driver.
// See include/topmg_b200.h for the reference interface each entry replaces.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/topmg_b200.h"
#include "kernels.h"

using namespace tmg;

namespace {
thread_local std::string g_create_error;

struct Fail {
  int code;
};
}  // namespace

struct tmg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  tmg_grid grid{};
  GridParams g{};
  int cb = 0;
  int64_t M = 0;
  std::string err;
  // problem
  double* kappa = nullptr;
  double* coef = nullptr;  // 4 x M operator coefficients (Tx+, Ty+, Tz+, diag)
  uint8_t* dmask = nullptr;
  bool have_problem = false;
  std::vector<Patch> patches;
  // preconditioner
  int kind = -1;
  bool have_setup = false;
  double* dinv = nullptr;
  double* phi = nullptr;
  double* evals = nullptr;
  int* eig_iters = nullptr;
  double* Gf = nullptr;
  double* Ac = nullptr;
  double* Bc = nullptr;
  double* Rcc = nullptr;
  double* cc_evals = nullptr;
  double* Winv = nullptr;
  double* Acc = nullptr;   // dense A_cc^-1 (set-up only)
  double* AccT = nullptr;  // its lower 64x64 tiles (per-cycle GEMV)
  double* symvP = nullptr; // GEMV partials
  int64_t n_cc = 0;
  // vectors
  double *b = nullptr, *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *z = nullptr,
         *r1 = nullptr, *stage = nullptr;
  double* pbuf[2] = {nullptr, nullptr};  // ping-pong search directions
  double *rc = nullptr, *rc0 = nullptr, *rcc = nullptr, *ecc = nullptr, *ec = nullptr,
         *rc1 = nullptr, *tc = nullptr;
  PcgState* st = nullptr;
  double* partials = nullptr;
  double* history = nullptr;
  int hist_cap = 0;
  int* d_status = nullptr;
  unsigned long long* d_count = nullptr;
  PcgState* h_state = nullptr;  // pinned, 2 slots
  // graph
  cudaGraphExec_t graph = nullptr;
  int graph_chunk = 0;
  int64_t graph_kernels = 0;  // kernel nodes in one captured chunk
  int64_t launches = 0;       // kernels enqueued by solves (incl. graph nodes)
  int64_t bytes = 0;
  std::vector<void*> allocs;
  // released buffers kept for reuse (re-setup with the same sizes allocates
  // nothing); byte size of every live or pooled buffer
  std::vector<std::pair<void*, size_t>> pool;
  std::unordered_map<void*, size_t> sizes;
  double setup_seconds = 0.0;
};

namespace {

int set_err(tmg_ctx* c, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  else g_create_error = buf;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      set_err(c, TMG_ECUDA, "CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__, \
              __LINE__, cudaGetErrorString(e_));                                          \
      throw Fail{TMG_ECUDA};                                                              \
    }                                                                                     \
  } while (0)

template <typename T>
T* dalloc(tmg_ctx* c, int64_t n) {
  void* p = nullptr;
  const size_t bytes = sizeof(T) * (size_t)std::max<int64_t>(n, 1);
  for (size_t i = 0; i < c->pool.size(); ++i)
    if (c->pool[i].second == bytes) {
      p = c->pool[i].first;
      c->pool.erase(c->pool.begin() + (std::ptrdiff_t)i);
      c->allocs.push_back(p);
      return (T*)p;
    }
  CK(cudaMalloc(&p, bytes));
  c->allocs.push_back(p);
  c->sizes[p] = bytes;
  c->bytes += (int64_t)bytes;
  return (T*)p;
}

// release to the context's pool (freed for real in tmg_destroy)
void dfree(tmg_ctx* c, void* p) {
  if (!p) return;
  auto it = std::find(c->allocs.begin(), c->allocs.end(), p);
  if (it == c->allocs.end()) return;
  c->allocs.erase(it);
  c->pool.emplace_back(p, c->sizes[p]);
}

void free_setup(tmg_ctx* c) {
  for (void** pp : {(void**)&c->dinv, (void**)&c->phi, (void**)&c->evals, (void**)&c->eig_iters,
                    (void**)&c->Gf, (void**)&c->Ac, (void**)&c->Bc, (void**)&c->Rcc,
                    (void**)&c->cc_evals, (void**)&c->Winv, (void**)&c->Acc, (void**)&c->AccT, (void**)&c->symvP, (void**)&c->rc,
                    (void**)&c->rc0, (void**)&c->rcc, (void**)&c->ecc, (void**)&c->ec,
                    (void**)&c->rc1, (void**)&c->tc}) {
    dfree(c, *pp);
    *pp = nullptr;
  }
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  c->have_setup = false;
  c->kind = -1;
}

int guard(tmg_ctx* c, const std::function<void()>& fn) {
  try {
    fn();
    return TMG_OK;
  } catch (const Fail& f) {
    return f.code;
  } catch (const std::exception& e) {
    return set_err(c, TMG_ECUDA, "internal error: %s", e.what());
  }
}

int validate_patches(tmg_ctx* c, const tmg_patch* p, int np) {
  // BoundarySpec::validate (grid.cpp:77-93)
  if (np < 0 || (np > 0 && !p)) return set_err(c, TMG_EARG, "patches: bad pointer/count");
  if (np > kMaxPatches) return set_err(c, TMG_ENOTSUP, "at most %d Dirichlet patches", kMaxPatches);
  for (int a = 0; a < np; ++a) {
    if (p[a].face < 0 || p[a].face > 5) return set_err(c, TMG_ECONFIG, "BoundarySpec: bad face");
    if (p[a].u1 < p[a].u0 || p[a].v1 < p[a].v0)
      return set_err(c, TMG_ECONFIG, "BoundarySpec: patch with negative extent");
    double lu, lv;
    if (p[a].face <= 1) { lu = c->grid.ly; lv = c->grid.lz; }
    else if (p[a].face <= 3) { lu = c->grid.lx; lv = c->grid.lz; }
    else { lu = c->grid.lx; lv = c->grid.ly; }
    if (p[a].u0 < 0.0 || p[a].v0 < 0.0 || p[a].u1 > lu || p[a].v1 > lv)
      return set_err(c, TMG_ECONFIG, "BoundarySpec: patch outside the domain face");
    for (int b = a + 1; b < np; ++b) {
      if (p[a].face != p[b].face) continue;
      if (p[a].u0 < p[b].u1 && p[b].u0 < p[a].u1 && p[a].v0 < p[b].v1 && p[b].v0 < p[a].v1)
        return set_err(c, TMG_ECONFIG, "BoundarySpec: overlapping patches");
    }
  }
  return TMG_OK;
}

// device kappa (brick layout) is in c->kappa; build mask, count faces
int finish_problem(tmg_ctx* c) {
  return guard(c, [&] {
    CK(cudaMemsetAsync(c->d_count, 0, sizeof(unsigned long long), c->stream));
    launch_boundary(c->g, c->cb, c->patches.data(), (int)c->patches.size(), c->grid.lx, c->grid.ly,
                    c->grid.lz, c->kappa, nullptr, c->dmask, nullptr, c->d_count, c->stream);
    CK(cudaGetLastError());
    unsigned long long cnt = 0;
    CK(cudaMemcpyAsync(&cnt, c->d_count, sizeof cnt, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (cnt == 0) {
      set_err(c, TMG_ECONFIG,
              "assemble_system: no Dirichlet face on the boundary, the system would be singular");
      throw Fail{TMG_ECONFIG};
    }
    launch_coefficients(c->g, c->cb, c->kappa, c->dmask, c->coef, c->stream);
    CK(cudaGetLastError());
    c->have_problem = true;
    free_setup(c);
  });
}

void upload_global(tmg_ctx* c, const double* host, double* dev_brick) {
  CK(cudaMemcpyAsync(c->stage, host, sizeof(double) * (size_t)c->M, cudaMemcpyHostToDevice,
                     c->stream));
  launch_to_brick(c->g, c->cb, c->stage, dev_brick, c->stream);
  CK(cudaGetLastError());
}

void download_global(tmg_ctx* c, const double* dev_brick, double* host) {
  launch_from_brick(c->g, c->cb, dev_brick, c->stage, c->stream);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(host, c->stage, sizeof(double) * (size_t)c->M, cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

// ---------------------------------------------------------------- V-cycle
void enqueue_vcycle(tmg_ctx* c, int init, PcgState* st, cudaStream_t s, const double* p) {
  const GridParams& g = c->g;
  launch_update(g, c->cb, c->coef, c->Gf, c->x, p, c->q, c->r, c->r1, st, c->partials,
                c->history, init, s);
  launch_restrict(g, c->cb, c->coef, c->phi, c->r, c->r1, c->rc, st, s);
  launch_coarse_cycle(g, &st->done, c->Ac, c->Winv, c->Rcc, c->AccT, c->symvP, c->n_cc, c->rc, c->rc0,
                      c->rcc, c->ecc, c->rc1, c->tc, c->ec, s);
  launch_post(g, c->cb, c->coef, c->phi, c->Gf, c->r, c->r1, c->ec, c->z, st,
              c->partials, init, s);
}

// Iteration with parity `par`: reads p from pbuf[par], writes pbuf[par ^ 1].
void enqueue_iteration(tmg_ctx* c, cudaStream_t s, int par) {
  const double* pold = c->pbuf[par];
  double* pnew = c->pbuf[par ^ 1];
  launch_search(c->g, c->cb, c->coef, c->z, pold, pnew, c->q, c->st, c->partials, s);
  if (c->kind == TMG_PRECOND_MMG) {
    enqueue_vcycle(c, 0, c->st, s, pnew);
  } else {
    launch_jacobi_step(c->g, c->cb, c->kind == TMG_PRECOND_JACOBI ? c->dinv : nullptr, c->x, pnew,
                       c->q, c->r, c->z, c->st, c->partials, c->history, 0, s);
  }
}

void build_graph(tmg_ctx* c, int chunk) {
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  // chunk is even so every graph launch starts from pbuf[0]
  for (int i = 0; i < chunk; ++i) enqueue_iteration(c, c->stream, i & 1);
  CK(cudaStreamEndCapture(c->stream, &graph));
  size_t nodes = 0;
  CK(cudaGraphGetNodes(graph, nullptr, &nodes));
  c->graph_kernels = (int64_t)nodes;
  CK(cudaGraphInstantiate(&c->graph, graph, 0));
  cudaGraphDestroy(graph);
  c->graph_chunk = chunk;
}

void ensure_history(tmg_ctx* c, int maxit) {
  if (maxit <= c->hist_cap) return;
  dfree(c, c->history);
  c->history = dalloc<double>(c, maxit);
  c->hist_cap = maxit;
  // the captured graph holds the history pointer
  if (c->graph) build_graph(c, c->graph_chunk);
}

// Runs the device solve on resident c->b (and c->x if use_x0).
void solve_device(tmg_ctx* c, double rtol, int maxit, int use_x0, tmg_report* rep,
                  double* ms_total, int* counts) {
  if (!c->have_setup) {
    set_err(c, TMG_EARG, "pcg: no preconditioner set up (call tmg_setup)");
    throw Fail{TMG_EARG};
  }
  ensure_history(c, std::max(maxit, 1));
  PcgState init{};
  init.rtol = rtol;
  init.maxit = maxit;
  init.hist_cap = c->hist_cap;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, c->stream));
  CK(cudaMemcpyAsync(c->st, &init, sizeof init, cudaMemcpyHostToDevice, c->stream));
  const bool prof = ms_total != nullptr;
  std::vector<cudaEvent_t> evs;
  auto timed = [&](int slot, const std::function<void()>& launch) {
    if (!prof) {
      launch();
      return;
    }
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, c->stream));
    launch();
    CK(cudaEventRecord(b, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    ms_total[slot] += ms;
    counts[slot] += 1;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  };
  timed(8, [&] {
    launch_init(c->g, c->cb, c->coef, c->b, c->x, use_x0, c->r, c->st, c->partials,
                c->stream);
  });
  c->launches += 1;                                          // init
  c->launches += c->kind == TMG_PRECOND_MMG ? c->graph_kernels / c->graph_chunk - 1 : 1;
  if (c->kind == TMG_PRECOND_MMG) {
    if (!prof) {
      enqueue_vcycle(c, 1, c->st, c->stream, c->pbuf[0]);
    } else {
      timed(1, [&] { launch_update(c->g, c->cb, c->coef, c->Gf, c->x, c->p, c->q, c->r, c->r1, c->st, c->partials, c->history, 1, c->stream); });
      timed(2, [&] { launch_restrict(c->g, c->cb, c->coef, c->phi, c->r, c->r1, c->rc, c->st, c->stream); });
      timed(3, [&] { launch_coarse_cycle(c->g, &c->st->done, c->Ac, c->Winv, c->Rcc, c->AccT, c->symvP, c->n_cc, c->rc, c->rc0, c->rcc, c->ecc, c->rc1, c->tc, c->ec, c->stream); });
      timed(6, [&] { launch_post(c->g, c->cb, c->coef, c->phi, c->Gf, c->r, c->r1, c->ec, c->z, c->st, c->partials, 1, c->stream); });
    }
  } else {
    timed(7, [&] {
      launch_jacobi_step(c->g, c->cb, c->kind == TMG_PRECOND_JACOBI ? c->dinv : nullptr, c->x,
                         c->p, c->q, c->r, c->z, c->st, c->partials, c->history, 1, c->stream);
    });
  }
  CK(cudaGetLastError());
  PcgState* hs = c->h_state;
  if (!prof) {
    // chunked graph launches; the next chunk is enqueued before the previous
    // one's state is polled, so the GPU never idles on the host.
    CK(cudaMemcpyAsync(&hs[0], c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (!hs[0].done && maxit > 0) {
      cudaEvent_t ev[2];
      CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
      int launched = 0;
      auto launch_chunk = [&](int sl) {
        CK(cudaGraphLaunch(c->graph, c->stream));
        c->launches += c->graph_kernels;
        CK(cudaMemcpyAsync(&hs[sl], c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaEventRecord(ev[sl], c->stream));
        launched += c->graph_chunk;
      };
      int cur = 0;
      launch_chunk(cur);
      while (true) {
        const bool more = launched < maxit;
        if (more) launch_chunk(cur ^ 1);
        CK(cudaEventSynchronize(ev[cur]));
        if (hs[cur].done || !more) break;
        cur ^= 1;
      }
      CK(cudaStreamSynchronize(c->stream));
      cudaEventDestroy(ev[0]);
      cudaEventDestroy(ev[1]);
    }
  } else {
    CK(cudaMemcpy(&hs[0], c->st, sizeof(PcgState), cudaMemcpyDeviceToHost));
    int guard_it = 0, par = 0;
    while (!hs[0].done && maxit > 0 && guard_it++ <= maxit) {
      const double* pold = c->pbuf[par];
      double* pnew = c->pbuf[par ^ 1];
      par ^= 1;
      timed(0, [&] { launch_search(c->g, c->cb, c->coef, c->z, pold, pnew, c->q, c->st, c->partials, c->stream); });
      if (c->kind == TMG_PRECOND_MMG) {
        timed(1, [&] { launch_update(c->g, c->cb, c->coef, c->Gf, c->x, pnew, c->q, c->r, c->r1, c->st, c->partials, c->history, 0, c->stream); });
        timed(2, [&] { launch_restrict(c->g, c->cb, c->coef, c->phi, c->r, c->r1, c->rc, c->st, c->stream); });
        timed(3, [&] { launch_coarse_cycle(c->g, &c->st->done, c->Ac, c->Winv, c->Rcc, c->AccT, c->symvP, c->n_cc, c->rc, c->rc0, c->rcc, c->ecc, c->rc1, c->tc, c->ec, c->stream); });
        timed(6, [&] { launch_post(c->g, c->cb, c->coef, c->phi, c->Gf, c->r, c->r1, c->ec, c->z, c->st, c->partials, 0, c->stream); });
      } else {
        timed(7, [&] {
          launch_jacobi_step(c->g, c->cb, c->kind == TMG_PRECOND_JACOBI ? c->dinv : nullptr,
                             c->x, pnew, c->q, c->r, c->z, c->st, c->partials, c->history, 0,
                             c->stream);
        });
      }
      CK(cudaMemcpy(&hs[0], c->st, sizeof(PcgState), cudaMemcpyDeviceToHost));
    }
  }
  CK(cudaEventRecord(e1, c->stream));
  CK(cudaMemcpyAsync(&hs[0], c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaGetLastError());
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  PcgState& f = hs[0];
  if (!f.done && maxit == 0) f.status = kStatusMaxIt;
  if (f.status == kStatusZeroRhs) {
    CK(cudaMemsetAsync(c->x, 0, sizeof(double) * (size_t)c->M, c->stream));  // solver.cpp:506-513
  }
  if (rep) {
    rep->iterations = f.it;
    rep->converged = (f.status == kStatusConverged || f.status == kStatusZeroRhs) ? 1 : 0;
    rep->status = f.status;
    rep->solve_seconds = 1e-3 * ms;
    rep->setup_seconds = c->setup_seconds;
    rep->final_relative_residual = f.bnorm > 0 ? f.rnorm / f.bnorm : 0.0;
  }
  if (f.status == kStatusIndefinite) {
    set_err(c, TMG_ESOLVER,
            "pcg: operator or preconditioner not positive definite (p^T A p = %g at iteration %d)",
            f.pq, f.it + 1);
    throw Fail{TMG_ESOLVER};
  }
  if (f.status == kStatusNonFinite) {
    set_err(c, TMG_ESOLVER, "pcg: non-finite residual at iteration %d", f.it);
    throw Fail{TMG_ESOLVER};
  }
}

}  // namespace

// =================================================================== C ABI

extern "C" {

const char* tmg_last_error(const tmg_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

int tmg_create(const tmg_grid* grid, int device, tmg_ctx** out) {
  if (!grid || !out) return set_err(nullptr, TMG_EARG, "tmg_create: null argument");
  *out = nullptr;
  const tmg_grid& G = *grid;
  if (G.nx <= 0 || G.ny <= 0 || G.nz <= 0)
    return set_err(nullptr, TMG_ECONFIG, "GridSpec: cell counts must be positive");
  if (G.lx <= 0 || G.ly <= 0 || G.lz <= 0)
    return set_err(nullptr, TMG_ECONFIG, "GridSpec: domain extents must be positive");
  if (G.ncc[0] <= 0 || G.ncc[1] <= 0 || G.ncc[2] <= 0 || G.sd <= 0)
    return set_err(nullptr, TMG_ECONFIG, "build_hierarchy: ncc and sd must be positive");
  const int64_t n[3] = {G.nx, G.ny, G.nz};
  int64_t cpc[3];
  for (int a = 0; a < 3; ++a) {
    const int64_t div = G.ncc[a] * G.sd;
    if (n[a] % div != 0)
      return set_err(nullptr, TMG_ECONFIG,
                     "build_hierarchy: axis %d has %lld cells, not divisible by ncc*sd = %lld*%lld "
                     "= %lld",
                     a, (long long)n[a], (long long)G.ncc[a], (long long)G.sd, (long long)div);
    cpc[a] = n[a] / div;
  }
  if (cpc[0] != cpc[1] || cpc[1] != cpc[2] || !(cpc[0] == 4 || cpc[0] == 8))
    return set_err(nullptr, TMG_ENOTSUP,
                   "GPU path builds cubic coarse cells of 4^3 or 8^3 fine cells (got %lldx%lldx%lld)",
                   (long long)cpc[0], (long long)cpc[1], (long long)cpc[2]);
  tmg_ctx* c = new tmg_ctx;
  c->grid = G;
  c->device = device;
  c->cb = (int)cpc[0];
  c->M = G.nx * G.ny * G.nz;
  GridParams& g = c->g;
  g.nx = G.nx; g.ny = G.ny; g.nz = G.nz;
  g.nbx = G.nx / c->cb; g.nby = G.ny / c->cb; g.nbz = G.nz / c->cb;
  g.nb = g.nbx * g.nby * g.nbz;
  g.ncx = G.ncc[0]; g.ncy = G.ncc[1]; g.ncz = G.ncc[2];
  g.ncc = g.ncx * g.ncy * g.ncz;
  g.sd = (int)G.sd;
  g.hx = G.lx / (double)G.nx;
  g.hy = G.ly / (double)G.ny;
  g.hz = G.lz / (double)G.nz;
  g.cpl[0] = g.hy * g.hz / g.hx;  // fvm.cpp:23-26
  g.cpl[1] = g.hx * g.hz / g.hy;
  g.cpl[2] = g.hx * g.hy / g.hz;
  g.vol = g.hx * g.hy * g.hz;
  g.lc = 4;
  g.lcc = 8;
  g.b0 = 0;
  g.nbo = g.nb;
  g.e0 = 0;
  g.neo = g.ncc;
  g.mst = c->M;
  g.dist = 0;
  const int rc = guard(c, [&] {
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    init_kernel_attributes();
    c->kappa = dalloc<double>(c, c->M);
    c->dmask = dalloc<uint8_t>(c, c->M);
    c->coef = dalloc<double>(c, 4 * c->M);
    for (double** v : {&c->b, &c->x, &c->r, &c->p, &c->q, &c->z, &c->r1, &c->stage})
      *v = dalloc<double>(c, c->M);
    c->pbuf[0] = c->p;
    c->pbuf[1] = dalloc<double>(c, c->M);
    c->st = dalloc<PcgState>(c, 1);
    c->partials = dalloc<double>(c, 4 * g.nb + 64);
    c->d_status = dalloc<int>(c, 4);
    c->d_count = dalloc<unsigned long long>(c, 1);
    CK(cudaMemset(c->st, 0, sizeof(PcgState)));
    CK(cudaMallocHost(&c->h_state, 2 * sizeof(PcgState)));
  });
  if (rc) {
    g_create_error = c->err;
    tmg_destroy(c);
    return rc;
  }
  *out = c;
  return TMG_OK;
}

void tmg_destroy(tmg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  for (void* p : c->allocs) cudaFree(p);
  for (auto& pb : c->pool) cudaFree(pb.first);
  if (c->h_state) cudaFreeHost(c->h_state);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int tmg_set_conductivity(tmg_ctx* c, const double* kappa, const tmg_patch* patches, int np) {
  if (!c || !kappa) return set_err(c, TMG_EARG, "tmg_set_conductivity: null argument");
  for (int64_t i = 0; i < c->M; ++i)
    if (!(kappa[i] > 0.0))  // fvm.cpp:42-44
      return set_err(c, TMG_ECONFIG, "assemble_system: conductivity must be positive");
  int rc = validate_patches(c, patches, np);
  if (rc) return rc;
  c->patches.clear();
  for (int i = 0; i < np; ++i)
    c->patches.push_back(Patch{patches[i].face, patches[i].u0, patches[i].v0, patches[i].u1,
                               patches[i].v1, patches[i].value});
  rc = guard(c, [&] {
    CK(cudaSetDevice(c->device));
    upload_global(c, kappa, c->kappa);
  });
  if (rc) return rc;
  return finish_problem(c);
}

int tmg_set_design(tmg_ctx* c, const double* rho, double lo, double hi, int p,
                   const tmg_patch* patches, int np) {
  if (!c || !rho) return set_err(c, TMG_EARG, "tmg_set_design: null argument");
  if (!(lo > 0.0) || !(hi > lo))  // material.cpp:11-12
    return set_err(c, TMG_ECONFIG, "MaterialModel: requires 0 < kappa_lo < kappa_hi");
  if (p < 1) return set_err(c, TMG_ECONFIG, "MaterialModel: penalization p must be >= 1");
  for (int64_t i = 0; i < c->M; ++i) {
    double r = 1.0;
    for (int k = 0; k < p; ++k) r *= rho[i];
    if (!(lo + r * (hi - lo) > 0.0))
      return set_err(c, TMG_ECONFIG, "assemble_system: conductivity must be positive");
  }
  int rc = validate_patches(c, patches, np);
  if (rc) return rc;
  c->patches.clear();
  for (int i = 0; i < np; ++i)
    c->patches.push_back(Patch{patches[i].face, patches[i].u0, patches[i].v0, patches[i].u1,
                               patches[i].v1, patches[i].value});
  rc = guard(c, [&] {
    CK(cudaSetDevice(c->device));
    upload_global(c, rho, c->r);  // r as scratch for rho (brick layout)
    launch_conductivity(c->g, c->cb, c->r, c->kappa, lo, hi, p, c->stream);
    CK(cudaGetLastError());
  });
  if (rc) return rc;
  return finish_problem(c);
}

int tmg_assemble_rhs(tmg_ctx* c, const double* source, double* rhs_out) {
  if (!c || !rhs_out) return set_err(c, TMG_EARG, "tmg_assemble_rhs: null argument");
  if (!c->have_problem) return set_err(c, TMG_EARG, "tmg_assemble_rhs: no problem set");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    double* src = nullptr;
    if (source) {
      upload_global(c, source, c->q);
      src = c->q;
    }
    launch_boundary(c->g, c->cb, c->patches.data(), (int)c->patches.size(), c->grid.lx,
                    c->grid.ly, c->grid.lz, c->kappa, src, c->dmask, c->z, nullptr, c->stream);
    CK(cudaGetLastError());
    download_global(c, c->z, rhs_out);
  });
}

int tmg_setup(tmg_ctx* c, const tmg_mmg_options* o) {
  if (!c || !o) return set_err(c, TMG_EARG, "tmg_setup: null argument");
  if (!c->have_problem) return set_err(c, TMG_EARG, "tmg_setup: no problem set");
  const int kind = o->kind;
  if (kind == TMG_PRECOND_BLOCK_JACOBI || kind == TMG_PRECOND_TWO_GRID)
    return set_err(c, TMG_ENOTSUP, "preconditioner kind %d is not built on the GPU path", kind);
  if (kind < 0 || kind > 4) return set_err(c, TMG_ECONFIG, "make_preconditioner: unknown kind");
  if (kind == TMG_PRECOND_MMG) {
    const int64_t cells = (int64_t)c->cb * c->cb * c->cb;
    if (o->num_local_basis > cells)
      return set_err(c, TMG_EARG, "local_spectral_basis: more eigenvectors than cells requested");
    if (o->num_local_basis != compiled_lc())
      return set_err(c, TMG_ENOTSUP, "GPU path is compiled for L_c = %d (got %lld)", compiled_lc(),
                     (long long)o->num_local_basis);
    const int64_t q = (int64_t)c->g.sd * c->g.sd * c->g.sd * o->num_local_basis;
    if (o->num_cc_basis > q)
      return set_err(c, TMG_EARG,
                     "coarse_coarse_basis: more eigenvectors than coarse basis functions");
    if (o->num_cc_basis < 1) return set_err(c, TMG_EARG, "num_cc_basis must be >= 1");
    if (q > 64)
      return set_err(c, TMG_ENOTSUP, "GPU coarse-coarse eigensolver handles sd^3*L_c <= 64 (got %lld)",
                     (long long)q);
    if (o->smoother_sweeps != 1)
      return set_err(c, TMG_ENOTSUP, "GPU smoother is built for smoother_sweeps = 1");
  }
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    free_setup(c);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, c->stream));
    GridParams& g = c->g;
    CK(cudaMemsetAsync(c->d_status, 0, 4 * sizeof(int), c->stream));
    if (kind == TMG_PRECOND_JACOBI) {
      c->dinv = dalloc<double>(c, c->M);
      launch_apply(g, c->cb, c->coef, nullptr, nullptr, c->dinv, c->stream);
    } else if (kind == TMG_PRECOND_MMG) {
      g.lc = (int)o->num_local_basis;
      g.lcc = (int)o->num_cc_basis;
      const int64_t C = (int64_t)c->cb * c->cb * c->cb;
      const int64_t q = (int64_t)g.sd * g.sd * g.sd * g.lc;
      c->phi = dalloc<double>(c, g.nb * g.lc * C);
      c->evals = dalloc<double>(c, g.nb * g.lc);
      c->eig_iters = dalloc<int>(c, g.nb);
      c->Gf = dalloc<double>(c, g.nb * thomas_doubles_per_brick(c->cb));
      c->Ac = dalloc<double>(c, g.nb * 7 * g.lc * g.lc);
      c->Bc = dalloc<double>(c, g.nb * g.lc * g.lc);
      c->Rcc = dalloc<double>(c, g.ncc * g.lcc * q);
      c->cc_evals = dalloc<double>(c, g.ncc * g.lcc);
      c->Winv = dalloc<double>(c, g.ncc * q * q);
      c->n_cc = g.ncc * g.lcc;
      c->Acc = dalloc<double>(c, c->n_cc * c->n_cc);
      c->rc = dalloc<double>(c, g.nb * g.lc);
      c->rc0 = dalloc<double>(c, g.nb * g.lc);
      c->ec = dalloc<double>(c, g.nb * g.lc);
      c->rc1 = dalloc<double>(c, g.nb * g.lc);
      c->tc = dalloc<double>(c, g.nb * g.lc);
      c->rcc = dalloc<double>(c, c->n_cc);
      c->ecc = dalloc<double>(c, c->n_cc);
      // TMG_SETUP_PROFILE=1: per-phase device times on stderr (diagnostics only)
      const bool sprof = getenv("TMG_SETUP_PROFILE") != nullptr;
      cudaEvent_t ph[10];
      int nph = 0;
      const char* phname[10];
      auto mark = [&](const char* name) {
        if (!sprof) return;
        CK(cudaEventCreate(&ph[nph]));
        CK(cudaEventRecord(ph[nph], c->stream));
        phname[nph++] = name;
      };
      mark("alloc");
      const double tol = o->eig_tol > 0 ? o->eig_tol : 1e-11;
      const int degree = o->eig_degree > 0 ? o->eig_degree : 32;
      const int max_outer = o->eig_max_outer > 0 ? o->eig_max_outer : 60;
      launch_local_basis(g, c->cb, c->kappa, c->phi, c->evals, c->eig_iters, tol, degree, max_outer,
                         c->stream);
      CK(cudaGetLastError());
      mark("local_basis");
      launch_coarse_blocks(g, c->cb, c->kappa, c->dmask, c->phi, c->Ac, c->Bc, c->stream);
      CK(cudaGetLastError());
      mark("coarse_blocks");
      launch_cc_basis(g, c->Ac, c->Bc, c->Rcc, c->cc_evals, c->stream);
      CK(cudaGetLastError());
      mark("cc_basis");
      launch_coarse_smoother(g, c->Ac, c->Winv, c->d_status + 1, c->stream);
      CK(cudaGetLastError());
      mark("coarse_smoother");
      launch_thomas_factor(g, c->cb, c->kappa, c->dmask, c->Gf, c->d_status, c->stream);
      CK(cudaGetLastError());
      mark("thomas_factor");
      launch_acc_assemble(g, c->Ac, c->Rcc, c->Acc, c->stream);
      CK(cudaGetLastError());
      mark("acc_assemble");
      double* work = dalloc<double>(c, dense_inverse_work_doubles(c->n_cc));
      dense_spd_inverse(c->Acc, c->n_cc, work, c->d_status + 2, c->stream);
      CK(cudaGetLastError());
      mark("acc_inverse");
      c->AccT = dalloc<double>(c, sym_tiles_doubles(c->n_cc));
      c->symvP = dalloc<double>(c, sym_partials_doubles(c->n_cc));
      pack_sym_tiles(c->Acc, c->n_cc, c->AccT, c->stream);
      CK(cudaGetLastError());
      mark("pack_tiles");
      CK(cudaStreamSynchronize(c->stream));
      for (int i = 1; i < nph; ++i) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, ph[i - 1], ph[i]));
        fprintf(stderr, "[setup] %-16s %9.3f ms\n", phname[i], t);
      }
      for (int i = 0; i < nph; ++i) cudaEventDestroy(ph[i]);
      dfree(c, work);
      dfree(c, c->Acc);
      c->Acc = nullptr;
    }
    CK(cudaEventRecord(e1, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaGetLastError());
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    c->setup_seconds = 1e-3 * ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    int status[4];
    CK(cudaMemcpy(status, c->d_status, sizeof status, cudaMemcpyDeviceToHost));
    if (status[0]) {
      set_err(c, TMG_ESOLVER,
              "BlockJacobiSmoother: singular block: DirectSolver: matrix numerically singular");
      throw Fail{TMG_ESOLVER};
    }
    if (status[1]) {
      set_err(c, TMG_ESOLVER, "BlockJacobiSmoother: singular block (coarse level)");
      throw Fail{TMG_ESOLVER};
    }
    if (status[2]) {
      set_err(c, TMG_ESOLVER, "DirectSolver: matrix numerically singular (A_cc)");
      throw Fail{TMG_ESOLVER};
    }
    c->kind = kind;
    c->have_setup = true;
    build_graph(c, 4);
  });
}

int tmg_upload_rhs(tmg_ctx* c, const double* b) {
  if (!c || !b) return set_err(c, TMG_EARG, "tmg_upload_rhs: null argument");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    upload_global(c, b, c->b);
  });
}

int tmg_upload_x0(tmg_ctx* c, const double* x0) {
  if (!c || !x0) return set_err(c, TMG_EARG, "tmg_upload_x0: null argument");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    upload_global(c, x0, c->x);
  });
}

int tmg_solve_resident(tmg_ctx* c, double rtol, int maxit, int use_x0, tmg_report* rep) {
  if (!c) return set_err(c, TMG_EARG, "null context");
  if (maxit < 0) return set_err(c, TMG_EARG, "pcg: negative max_iterations");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    solve_device(c, rtol, maxit, use_x0, rep, nullptr, nullptr);
  });
}

int tmg_download_solution(tmg_ctx* c, double* x) {
  if (!c || !x) return set_err(c, TMG_EARG, "tmg_download_solution: null argument");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    download_global(c, c->x, x);
  });
}

int tmg_pcg(tmg_ctx* c, const double* b, const double* x0, double rtol, int maxit, double* x_out,
            double* history, tmg_report* rep) {
  if (!c || !b || !x_out) return set_err(c, TMG_EARG, "pcg: null argument");
  if (maxit < 0) return set_err(c, TMG_EARG, "pcg: negative max_iterations");
  tmg_report local{};
  const int rc = guard(c, [&] {
    CK(cudaSetDevice(c->device));
    upload_global(c, b, c->b);
    if (x0) upload_global(c, x0, c->x);
    solve_device(c, rtol, maxit, x0 ? 1 : 0, &local, nullptr, nullptr);
    download_global(c, c->x, x_out);
    if (history && local.iterations > 0)
      CK(cudaMemcpy(history, c->history, sizeof(double) * (size_t)local.iterations,
                    cudaMemcpyDeviceToHost));
  });
  if (rep) *rep = local;
  return rc;
}

int tmg_apply_operator(tmg_ctx* c, const double* x, double* y) {
  if (!c || !x || !y) return set_err(c, TMG_EARG, "SparseOperator::apply: null argument");
  if (!c->have_problem) return set_err(c, TMG_EARG, "apply: no problem set");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    upload_global(c, x, c->p);
    launch_apply(c->g, c->cb, c->coef, c->p, c->q, nullptr, c->stream);
    CK(cudaGetLastError());
    download_global(c, c->q, y);
  });
}

int tmg_apply_preconditioner(tmg_ctx* c, const double* rin, double* zout) {
  if (!c || !rin || !zout) return set_err(c, TMG_EARG, "Preconditioner::apply: null argument");
  if (!c->have_setup) return set_err(c, TMG_EARG, "apply: no preconditioner set up");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    ensure_history(c, 1);
    PcgState init{};
    init.rtol = 0.0;
    init.maxit = 1;
    init.hist_cap = c->hist_cap;
    CK(cudaMemcpyAsync(c->st, &init, sizeof init, cudaMemcpyHostToDevice, c->stream));
    upload_global(c, rin, c->r);
    if (c->kind == TMG_PRECOND_MMG) {
      enqueue_vcycle(c, 1, c->st, c->stream, c->p);
    } else {
      launch_jacobi_step(c->g, c->cb, c->kind == TMG_PRECOND_JACOBI ? c->dinv : nullptr, c->x,
                         c->p, c->q, c->r, c->z, c->st, c->partials, c->history, 1, c->stream);
    }
    CK(cudaGetLastError());
    download_global(c, c->z, zout);
  });
}

int tmg_get_sizes(tmg_ctx* c, int64_t* s) {
  if (!c || !s) return set_err(c, TMG_EARG, "null argument");
  const int64_t C = (int64_t)c->cb * c->cb * c->cb;
  s[0] = c->M;
  s[1] = c->g.nb;
  s[2] = c->g.nb * c->g.lc;
  s[3] = c->g.ncc;
  s[4] = c->g.ncc * c->g.lcc;
  s[5] = C;
  return TMG_OK;
}

int tmg_get_local_bases(tmg_ctx* c, double* phi, double* evals, int* iters) {
  if (!c || !c->have_setup || c->kind != TMG_PRECOND_MMG)
    return set_err(c, TMG_EARG, "no MMG hierarchy set up");
  return guard(c, [&] {
    const int64_t C = (int64_t)c->cb * c->cb * c->cb;
    if (phi)
      CK(cudaMemcpy(phi, c->phi, sizeof(double) * (size_t)(c->g.nb * c->g.lc * C),
                    cudaMemcpyDeviceToHost));
    if (evals)
      CK(cudaMemcpy(evals, c->evals, sizeof(double) * (size_t)(c->g.nb * c->g.lc),
                    cudaMemcpyDeviceToHost));
    if (iters)
      CK(cudaMemcpy(iters, c->eig_iters, sizeof(int) * (size_t)c->g.nb, cudaMemcpyDeviceToHost));
  });
}

int tmg_get_coarse_operator(tmg_ctx* c, double* ac) {
  if (!c || !c->have_setup || c->kind != TMG_PRECOND_MMG || !ac)
    return set_err(c, TMG_EARG, "no MMG hierarchy set up");
  return guard(c, [&] {
    const GridParams& g = c->g;
    const int L = g.lc;
    std::vector<double> blk((size_t)(g.nb * 7 * L * L));
    CK(cudaMemcpy(blk.data(), c->Ac, sizeof(double) * blk.size(), cudaMemcpyDeviceToHost));
    const int64_t nc = g.nb * L;
    std::fill(ac, ac + nc * nc, 0.0);
    for (int64_t I = 0; I < g.nb; ++I) {
      const int64_t bi = I % g.nbx, bj = (I / g.nbx) % g.nby, bk = I / (g.nbx * g.nby);
      const int64_t nbr[7] = {I,
                              bi > 0 ? I - 1 : -1,
                              bi + 1 < g.nbx ? I + 1 : -1,
                              bj > 0 ? I - g.nbx : -1,
                              bj + 1 < g.nby ? I + g.nbx : -1,
                              bk > 0 ? I - g.nbx * g.nby : -1,
                              bk + 1 < g.nbz ? I + g.nbx * g.nby : -1};
      for (int d = 0; d < 7; ++d) {
        if (nbr[d] < 0) continue;
        for (int a = 0; a < L; ++a)
          for (int b = 0; b < L; ++b)
            ac[(I * L + a) * nc + nbr[d] * L + b] = blk[(size_t)((I * 7 + d) * L * L + a * L + b)];
      }
    }
  });
}

int tmg_get_cc_restriction(tmg_ctx* c, double* rcc) {
  if (!c || !c->have_setup || c->kind != TMG_PRECOND_MMG || !rcc)
    return set_err(c, TMG_EARG, "no MMG hierarchy set up");
  return guard(c, [&] {
    const GridParams& g = c->g;
    const int64_t q = (int64_t)g.sd * g.sd * g.sd * g.lc, nc = g.nb * g.lc;
    std::vector<double> R((size_t)(g.ncc * g.lcc * q));
    CK(cudaMemcpy(R.data(), c->Rcc, sizeof(double) * R.size(), cudaMemcpyDeviceToHost));
    std::fill(rcc, rcc + g.ncc * g.lcc * nc, 0.0);
    for (int64_t e = 0; e < g.ncc; ++e) {
      const int64_t ei = e % g.ncx, ej = (e / g.ncx) % g.ncy, ek = e / (g.ncx * g.ncy);
      for (int64_t ch = 0; ch < (int64_t)g.sd * g.sd * g.sd; ++ch) {
        const int64_t di = ch % g.sd, dj = (ch / g.sd) % g.sd, dk = ch / (g.sd * g.sd);
        const int64_t I = (ei * g.sd + di) + g.nbx * ((ej * g.sd + dj) + g.nby * (ek * g.sd + dk));
        for (int k = 0; k < g.lcc; ++k)
          for (int a = 0; a < g.lc; ++a)
            rcc[(e * g.lcc + k) * nc + I * g.lc + a] = R[(size_t)((e * g.lcc + k) * q + ch * g.lc + a)];
      }
    }
  });
}

int tmg_profile_solve(tmg_ctx* c, double rtol, int maxit, double* ms_total, int* count) {
  if (!c || !ms_total || !count) return set_err(c, TMG_EARG, "null argument");
  for (int i = 0; i < 9; ++i) {
    ms_total[i] = 0.0;
    count[i] = 0;
  }
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    tmg_report rep{};
    solve_device(c, rtol, maxit, 0, &rep, ms_total, count);
  });
}

int64_t tmg_device_bytes(const tmg_ctx* c) { return c ? c->bytes : 0; }

int64_t tmg_kernel_launches(const tmg_ctx* c) { return c ? c->launches : 0; }

void* tmg_stream(tmg_ctx* c) { return c ? (void*)c->stream : nullptr; }

}  // extern "C"
