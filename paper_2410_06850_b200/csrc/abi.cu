// C-ABI implementation: context, set-up orchestration and the PCG driver.
// See include/topmg_b200.h for the reference interface each entry replaces.
//
// A context holds one or more z-slabs of the grid:
//  * tmg_create            one slab = the whole grid (single GPU);
//  * tmg_create_slabs      S slabs in this process on one GPU (the partitioned
//                          path with in-process ghost copies — how the
//                          multi-GPU data path is exercised on one device);
//  * tmg_create_dist       one slab per process/GPU, ghosts and reductions
//                          over NCCL (NVLink/NVSwitch).
// A slab owns whole z-layers of cc elements. Its device arrays are windows of
// the global brick-layout arrays: the own bricks plus one ghost brick layer
// per neighbouring slab, addressed through "virtual global" base pointers so
// the kernels index global bricks unchanged. Ghost layers are contiguous
// (bricks are z-slowest), so a halo exchange is one send/recv (or one device
// copy) per neighbour and array, with no packing.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <unordered_map>
#include <vector>

#include <nccl.h>

#include "../../include/topmg_b200.h"
#include "kernels.h"
#include <nvtx3/nvToolsExt.h>

using namespace tmg;

// NVTX ranges (SURVEY.md §5 tracing): every ABI entry point that launches
// work and every set-up phase shows up as a named range in Nsight Systems /
// Compute timelines. Header-only NVTX v3; free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace {
thread_local std::string g_create_error;

struct Fail {
  int code;
};

// Partition of the cc-element z-layers over `total` slabs.
struct Part {
  int64_t cz0, cz1;  // coarse-cell z layers [cz0, cz1)
  int64_t b0, nbo, e0, neo;
  int lo, hi;        // ghost layers below / above
};

Part partition(const GridParams& g, int slab, int total) {
  Part p{};
  const int64_t per = g.ncz / total;  // cc layers per slab
  const int64_t ccz0 = per * slab, ccz1 = per * (slab + 1);
  p.cz0 = ccz0 * g.sd;
  p.cz1 = ccz1 * g.sd;
  const int64_t L = g.nbx * g.nby, Le = g.ncx * g.ncy;
  p.b0 = p.cz0 * L;
  p.nbo = (p.cz1 - p.cz0) * L;
  p.e0 = ccz0 * Le;
  p.neo = (ccz1 - ccz0) * Le;
  p.lo = slab > 0;
  p.hi = slab + 1 < total;
  return p;
}
}  // namespace

// One rank's halo exchange as a list of point-to-point operations, in
// global units (bricks, or cc elements with elem): the own bottom layer goes
// to rank - 1 and its top layer comes back as the lower ghost, symmetrically
// above. exchange() issues exactly these as grouped ncclSend / ncclRecv;
// tmg_halo_plan exports them so the multi-process host logic is tested with
// gloo on CPU (tests/test_dist_cpu.py).
struct HaloOp {
  int send;  // 1 send, 0 receive
  int peer;
  int64_t unit0, units;
};
std::vector<HaloOp> halo_ops(const Part& p, int rank, int64_t Lu, bool elem) {
  const int64_t u0 = elem ? p.e0 : p.b0, nu = elem ? p.neo : p.nbo;
  std::vector<HaloOp> ops;
  if (p.lo) {
    ops.push_back({1, rank - 1, u0, Lu});
    ops.push_back({0, rank - 1, u0 - Lu, Lu});
  }
  if (p.hi) {
    ops.push_back({1, rank + 1, u0 + nu - Lu, Lu});
    ops.push_back({0, rank + 1, u0 + nu, Lu});
  }
  return ops;
}

struct Slab {
  int id = 0;  // global slab index (= rank for NCCL contexts)
  GridParams g{};
  int lo = 0, hi = 0;
  int64_t L = 0, Le = 0;      // bricks / cc elements per z-layer
  int64_t bs0 = 0, nbs = 0;   // stored bricks (incl. ghost layers)
  int64_t es0 = 0, nes = 0;   // stored cc elements (incl. ghost layers)
  int64_t xoff = 0, xcells = 0;  // x-fastest cells of the slab: global offset, count
  // problem (virtual global pointers)
  double* kappa = nullptr;
  double* coef = nullptr;  // 4 x mst operator coefficients (Tx+, Ty+, Tz+, diag)
  double* tf = nullptr;    // face-major T of the owned bricks' 6 faces (k_face_t)
  uint8_t* dmask = nullptr;
  // preconditioner
  double* dinv = nullptr;
  double* phi = nullptr;
  double* phif = nullptr;  // Phi on each brick's 6 face layers, face-major (k_phi_faces)
  double* phi_keep = nullptr;  // last set-up's bases (warm start of the next one)
  double* evals = nullptr;
  int* eig_iters = nullptr;
  double* Gf = nullptr;        // fine block factors: compact slots (tuned bricks) or boxes
  GSlot* gmap = nullptr;       // brick -> factor slot + scale (owned, virtual global)
  int64_t* flist = nullptr;    // factor slot -> brick
  int64_t nslots = 0;
  FineFactors ff() const { return FineFactors{Gf, gmap}; }
  double* Ac = nullptr;
  double* Bc = nullptr;
  double* Rcc = nullptr;
  double* cc_evals = nullptr;
  double* Winv = nullptr;
  double* Gbj = nullptr;  // block-Jacobi plane Schur inverses (virtual-global per element)
  double* ybj = nullptr;  // E = 32 block-Jacobi apply: per-cell plane-sweep values
  double* accRows = nullptr;  // row-distributed A_cc planes: this slab's rows [ncz][P/total][P]
  double *r2 = nullptr, *t2 = nullptr;  // cc-block-smoothed V-cycle: r1 + R_c^T e_c, r - A r2
  // vectors
  double *b = nullptr, *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *z = nullptr,
         *r1 = nullptr, *stage = nullptr;
  double* r1f = nullptr;  // r1 on each brick's 6 face layers, face-major (k_update)
  double* pbuf[2] = {nullptr, nullptr};  // ping-pong search directions
  double *rc = nullptr, *rc0 = nullptr, *ec = nullptr, *rc1 = nullptr, *tc = nullptr;
  PcgState* st = nullptr;
  double* partials = nullptr;
  double* history = nullptr;
  int* d_status = nullptr;
  unsigned long long* d_count = nullptr;
};

struct tmg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  tmg_grid grid{};
  GridParams g{};  // global grid (b0 = 0, nbo = nb, ...)
  int cb = 0;       // cubic brick edge of the templated kernels; 0 = generic shape (generic.cu)
  int fine_bj = 0;  // fine smoother blocks = cc elements (tmg_mmg_options.fine_blocks)
  // exact fine blocks by the generic box block Thomas (generic.cu): -1 none,
  // 0 = one box per brick, 1 = one box per cc element
  int box_kind = -1;
  int nu = 1;       // smoother sweeps (MmgOptions::smoother_sweeps); != 1: enqueue_vcycle_nu
  int64_t M = 0;   // global cells
  std::string err;
  // partition
  int total = 1;                 // slabs over all processes
  ncclComm_t comm = nullptr;     // NCCL contexts only
  std::vector<Slab> slabs;       // slabs held by this process
  // TMG_FORCE_DIST=1 (diagnostics): a one-slab context runs the partitioned
  // path over a one-rank NCCL communicator (all-reduce, all-gather, captured
  // NCCL calls), which is all of the NCCL transport but the halo send/recv
  bool force_dist = false;
  bool dist() const { return total > 1 || force_dist; }
  bool nccl() const { return comm != nullptr; }
  // problem
  bool have_problem = false;
  std::vector<Patch> patches;
  // preconditioner
  int kind = -1;
  bool have_setup = false;
  int lc = 4, lcc = 8;
  int lc_keep = 0;  // L_c of the kept bases
  int64_t n_cc = 0;
  double* AccT = nullptr;   // single slab: lower 64x64 tiles of A_cc^-1
  double* accP = nullptr;   // single slab, plane-Thomas A_cc solve: tiles + couplings + work
  bool acc_planes = false;
  bool acc_rows = false;  // partitioned: row blocks of the plane inverses per slab
  AccPlanesRef planes{};
  double* symvP = nullptr;  // single slab: GEMV partials
  double* Ainv = nullptr;   // partitioned: dense A_cc^-1 (row blocks per slab)
  double *rcc = nullptr, *ecc = nullptr;  // full-length cc vectors (one per process)
  unsigned int* gbar = nullptr;           // grid-barrier state of the fused coarse kernel
  int hist_cap = 0;
  PcgState* h_state = nullptr;  // pinned, 2 slots
  // graph
  cudaGraphExec_t graph = nullptr;
  int graph_chunk = 0;
  int64_t graph_kernels = 0;  // kernel nodes in one captured chunk
  int64_t kcount = 0;         // kernels enqueued (running count)
  int64_t launches = 0;       // kernels enqueued by solves (incl. graph nodes)
  int64_t bytes = 0;
  std::vector<void*> allocs;
  // released buffers kept for reuse (re-setup with the same sizes allocates
  // nothing); byte size of every live or pooled buffer
  std::vector<std::pair<void*, size_t>> pool;
  std::unordered_map<void*, size_t> sizes;
  std::unordered_map<void*, void*> virt;  // windowed pointer -> allocation
  double setup_seconds = 0.0;
  // SIMP design loop (tmg_simp_*): x-fastest design arrays + warm starts
  struct Simp {
    bool on = false;
    tmg_simp_options o{};
    tmg_mmg_options mmg{};
    int iter = 0;
    double *x = nullptr, *xphys = nullptr, *xnew = nullptr, *dc = nullptr, *dv = nullptr,
           *W = nullptr, *tmp = nullptr, *part = nullptr, *scal = nullptr;
    double *T = nullptr, *U = nullptr;  // previous state / adjoint (brick layout)
  } simp;
  // reference design loop with MMA (tmg_optim_*): x-fastest design arrays
  struct Optim {
    bool on = false;
    tmg_optim_options o{};
    tmg_mmg_options mmg{};
    int iter = 0;  // MmaState::iteration
    double *x = nullptr, *xp = nullptr, *xp2 = nullptr, *xnew = nullptr, *low = nullptr,
           *upp = nullptr, *grad = nullptr, *xb = nullptr, *part = nullptr, *sp = nullptr,
           *scal = nullptr;
    double *T = nullptr, *U = nullptr;  // last state / adjoint (brick layout)
    unsigned int* bar = nullptr;
    bool have_T = false;
  } opt;
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

#define NK(call)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess) {                                                            \
      set_err(c, TMG_ECUDA, "NCCL error %s at %s:%d", ncclGetErrorString(r_), __FILE__, \
              __LINE__);                                                                \
      throw Fail{TMG_ECUDA};                                                            \
    }                                                                                   \
  } while (0)

// Every pointer the context hands out is a handle dfree() must map back to
// one allocation: a plain allocation's address, or a windowed array's
// virtual base (allocation - offset, `virt`). The two sets never overlap: an
// address that equals a live virtual base is not handed out as a plain
// allocation, and a window whose virtual base equals another allocation's
// address is moved (otherwise freeing one array would release the other's
// storage to the pool while it is still in use).
void dfree(tmg_ctx* c, void* p);

template <typename T>
T* dalloc(tmg_ctx* c, int64_t n) {
  const size_t bytes = sizeof(T) * (size_t)std::max<int64_t>(n, 1);
  std::vector<void*> aside;
  void* p = nullptr;
  for (;;) {
    p = nullptr;
    for (size_t i = 0; i < c->pool.size(); ++i)
      if (c->pool[i].second == bytes && !c->virt.count(c->pool[i].first)) {
        p = c->pool[i].first;
        c->pool.erase(c->pool.begin() + (std::ptrdiff_t)i);
        break;
      }
    if (!p) {
      CK(cudaMalloc(&p, bytes));
      c->sizes[p] = bytes;
      c->bytes += (int64_t)bytes;
    }
    if (!c->virt.count(p)) break;
    aside.push_back(p);  // a windowed array's handle: not usable as a plain one
  }
  for (void* q : aside) c->pool.emplace_back(q, c->sizes[q]);
  c->allocs.push_back(p);
  return (T*)p;
}

// windowed allocation of n elements addressed as (virtual base + i), i in
// [off, off + n)
template <typename T>
T* wwindow(tmg_ctx* c, int64_t n, int64_t off) {
  std::vector<T*> aside;
  for (;;) {
    T* a = dalloc<T>(c, n + (int64_t)aside.size());  // a new size: not a pooled twin
    T* v = a - off;
    if (!c->virt.count((void*)v) && (v == a || !c->sizes.count((void*)v))) {
      for (T* q : aside) dfree(c, (void*)q);
      c->virt[(void*)v] = (void*)a;
      return v;
    }
    aside.push_back(a);
  }
}

// windowed allocation: `units` stored, first stored global unit `first`
template <typename T>
T* walloc(tmg_ctx* c, int64_t units, int64_t per, int64_t first) {
  return wwindow<T>(c, units * per, first * per);
}
template <typename T>
T* ghosted(tmg_ctx* c, const Slab& s, int64_t per) { return walloc<T>(c, s.nbs, per, s.bs0); }
template <typename T>
T* owned(tmg_ctx* c, const Slab& s, int64_t per) { return walloc<T>(c, s.g.nbo, per, s.g.b0); }
template <typename T>
T* owned_e(tmg_ctx* c, const Slab& s, int64_t per) { return walloc<T>(c, s.g.neo, per, s.g.e0); }
template <typename T>
T* ghosted_e(tmg_ctx* c, const Slab& s, int64_t per) { return walloc<T>(c, s.nes, per, s.es0); }

// release to the context's pool (freed for real in tmg_destroy)
void dfree(tmg_ctx* c, void* p) {
  if (!p) return;
  auto v = c->virt.find(p);
  if (v != c->virt.end()) {
    p = v->second;
    c->virt.erase(v);
  }
  auto it = std::find(c->allocs.begin(), c->allocs.end(), p);
  if (it == c->allocs.end()) return;
  c->allocs.erase(it);
  c->pool.emplace_back(p, c->sizes[p]);
}

template <typename T>
void dfree_null(tmg_ctx* c, T*& p) {
  dfree(c, (void*)p);
  p = nullptr;
}

void free_setup(tmg_ctx* c) {
  for (Slab& s : c->slabs) {
    dfree_null(c, s.dinv);
    if (s.phi) {  // kept for a warm-started re-set-up (tmg_mmg_options.warm_start)
      dfree_null(c, s.phi_keep);
      s.phi_keep = s.phi;
      s.phi = nullptr;
      c->lc_keep = c->lc;
    }
    dfree_null(c, s.phif);
    dfree_null(c, s.evals);
    dfree_null(c, s.eig_iters);
    dfree_null(c, s.Gf);
    dfree_null(c, s.gmap);
    dfree_null(c, s.flist);
    s.nslots = 0;
    dfree_null(c, s.Ac);
    dfree_null(c, s.Bc);
    dfree_null(c, s.Rcc);
    dfree_null(c, s.cc_evals);
    dfree_null(c, s.Winv);
    dfree_null(c, s.Gbj);
    dfree_null(c, s.ybj);
    dfree_null(c, s.r2);
    dfree_null(c, s.t2);
    dfree_null(c, s.rc);
    dfree_null(c, s.rc0);
    dfree_null(c, s.ec);
    dfree_null(c, s.rc1);
    dfree_null(c, s.tc);
  }
  dfree_null(c, c->AccT);
  dfree_null(c, c->accP);
  c->acc_planes = false;
  c->acc_rows = false;
  for (Slab& s : c->slabs) dfree_null(c, s.accRows);
  dfree_null(c, c->symvP);
  dfree_null(c, c->Ainv);
  dfree_null(c, c->rcc);
  dfree_null(c, c->ecc);
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  c->have_setup = false;
  c->kind = -1;
  c->box_kind = -1;
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

// cells of the host arrays this context reads/writes (NCCL: the own slab)
int64_t host_cells(const tmg_ctx* c) { return c->nccl() ? c->slabs[0].xcells : c->M; }

int64_t cells_per_brick(const tmg_ctx* c) { return brick_cells(c->g); }

// ------------------------------------------------------- ghost exchanges
//
// Fill the ghost layers of a windowed array: unit = brick (elem = false) or
// cc element (elem = true), `bytes` per unit. get(s) returns slab s's
// windowed base pointer.
void exchange(tmg_ctx* c, const std::function<void*(Slab&)>& get, size_t bytes, bool elem) {
  if (!c->dist()) return;
  cudaStream_t st = c->stream;
  auto unit = [&](Slab& s, int64_t u) { return (char*)get(s) + (int64_t)bytes * u; };
  if (!c->nccl()) {
    for (size_t k = 0; k < c->slabs.size(); ++k) {
      Slab& s = c->slabs[k];
      const int64_t u0 = elem ? s.g.e0 : s.g.b0, nu = elem ? s.g.neo : s.g.nbo;
      const int64_t Lu = elem ? s.Le : s.L;
      const size_t lb = (size_t)Lu * bytes;
      if (s.lo)
        CK(cudaMemcpyAsync(unit(s, u0 - Lu), unit(c->slabs[k - 1], u0 - Lu), lb,
                           cudaMemcpyDeviceToDevice, st));
      if (s.hi)
        CK(cudaMemcpyAsync(unit(s, u0 + nu), unit(c->slabs[k + 1], u0 + nu), lb,
                           cudaMemcpyDeviceToDevice, st));
    }
    return;
  }
  Slab& s = c->slabs[0];
  const std::vector<HaloOp> ops =
      halo_ops(partition(c->g, s.id, c->total), s.id, elem ? s.Le : s.L, elem);
  NK(ncclGroupStart());
  for (const HaloOp& o : ops) {
    const size_t nb = (size_t)o.units * bytes;
    if (o.send) NK(ncclSend(unit(s, o.unit0), nb, ncclChar, o.peer, c->comm, st));
    else NK(ncclRecv(unit(s, o.unit0), nb, ncclChar, o.peer, c->comm, st));
  }
  NK(ncclGroupEnd());
}

#define XCH(member, per_unit_bytes, elem) \
  exchange(c, [&](Slab& s_) { return (void*)s_.member; }, (per_unit_bytes), (elem))

void exchange_coef(tmg_ctx* c) {
  const int64_t C = cells_per_brick(c);
  for (int k = 0; k < 4; ++k)
    exchange(c, [&](Slab& s) { return (void*)(s.coef + (size_t)k * s.g.mst); },
             sizeof(double) * (size_t)C, false);
}

// cross-slab sum of PcgState::loc[which..] and the scalar update on every slab
void reduce_finalize(tmg_ctx* c, int which, int init) {
  const int nv = (which == kRedInit || which == kRedJacobi) ? 2 : 1;
  if (c->nccl())
    NK(ncclAllReduce(c->slabs[0].st->loc + which, c->slabs[0].st->loc + which, nv, ncclDouble,
                     ncclSum, c->comm, c->stream));
  FinArgs a{};
  a.ns = (int)c->slabs.size();
  for (int j = 0; j < a.ns; ++j) {
    a.st[j] = c->slabs[j].st;
    a.hist[j] = c->slabs[j].history;
  }
  launch_finalize(a, which, init, c->stream);
  ++c->kcount;
}

// ------------------------------------------------------ host <-> device
void upload(tmg_ctx* c, const double* host, const std::function<double*(Slab&)>& dst) {
  for (Slab& s : c->slabs) {
    const double* h = host + (c->nccl() ? 0 : s.xoff);
    CK(cudaMemcpyAsync(s.stage, h, sizeof(double) * (size_t)s.xcells, cudaMemcpyHostToDevice,
                       c->stream));
    launch_to_brick(s.g, c->cb, s.stage, dst(s), c->stream);
    CK(cudaGetLastError());
  }
}

void download(tmg_ctx* c, const std::function<double*(Slab&)>& src, double* host) {
  for (Slab& s : c->slabs) {
    launch_from_brick(s.g, c->cb, src(s), s.stage, c->stream);
    CK(cudaGetLastError());
    double* h = host + (c->nccl() ? 0 : s.xoff);
    CK(cudaMemcpyAsync(h, s.stage, sizeof(double) * (size_t)s.xcells, cudaMemcpyDeviceToHost,
                       c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
}

#define UP(host, member) upload(c, (host), [&](Slab& s_) { return s_.member; })
#define DOWN(member, host) download(c, [&](Slab& s_) { return s_.member; }, (host))

// device kappa (brick layout) is in s.kappa: ghosts, Dirichlet mask, faces,
// coefficients
int finish_problem(tmg_ctx* c) {
  return guard(c, [&] {
    const int64_t C = cells_per_brick(c);
    XCH(kappa, sizeof(double) * C, false);
    for (Slab& s : c->slabs) {
      CK(cudaMemsetAsync(s.d_count, 0, sizeof(unsigned long long), c->stream));
      launch_boundary(s.g, c->cb, c->patches.data(), (int)c->patches.size(), c->grid.lx,
                      c->grid.ly, c->grid.lz, s.kappa, nullptr, s.dmask, nullptr, s.d_count,
                      c->stream);
      CK(cudaGetLastError());
    }
    if (c->nccl())
      NK(ncclAllReduce(c->slabs[0].d_count, c->slabs[0].d_count, 1, ncclUint64, ncclSum, c->comm,
                       c->stream));
    unsigned long long cnt = 0;
    for (Slab& s : c->slabs) {
      unsigned long long v = 0;
      CK(cudaMemcpyAsync(&v, s.d_count, sizeof v, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      cnt += v;
    }
    if (cnt == 0) {
      set_err(c, TMG_ECONFIG,
              "assemble_system: no Dirichlet face on the boundary, the system would be singular");
      throw Fail{TMG_ECONFIG};
    }
    XCH(dmask, C, false);
    for (Slab& s : c->slabs) {
      launch_coefficients(s.g, c->cb, s.kappa, s.dmask, s.coef, c->stream);
      CK(cudaGetLastError());
    }
    exchange_coef(c);
    for (Slab& s : c->slabs) {  // face-major T (after the ghost coefficients)
      if (c->cb == 0) break;    // read only by the templated boundary-form kernels
      if (!s.tf) s.tf = owned<double>(c, s, 6 * c->cb * c->cb);
      launch_face_t(s.g, c->cb, s.coef, s.tf, c->stream);
      CK(cudaGetLastError());
    }
    c->have_problem = true;
    free_setup(c);
  });
}

// Factor slots of the per-brick exact fine blocks (FineFactors): interior
// bricks of one uniform conductivity (cells and face halo) need no factor
// (slot -1, fast diagonalisation with scale 1 / face_t(k, k)); every other
// brick gets its own slot. TMG_G_SHARE=0 gives every brick a slot (A/B).
void plan_fine_factors(tmg_ctx* c, Slab& s) {
  const char* e = getenv("TMG_G_SHARE");
  const bool share = !(e && e[0] == '0');
  const int64_t nbo = s.g.nbo;
  std::vector<int> flag((size_t)nbo, 0);
  int* dflag = dalloc<int>(c, nbo);
  if (share) {
    launch_uniform_bricks(s.g, c->cb, s.kappa, dflag, c->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(flag.data(), dflag, sizeof(int) * (size_t)nbo, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  std::vector<GSlot> map((size_t)nbo);
  std::vector<int64_t> list;
  list.reserve((size_t)nbo);
  for (int64_t i = 0; i < nbo; ++i) {
    if (flag[(size_t)i]) {
      map[(size_t)i] = GSlot{-1, 1.0};
    } else {
      map[(size_t)i] = GSlot{(int64_t)list.size(), 1.0};
      list.push_back(s.g.b0 + i);
    }
  }
  s.nslots = (int64_t)list.size();
  s.gmap = owned<GSlot>(c, s, 1);
  s.flist = dalloc<int64_t>(c, std::max<int64_t>(s.nslots, 1));
  CK(cudaMemcpyAsync(s.gmap + s.g.b0, map.data(), sizeof(GSlot) * (size_t)nbo,
                     cudaMemcpyHostToDevice, c->stream));
  if (s.nslots)
    CK(cudaMemcpyAsync(s.flist, list.data(), sizeof(int64_t) * (size_t)s.nslots,
                       cudaMemcpyHostToDevice, c->stream));
  if (share) launch_factor_scales(s.g, c->cb, s.kappa, dflag, s.gmap, c->stream);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));  // the host vectors die here
  dfree(c, dflag);
}

// ---------------------------------------------------------------- V-cycle
#define KL(n_kernels, call)     \
  do {                          \
    call;                       \
    c->kcount += (n_kernels);   \
  } while (0)
#define KLR(call) /* launcher returns its kernel count */ \
  do {                                                    \
    c->kcount += (call);                                  \
  } while (0)

// single slab: coarse + coarse-coarse levels as one cooperative kernel
void enqueue_coarse_single(tmg_ctx* c) {
  Slab& s = c->slabs[0];
  if (c->acc_planes)
    KL(5 + acc_planes_solve_kernels(s.g),
       launch_coarse_cycle(s.g, &s.st->done, s.Ac, s.Winv, s.Rcc, nullptr, c->symvP, c->n_cc,
                           s.rc, s.rc0, c->rcc, c->ecc, s.rc1, s.tc, s.ec, &c->planes, c->stream));
  else if (getenv("TMG_UNFUSED_COARSE") || !coarse_fused_supported(s.g, c->n_cc))
    KL(7, launch_coarse_cycle(s.g, &s.st->done, s.Ac, s.Winv, s.Rcc, c->AccT, c->symvP, c->n_cc,
                              s.rc, s.rc0, c->rcc, c->ecc, s.rc1, s.tc, s.ec, nullptr, c->stream));
  else
    KL(1, launch_coarse_fused(s.g, &s.st->done, s.Ac, s.Winv, s.Rcc, c->AccT, c->symvP, c->n_cc,
                              s.rc, s.rc0, c->rcc, s.rc1, s.ec, c->gbar, c->stream));
}

// rc = R_c (r - A r1) after the per-brick fine block solve: the boundary form
// (k_restrict_bnd) unless TMG_RESTRICT_BND=0 at build time
static void restrict_fine(tmg_ctx* c, Slab& s, cudaStream_t st) {
#if TMG_RESTRICT_BND
  launch_restrict_bnd(s.g, c->cb, s.tf, s.phif, s.r1f, s.rc, s.st, st);
#else
  launch_restrict(s.g, c->cb, s.coef, s.phi, s.r, s.r1, s.rc, s.st, st);
#endif
}

// single slab: the fused path (device-side scalars, symmetric tiled A_cc GEMV)
void enqueue_vcycle_single(tmg_ctx* c, int init, const double* p) {
  Slab& s = c->slabs[0];
  const GridParams& g = s.g;
  cudaStream_t st = c->stream;
  KLR(launch_update(g, c->cb, s.coef, s.ff(), s.x, p, s.q, s.r, s.r1, s.r1f, s.st, s.partials,
                      s.history, init, st));
  KL(1, restrict_fine(c, s, st));
  enqueue_coarse_single(c);
  KLR(launch_post(g, c->cb, s.coef, s.tf, s.phi, s.phif, s.ff(), s.r, s.r1, s.r1f, s.ec, s.z, s.st, s.partials, init,
                    st));
}

// ecc = A_cc^-1 rcc on the full-length process vectors (rcc complete on
// every process): the plane block Thomas (replicated, or row-distributed with
// an in-place all-gather per plane step), the symmetric-tiles GEMV (single
// slab), or the row blocks of the dense inverse (partitioned).
void enqueue_acc_solve(tmg_ctx* c) {
  cudaStream_t st = c->stream;
  const int* done = &c->slabs[0].st->done;
  if (c->acc_rows) {
    const int64_t P = c->g.ncx * c->g.ncy * c->lcc, nr = P / c->total;
    std::vector<AccRowBlock> blocks;
    for (Slab& s : c->slabs) blocks.push_back(AccRowBlock{s.accRows, (int64_t)s.id * nr, nr});
    const int rank = c->slabs[0].id;
    KL(acc_rows_solve_kernels(c->g, (int)blocks.size()),
       launch_acc_rows_solve(c->g, done, c->planes.C, c->rcc, c->ecc, c->planes.wv, blocks,
                             [&](double* plane) {
                               if (c->nccl())
                                 NK(ncclAllGather(plane + (int64_t)rank * nr, plane, (size_t)nr,
                                                  ncclDouble, c->comm, st));
                             },
                             st));
  } else if (c->acc_planes) {
    KL(acc_planes_solve_kernels(c->g),
       launch_acc_planes_solve(c->g, done, c->planes.T, c->planes.C, c->rcc, c->ecc,
                               c->planes.wv, c->symvP, st));
  } else if (c->AccT) {
    KL(2, launch_symv(done, c->AccT, c->n_cc, c->rcc, c->symvP, c->ecc, st));
  } else {
    for (Slab& s : c->slabs)
      KL(1, launch_gemv_rows(&s.st->done, c->Ainv, c->n_cc, s.g.e0 * c->lcc, s.g.neo * c->lcc,
                             c->rcc, c->ecc, st));
  }
}

// partitioned coarse + coarse-coarse levels (solver.cpp:292-319): rc -> ec
void enqueue_coarse_dist(tmg_ctx* c) {
  cudaStream_t st = c->stream;
  const size_t cvec = sizeof(double) * (size_t)c->lc;
  for (Slab& s : c->slabs)
    KL(1, launch_coarse_smooth(s.g, &s.st->done, s.Winv, s.rc, nullptr, s.rc0, st));
  XCH(rc0, cvec, false);
  for (Slab& s : c->slabs)
    KL(1, launch_coarse_restrict(s.g, &s.st->done, s.Ac, s.Rcc, s.rc, s.rc0, c->rcc, st));
  if (c->nccl()) {
    const Slab& s = c->slabs[0];
    const int64_t own = s.g.neo * c->lcc;
    NK(ncclAllGather(c->rcc + s.g.e0 * c->lcc, c->rcc, (size_t)own, ncclDouble, c->comm, st));
  }
  enqueue_acc_solve(c);  // replicated or row-distributed (once for in-process slabs)
  for (Slab& s : c->slabs)
    KL(1, launch_coarse_prolong(s.g, &s.st->done, s.Rcc, s.rc0, c->ecc, s.rc1, st));
  XCH(rc1, cvec, false);
  for (Slab& s : c->slabs)
    KL(1, launch_coarse_resid(s.g, &s.st->done, s.Ac, s.rc, s.rc1, s.tc, st));
  for (Slab& s : c->slabs)
    KL(1, launch_coarse_smooth(s.g, &s.st->done, s.Winv, s.tc, s.rc1, s.ec, st));
  XCH(ec, cvec, false);
}

// partitioned: the same kernels per slab, ghost exchanges and cross-slab
// reductions between them (SURVEY.md §8(e) "collectives per PCG iteration")
void enqueue_vcycle_dist(tmg_ctx* c, int init, int par_new) {
  cudaStream_t st = c->stream;
  const int64_t C = cells_per_brick(c);
  for (Slab& s : c->slabs)
    KLR(launch_update(s.g, c->cb, s.coef, s.ff(), s.x, s.pbuf[par_new], s.q, s.r, s.r1, s.r1f, s.st,
                        s.partials, s.history, init, st));
  if (!init) reduce_finalize(c, kRedUpdate, 0);
  XCH(r1f, sizeof(double) * 6 * c->cb * c->cb, false);  // the boundary kernels read r1's face layers
  if (TMG_R1_FULL) XCH(r1, sizeof(double) * C, false);
  for (Slab& s : c->slabs) KL(1, restrict_fine(c, s, st));
  enqueue_coarse_dist(c);
  for (Slab& s : c->slabs)
    KLR(launch_post(s.g, c->cb, s.coef, s.tf, s.phi, s.phif, s.ff(), s.r, s.r1, s.r1f, s.ec, s.z, s.st, s.partials,
                      init, st));
  reduce_finalize(c, kRedPost, init);
  XCH(z, sizeof(double) * C, false);
}

// block_jacobi (BlockJacobiPreconditioner, solver.cpp:444-458): x, r update
// and the stopping test, then z = A_BB^-1 r per cc element and r.z
void enqueue_block_jacobi(tmg_ctx* c, int init, int par_new) {
  const int64_t C = cells_per_brick(c);
  if (!init) {
    for (Slab& s : c->slabs)
      KL(1, launch_jacobi_step(s.g, c->cb, nullptr, s.x, s.pbuf[par_new], s.q, s.r, s.z, s.st,
                               s.partials, s.history, 0, 1, c->stream));
    if (c->dist()) reduce_finalize(c, kRedUpdate, 0);
  }
  if (c->box_kind == 1) {  // box block Thomas over the cc elements (generic.cu)
    const int64_t per = box_doubles(c->g, 1);
    for (Slab& s : c->slabs)
      KL(box_apply_kernels(s.g, 1),
         launch_box_apply(s.g, 1, s.coef, s.Gbj + s.g.e0 * per, s.r, nullptr, s.z, s.r, s.st,
                          s.partials, init, s.ybj, c->stream));
  } else {
    const int64_t per = bj_doubles_per_element(c->cb, c->g.sd);
    const int nk = bj_apply_kernels(c->cb, c->g.sd);
    for (Slab& s : c->slabs)
      KL(nk, launch_bj_apply(s.g, c->cb, s.coef, s.Gbj + s.g.e0 * per, s.r, nullptr, s.z, s.r,
                             s.st, s.partials, init, s.ybj, c->stream));
  }
  if (c->dist()) {
    reduce_finalize(c, kRedPost, init);
    XCH(z, sizeof(double) * C, false);
  }
}

void enqueue_jacobi(tmg_ctx* c, int init, int par_new) {
  if (c->kind == TMG_PRECOND_BLOCK_JACOBI) return enqueue_block_jacobi(c, init, par_new);
  const int64_t C = cells_per_brick(c);
  for (Slab& s : c->slabs)
    KL(1, launch_jacobi_step(s.g, c->cb, c->kind == TMG_PRECOND_JACOBI ? s.dinv : nullptr, s.x,
                             s.pbuf[par_new], s.q, s.r, s.z, s.st, s.partials, s.history, init,
                             0, c->stream));
  if (c->dist()) {
    reduce_finalize(c, kRedJacobi, init);
    XCH(z, sizeof(double) * C, false);
  }
}

// V-cycle with the reference build_mmg fine blocks (one per cc element,
// tmg_mmg_options.fine_blocks = TMG_FINE_BLOCKS_CC), solver.cpp:272-334:
//   r1 = B^-1 r; rc = R_c (r - A r1); coarse levels; r2 = r1 + R_c^T ec;
//   z = r2 + B^-1 (r - A r2); r.z
void enqueue_vcycle_bj(tmg_ctx* c, int init, int par_new) {
  const int64_t C = cells_per_brick(c);
  cudaStream_t st = c->stream;
  if (!init) {
    for (Slab& s : c->slabs)
      KL(1, launch_jacobi_step(s.g, c->cb, nullptr, s.x, s.pbuf[par_new], s.q, s.r, s.z, s.st,
                               s.partials, s.history, 0, 1, st));
    if (c->dist()) reduce_finalize(c, kRedUpdate, 0);
  }
  const int64_t per = bj_doubles_per_element(c->cb, c->g.sd);
  const int nk = bj_apply_kernels(c->cb, c->g.sd);
  for (Slab& s : c->slabs)
    KL(nk, launch_bj_apply(s.g, c->cb, s.coef, s.Gbj + s.g.e0 * per, s.r, nullptr, s.r1, nullptr,
                           s.st, s.partials, init, s.ybj, st));
  if (c->dist()) XCH(r1, sizeof(double) * C, false);
  for (Slab& s : c->slabs)
    KL(1, launch_restrict(s.g, c->cb, s.coef, s.phi, s.r, s.r1, s.rc, s.st, st));
  if (c->dist()) enqueue_coarse_dist(c);
  else enqueue_coarse_single(c);
  for (Slab& s : c->slabs)
    KL(1, launch_prolong_add(s.g, c->cb, s.phi, s.r1, s.ec, s.r2, s.st, st));
  if (c->dist()) XCH(r2, sizeof(double) * C, false);
  for (Slab& s : c->slabs) KL(1, launch_resid(s.g, c->cb, s.coef, s.r, s.r2, s.t2, s.st, st));
  for (Slab& s : c->slabs)
    KL(nk, launch_bj_apply(s.g, c->cb, s.coef, s.Gbj + s.g.e0 * per, s.t2, s.r2, s.z, s.r, s.st,
                           s.partials, init, s.ybj, st));
  if (c->dist()) {
    reduce_finalize(c, kRedPost, init);
    XCH(z, sizeof(double) * C, false);
  }
}

// The V-cycle of solver.cpp:272-334 with any number nu of smoother sweeps
// (MmgOptions::smoother_sweeps; BlockJacobiSmoother::apply, :221-243) on
// both levels, from unfused phase kernels. Every smoothing stage iterates on
// its output: y = a + S(b - A a) first, then y += S(b - A y) for each further
// sweep (from a = 0 for the pre-smoothers), which is the reference's sweep
// loop written on y; nu = 0 leaves the coarse corrections only.
void enqueue_vcycle_nu(tmg_ctx* c, int init, int par_new) {
  const int64_t C = cells_per_brick(c);
  cudaStream_t st = c->stream;
  const int nu = c->nu;
  const size_t cvec = sizeof(double) * (size_t)c->lc;
  const bool gen = c->box_kind >= 0;
  const int64_t per = gen ? box_doubles(c->g, c->box_kind)
                          : bj_doubles_per_element(c->cb, c->g.sd);
  const int nk = gen ? box_apply_kernels(c->g, c->box_kind)
                     : c->fine_bj ? bj_apply_kernels(c->cb, c->g.sd) : 1;
  if (!init) {  // x, r update + stopping test (the z write is deferred)
    for (Slab& s : c->slabs)
      KL(1, launch_jacobi_step(s.g, c->cb, nullptr, s.x, s.pbuf[par_new], s.q, s.r, s.z, s.st,
                               s.partials, s.history, 0, 1, st));
    if (c->dist()) reduce_finalize(c, kRedUpdate, 0);
  }
  // out = add + B^-1 in (per coarse cell or per cc element), optional r.out
  auto fine_solve = [&](Slab& s, const double* in, const double* add, double* out,
                        const double* rdot) {
    if (c->box_kind == 1)  // box block Thomas (generic.cu)
      KL(nk, launch_box_apply(s.g, 1, s.coef, s.Gbj + s.g.e0 * per, in, add, out, rdot, s.st,
                              s.partials, init, s.ybj, st));
    else if (c->box_kind == 0)
      KL(nk, launch_box_apply(s.g, 0, s.coef, s.Gf + s.g.b0 * per, in, add, out, rdot, s.st,
                              s.partials, init, s.ybj, st));
    else if (c->fine_bj)
      KL(nk, launch_bj_apply(s.g, c->cb, s.coef, s.Gbj + s.g.e0 * per, in, add, out, rdot, s.st,
                             s.partials, init, s.ybj, st));
    else
      KL(1, launch_brick_solve(s.g, c->cb, s.coef, s.ff(), in, add, out, rdot, s.st, s.partials,
                               init, st));
  };
  // ---- fine pre-smoothing r1 = S_nu(r) ----
  for (int sw = 0; sw < nu; ++sw) {
    if (sw == 0) {
      for (Slab& s : c->slabs) fine_solve(s, s.r, nullptr, s.r1, nullptr);
    } else {
      XCH(r1, sizeof(double) * C, false);
      for (Slab& s : c->slabs) KL(1, launch_resid(s.g, c->cb, s.coef, s.r, s.r1, s.t2, s.st, st));
      for (Slab& s : c->slabs) fine_solve(s, s.t2, s.r1, s.r1, nullptr);
    }
  }
  if (nu == 0)
    for (Slab& s : c->slabs)
      CK(cudaMemsetAsync(s.r1 + s.g.b0 * C, 0, sizeof(double) * (size_t)(s.g.nbo * C), st));
  XCH(r1, sizeof(double) * C, false);
  for (Slab& s : c->slabs)  // rc = R_c (r - A r1)
    KL(1, launch_restrict(s.g, c->cb, s.coef, s.phi, s.r, s.r1, s.rc, s.st, st));
  // ---- coarse pre-smoothing rc0 = S_nu(rc) ----
  for (int sw = 0; sw < nu; ++sw) {
    if (sw == 0) {
      for (Slab& s : c->slabs)
        KL(1, launch_coarse_smooth(s.g, &s.st->done, s.Winv, s.rc, nullptr, s.rc0, st));
    } else {
      XCH(rc0, cvec, false);
      for (Slab& s : c->slabs)
        KL(1, launch_coarse_resid(s.g, &s.st->done, s.Ac, s.rc, s.rc0, s.tc, st));
      for (Slab& s : c->slabs)
        KL(1, launch_coarse_smooth(s.g, &s.st->done, s.Winv, s.tc, s.rc0, s.rc0, st));
    }
  }
  if (nu == 0)
    for (Slab& s : c->slabs)
      CK(cudaMemsetAsync(s.rc0 + s.bs0 * c->lc, 0, sizeof(double) * (size_t)(s.nbs * c->lc), st));
  XCH(rc0, cvec, false);
  // ---- coarse-coarse: rcc = R_cc (rc - A_c rc0); ecc = A_cc^-1 rcc ----
  for (Slab& s : c->slabs)
    KL(1, launch_coarse_restrict(s.g, &s.st->done, s.Ac, s.Rcc, s.rc, s.rc0, c->rcc, st));
  if (c->nccl()) {
    const Slab& s = c->slabs[0];
    NK(ncclAllGather(c->rcc + s.g.e0 * c->lcc, c->rcc, (size_t)(s.g.neo * c->lcc), ncclDouble,
                     c->comm, st));
  }
  enqueue_acc_solve(c);
  for (Slab& s : c->slabs)  // rc1 = rc0 + R_cc^T ecc
    KL(1, launch_coarse_prolong(s.g, &s.st->done, s.Rcc, s.rc0, c->ecc, s.rc1, st));
  // ---- coarse post-smoothing ec = rc1 + S_nu(rc - A_c rc1) ----
  if (nu == 0)
    for (Slab& s : c->slabs)
      CK(cudaMemcpyAsync(s.ec + s.bs0 * c->lc, s.rc1 + s.bs0 * c->lc,
                         sizeof(double) * (size_t)(s.nbs * c->lc), cudaMemcpyDeviceToDevice, st));
  for (int sw = 0; sw < nu; ++sw) {
    if (sw == 0) {
      XCH(rc1, cvec, false);
      for (Slab& s : c->slabs)
        KL(1, launch_coarse_resid(s.g, &s.st->done, s.Ac, s.rc, s.rc1, s.tc, st));
      for (Slab& s : c->slabs)
        KL(1, launch_coarse_smooth(s.g, &s.st->done, s.Winv, s.tc, s.rc1, s.ec, st));
    } else {
      XCH(ec, cvec, false);
      for (Slab& s : c->slabs)
        KL(1, launch_coarse_resid(s.g, &s.st->done, s.Ac, s.rc, s.ec, s.tc, st));
      for (Slab& s : c->slabs)
        KL(1, launch_coarse_smooth(s.g, &s.st->done, s.Winv, s.tc, s.ec, s.ec, st));
    }
  }
  // ---- fine: r2 = r1 + R_c^T ec; z = r2 + S_nu(r - A r2); r.z ----
  for (Slab& s : c->slabs)
    KL(1, launch_prolong_add(s.g, c->cb, s.phi, s.r1, s.ec, s.r2, s.st, st));
  if (nu == 0) {
    for (Slab& s : c->slabs)
      KL(1, launch_add_finish(s.g, c->cb, s.r2, nullptr, s.z, s.r, s.st, s.partials, init, st));
  }
  for (int sw = 0; sw < nu; ++sw) {
    const bool last = sw + 1 == nu;
    if (sw == 0) {
      XCH(r2, sizeof(double) * C, false);
      for (Slab& s : c->slabs) KL(1, launch_resid(s.g, c->cb, s.coef, s.r, s.r2, s.t2, s.st, st));
      for (Slab& s : c->slabs) fine_solve(s, s.t2, s.r2, s.z, last ? s.r : nullptr);
    } else {
      XCH(z, sizeof(double) * C, false);
      for (Slab& s : c->slabs) KL(1, launch_resid(s.g, c->cb, s.coef, s.r, s.z, s.t2, s.st, st));
      for (Slab& s : c->slabs) fine_solve(s, s.t2, s.z, s.z, last ? s.r : nullptr);
    }
  }
  if (c->dist()) {
    reduce_finalize(c, kRedPost, init);
    XCH(z, sizeof(double) * C, false);
  }
}

// p = z + beta p_old, q = A p, p.q from the stored coefficients (64 B/cell).
// TMG_SEARCH_KAPPA=1 recomputes them from kappa instead (40 B/cell, bitwise
// the same q): measured slower at configs[3], 3.94 against 2.35 ms per launch
// -- the 3.4 face divisions per cell and the face/diagonal assembly make the
// kernel issue-bound.
void search(tmg_ctx* c, Slab& s, const double* pold, double* pnew, cudaStream_t st) {
  static const bool from_kappa = getenv("TMG_SEARCH_KAPPA") && getenv("TMG_SEARCH_KAPPA")[0] == '1';
  if (c->cb != 0 && from_kappa)
    launch_search_kappa(s.g, c->cb, s.kappa, s.dmask, s.z, pold, pnew, s.q, s.st, s.partials, st);
  else
    launch_search(s.g, c->cb, s.coef, s.z, pold, pnew, s.q, s.st, s.partials, st);
}

bool hierarchical(const tmg_ctx* c) {
  return c->kind == TMG_PRECOND_MMG || c->kind == TMG_PRECOND_TWO_GRID;
}

// z = M^-1 r and r.z for the current preconditioner (init: first application,
// x0 residual already in r); otherwise after the search step of an iteration.
void enqueue_precond(tmg_ctx* c, int init, int par_new) {
  if (!hierarchical(c)) return enqueue_jacobi(c, init, par_new);
  if (c->nu != 1 || c->cb == 0 || c->box_kind >= 0) enqueue_vcycle_nu(c, init, par_new);
  else if (c->fine_bj) enqueue_vcycle_bj(c, init, par_new);
  else if (c->dist()) enqueue_vcycle_dist(c, init, par_new);
  else enqueue_vcycle_single(c, init, c->slabs[0].pbuf[par_new]);
}

void enqueue_precond_init(tmg_ctx* c) { enqueue_precond(c, 1, 0); }

// Iteration with parity `par`: reads p from pbuf[par], writes pbuf[par ^ 1].
void enqueue_iteration(tmg_ctx* c, int par) {
  const int64_t C = cells_per_brick(c);
  for (Slab& s : c->slabs)
    KL(search_kernels(c->cb), search(c, s, s.pbuf[par], s.pbuf[par ^ 1], c->stream));
  if (c->dist()) {
    reduce_finalize(c, kRedSearch, 0);
    exchange(c, [&](Slab& s) { return (void*)s.pbuf[par ^ 1]; }, sizeof(double) * C, false);
  }
  enqueue_precond(c, 0, par ^ 1);
}

void build_graph(tmg_ctx* c, int chunk) {
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  cudaGraph_t graph;
  const int64_t k0 = c->kcount;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  // chunk is even so every graph launch starts from pbuf[0]
  for (int i = 0; i < chunk; ++i) enqueue_iteration(c, i & 1);
  CK(cudaStreamEndCapture(c->stream, &graph));
  c->graph_kernels = c->kcount - k0;
  c->kcount = k0;
  CK(cudaGraphInstantiate(&c->graph, graph, 0));
  cudaGraphDestroy(graph);
  c->graph_chunk = chunk;
}

void ensure_history(tmg_ctx* c, int maxit) {
  if (maxit <= c->hist_cap) return;
  for (Slab& s : c->slabs) {
    dfree_null(c, s.history);
    s.history = dalloc<double>(c, maxit);
  }
  c->hist_cap = maxit;
  // the captured graph holds the history pointers
  if (c->graph) build_graph(c, c->graph_chunk);
}

void init_states(tmg_ctx* c, double rtol, int maxit) {
  PcgState init{};
  init.rtol = rtol;
  init.maxit = maxit;
  init.hist_cap = c->hist_cap;
  for (Slab& s : c->slabs)
    CK(cudaMemcpyAsync(s.st, &init, sizeof init, cudaMemcpyHostToDevice, c->stream));
}

// Runs the device solve on resident b (and x if use_x0).
void solve_device(tmg_ctx* c, double rtol, int maxit, int use_x0, tmg_report* rep,
                  double* ms_total, int* counts) {
  if (!c->have_setup) {
    set_err(c, TMG_EARG, "pcg: no preconditioner set up (call tmg_setup)");
    throw Fail{TMG_EARG};
  }
  ensure_history(c, std::max(maxit, 1));
  const int64_t C = cells_per_brick(c);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, c->stream));
  init_states(c, rtol, maxit);
  const bool prof = ms_total != nullptr && !c->dist();
  Slab& s0 = c->slabs[0];
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
  const int64_t k_before = c->kcount;
  if (use_x0) XCH(x, sizeof(double) * C, false);
  timed(8, [&] {
    for (Slab& s : c->slabs)
      KL(1, launch_init(s.g, c->cb, s.coef, s.b, s.x, use_x0, s.r, s.st, s.partials, c->stream));
    if (c->dist()) reduce_finalize(c, kRedInit, 0);
  });
  if (!prof) {
    enqueue_precond_init(c);
  } else if (hierarchical(c) && !c->fine_bj && c->nu == 1 && c->cb != 0) {
    Slab& s = s0;
    const GridParams& g = s.g;
    timed(1, [&] { KLR(launch_update(g, c->cb, s.coef, s.ff(), s.x, s.p, s.q, s.r, s.r1, s.r1f, s.st, s.partials, s.history, 1, c->stream)); });
    timed(2, [&] { KL(1, restrict_fine(c, s, c->stream)); });
    timed(3, [&] { enqueue_coarse_single(c); });
    timed(6, [&] { KLR(launch_post(g, c->cb, s.coef, s.tf, s.phi, s.phif, s.ff(), s.r, s.r1, s.r1f, s.ec, s.z, s.st, s.partials, 1, c->stream)); });
  } else {
    timed(7, [&] { enqueue_precond(c, 1, 0); });
  }
  CK(cudaGetLastError());
  c->launches += c->kcount - k_before;
  PcgState* hs = c->h_state;
  if (!prof) {
    // chunked graph launches; the next chunk is enqueued before the previous
    // one's state is polled, so the GPU never idles on the host.
    CK(cudaMemcpyAsync(&hs[0], s0.st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (!hs[0].done && maxit > 0) {
      cudaEvent_t ev[2];
      CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
      int launched = 0;
      auto launch_chunk = [&](int sl) {
        CK(cudaGraphLaunch(c->graph, c->stream));
        c->launches += c->graph_kernels;
        CK(cudaMemcpyAsync(&hs[sl], s0.st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
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
    Slab& s = s0;
    CK(cudaMemcpy(&hs[0], s.st, sizeof(PcgState), cudaMemcpyDeviceToHost));
    int guard_it = 0, par = 0;
    while (!hs[0].done && maxit > 0 && guard_it++ <= maxit) {
      const double* pold = s.pbuf[par];
      double* pnew = s.pbuf[par ^ 1];
      par ^= 1;
      const int64_t kb = c->kcount;
      timed(0, [&] { KL(search_kernels(c->cb), search(c, s, pold, pnew, c->stream)); });
      if (hierarchical(c) && !c->fine_bj && c->nu == 1 && c->cb != 0) {
        timed(1, [&] { KLR(launch_update(s.g, c->cb, s.coef, s.ff(), s.x, pnew, s.q, s.r, s.r1, s.r1f, s.st, s.partials, s.history, 0, c->stream)); });
        timed(2, [&] { KL(1, restrict_fine(c, s, c->stream)); });
        timed(3, [&] { enqueue_coarse_single(c); });
        timed(6, [&] { KLR(launch_post(s.g, c->cb, s.coef, s.tf, s.phi, s.phif, s.ff(), s.r, s.r1, s.r1f, s.ec, s.z, s.st, s.partials, 0, c->stream)); });
      } else {
        timed(7, [&] { enqueue_precond(c, 0, par); });
      }
      c->launches += c->kcount - kb;
      CK(cudaMemcpy(&hs[0], s.st, sizeof(PcgState), cudaMemcpyDeviceToHost));
    }
  }
  CK(cudaEventRecord(e1, c->stream));
  CK(cudaMemcpyAsync(&hs[0], s0.st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaGetLastError());
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  PcgState& f = hs[0];
  if (!f.done && maxit == 0) f.status = kStatusMaxIt;
  if (f.status == kStatusZeroRhs) {
    for (Slab& s : c->slabs)  // solver.cpp:506-513
      CK(cudaMemsetAsync(s.x + s.g.b0 * C, 0, sizeof(double) * (size_t)(s.g.nbo * C), c->stream));
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

// Validates the hierarchy like build_hierarchy (grid.cpp:191-218) and picks
// the kernels: cubic 4^3 / 8^3 coarse cells run the templated ones (*cb_out =
// edge), every other shape the generic ones (*cb_out = 0; TMG_FORCE_GENERIC=1
// forces them for 4^3 / 8^3 too, for A/B tests).
int check_grid(const tmg_grid* grid, int64_t* cb_out) {
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
  if (cpc[0] * cpc[1] * cpc[2] > (int64_t)1 << 20)
    return set_err(nullptr, TMG_ENOTSUP,
                   "GPU path handles coarse cells of up to 2^20 fine cells (got %lldx%lldx%lld)",
                   (long long)cpc[0], (long long)cpc[1], (long long)cpc[2]);
  const char* fg = getenv("TMG_FORCE_GENERIC");
  const bool force = fg && atoi(fg) > 0;
  const bool tuned = cpc[0] == cpc[1] && cpc[1] == cpc[2] && (cpc[0] == 4 || cpc[0] == 8);
  *cb_out = tuned && !force ? cpc[0] : 0;
  return TMG_OK;
}

GridParams global_params(const tmg_grid& G) {
  GridParams g{};
  g.nx = G.nx; g.ny = G.ny; g.nz = G.nz;
  g.nbx = G.ncc[0] * G.sd; g.nby = G.ncc[1] * G.sd; g.nbz = G.ncc[2] * G.sd;
  g.bx = (int)(G.nx / g.nbx); g.by = (int)(G.ny / g.nby); g.bz = (int)(G.nz / g.nbz);
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
  g.mst = G.nx * G.ny * G.nz;
  g.dist = 0;
  return g;
}

int check_partition(const tmg_grid* grid, int total) {
  if (total < 1 || total > kMaxSlabs)
    return set_err(nullptr, TMG_EARG, "partition: 1..%d slabs (got %d)", kMaxSlabs, total);
  if (grid->ncc[2] % total != 0)
    return set_err(nullptr, TMG_ECONFIG,
                   "partition: %d slabs must divide the %lld cc-element layers along z", total,
                   (long long)grid->ncc[2]);
  return TMG_OK;
}

// create a context holding slabs [first, first + count) of `total`
int create_impl(const tmg_grid* grid, int device, int first, int count, int total,
                const void* nccl_id, tmg_ctx** out) {
  if (!grid || !out) return set_err(nullptr, TMG_EARG, "tmg_create: null argument");
  *out = nullptr;
  int64_t cb = 0;
  int rc = check_grid(grid, &cb);
  if (rc) return rc;
  rc = check_partition(grid, total);
  if (rc) return rc;
  if (count < 1 || first < 0 || first + count > total)
    return set_err(nullptr, TMG_EARG, "partition: bad slab range %d+%d of %d", first, count, total);
  tmg_ctx* c = new tmg_ctx;
  c->grid = *grid;
  c->device = device;
  c->cb = (int)cb;
  c->M = grid->nx * grid->ny * grid->nz;
  c->g = global_params(*grid);
  c->total = total;
  const int64_t C = cells_per_brick(c);
  rc = guard(c, [&] {
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    init_kernel_attributes();
    if (nccl_id) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof id);
      NK(ncclCommInitRank(&c->comm, total, id, first));
    } else if (total == 1 && getenv("TMG_FORCE_DIST") && atoi(getenv("TMG_FORCE_DIST")) > 0) {
      ncclUniqueId id;
      NK(ncclGetUniqueId(&id));
      NK(ncclCommInitRank(&c->comm, 1, id, 0));
      c->force_dist = true;
    }
    c->slabs.resize((size_t)count);
    for (int k = 0; k < count; ++k) {
      Slab& s = c->slabs[(size_t)k];
      s.id = first + k;
      const Part p = partition(c->g, s.id, total);
      s.g = c->g;
      s.g.b0 = p.b0;
      s.g.nbo = p.nbo;
      s.g.e0 = p.e0;
      s.g.neo = p.neo;
      s.g.dist = c->dist();
      s.lo = p.lo;
      s.hi = p.hi;
      s.L = c->g.nbx * c->g.nby;
      s.Le = c->g.ncx * c->g.ncy;
      s.bs0 = p.b0 - p.lo * s.L;
      s.nbs = p.nbo + (p.lo + p.hi) * s.L;
      s.es0 = p.e0 - p.lo * s.Le;
      s.nes = p.neo + (p.lo + p.hi) * s.Le;
      s.xoff = p.cz0 * c->g.bz * c->g.nx * c->g.ny;
      s.xcells = (p.cz1 - p.cz0) * c->g.bz * c->g.nx * c->g.ny;
      s.g.mst = s.nbs * C;
      s.kappa = ghosted<double>(c, s, C);
      s.dmask = ghosted<uint8_t>(c, s, C);
      s.coef = wwindow<double>(c, 4 * s.g.mst, s.bs0 * C);
      for (double** v : {&s.b, &s.x, &s.r, &s.q, &s.z, &s.r1}) *v = ghosted<double>(c, s, C);
      s.pbuf[0] = ghosted<double>(c, s, C);
      s.pbuf[1] = ghosted<double>(c, s, C);
      s.r1f = ghosted<double>(c, s, 6 * c->cb * c->cb);
      CK(cudaMemset(s.r1f + s.bs0 * 6 * c->cb * c->cb, 0, sizeof(double) * (size_t)(s.nbs * 6 * c->cb * c->cb)));
      s.p = s.pbuf[0];
      s.stage = dalloc<double>(c, s.xcells);
      s.st = dalloc<PcgState>(c, 1);
      s.partials = dalloc<double>(c, 4 * s.g.nbo + 64);
      s.d_status = dalloc<int>(c, 4);
      s.d_count = dalloc<unsigned long long>(c, 1);
      CK(cudaMemset(s.st, 0, sizeof(PcgState)));
      CK(cudaMemset(s.d_status, 0, 4 * sizeof(int)));
      // ghost cells of vectors read before their first exchange stay finite
      for (double* v : {s.b, s.x, s.r, s.q, s.z, s.r1, s.pbuf[0], s.pbuf[1], s.kappa})
        CK(cudaMemset(v + s.bs0 * C, 0, sizeof(double) * (size_t)(s.nbs * C)));
    }
    CK(cudaMallocHost(&c->h_state, 2 * sizeof(PcgState)));
    c->gbar = dalloc<unsigned int>(c, 2);
    CK(cudaMemset(c->gbar, 0, 2 * sizeof(unsigned int)));
    CK(cudaDeviceSynchronize());
  });
  if (rc) {
    g_create_error = c->err;
    tmg_destroy(c);
    return rc;
  }
  *out = c;
  return TMG_OK;
}

bool single(const tmg_ctx* c) { return !c->dist(); }

}  // namespace

extern "C" int tmg_setup(tmg_ctx* c, const tmg_mmg_options* o);

// =================================================================== C ABI

extern "C" {

const char* tmg_last_error(const tmg_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

int tmg_create(const tmg_grid* grid, int device, tmg_ctx** out) {
  return create_impl(grid, device, 0, 1, 1, nullptr, out);
}

int tmg_create_slabs(const tmg_grid* grid, int device, int nslabs, tmg_ctx** out) {
  return create_impl(grid, device, 0, nslabs, nslabs, nullptr, out);
}

int tmg_nccl_unique_id(void* id, int bytes) {
  if (!id || bytes < (int)sizeof(ncclUniqueId))
    return set_err(nullptr, TMG_EARG, "tmg_nccl_unique_id: need %d bytes", (int)sizeof(ncclUniqueId));
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess)
    return set_err(nullptr, TMG_ECUDA, "ncclGetUniqueId failed");
  std::memcpy(id, &u, sizeof u);
  return TMG_OK;
}

int tmg_create_dist(const tmg_grid* grid, int device, int rank, int nranks, const void* nccl_id,
                    tmg_ctx** out) {
  if (nranks > 1 && !nccl_id) return set_err(nullptr, TMG_EARG, "tmg_create_dist: null NCCL id");
  return create_impl(grid, device, rank, 1, nranks, nranks > 1 ? nccl_id : nullptr, out);
}

int tmg_partition(const tmg_grid* grid, int nranks, int rank, int64_t* out) {
  if (!grid || !out) return set_err(nullptr, TMG_EARG, "tmg_partition: null argument");
  int64_t cb = 0;
  int rc = check_grid(grid, &cb);
  if (rc) return rc;
  rc = check_partition(grid, nranks);
  if (rc) return rc;
  if (rank < 0 || rank >= nranks)
    return set_err(nullptr, TMG_EARG, "tmg_partition: bad rank %d of %d", rank, nranks);
  const GridParams g = global_params(*grid);
  const Part p = partition(g, rank, nranks);
  out[0] = p.cz0 * g.bz;                        // first fine z layer
  out[1] = p.cz1 * g.bz;                        // end fine z layer
  out[2] = p.b0;                                // first owned brick
  out[3] = p.nbo;                               // owned bricks
  out[4] = p.e0;                                // first owned cc element
  out[5] = p.neo;                               // owned cc elements
  out[6] = p.cz0 * g.bz * g.nx * g.ny;            // first x-fastest cell
  out[7] = (p.cz1 - p.cz0) * g.bz * g.nx * g.ny;  // cells
  out[8] = p.lo;                                // neighbour below
  out[9] = p.hi;                                // neighbour above
  return TMG_OK;
}

int tmg_halo_plan(const tmg_grid* grid, int nranks, int rank, int elem, int64_t* ops,
                  int max_ops) {
  if (!grid || !ops) return -set_err(nullptr, TMG_EARG, "tmg_halo_plan: null argument");
  int64_t cb = 0;
  int rc = check_grid(grid, &cb);
  if (!rc) rc = check_partition(grid, nranks);
  if (rc) return -rc;
  if (rank < 0 || rank >= nranks)
    return -set_err(nullptr, TMG_EARG, "tmg_halo_plan: bad rank %d of %d", rank, nranks);
  const GridParams g = global_params(*grid);
  const std::vector<HaloOp> v =
      halo_ops(partition(g, rank, nranks), rank, elem ? g.ncx * g.ncy : g.nbx * g.nby, elem != 0);
  if ((int)v.size() > max_ops)
    return -set_err(nullptr, TMG_EARG, "tmg_halo_plan: %d operations, buffer holds %d",
                    (int)v.size(), max_ops);
  for (size_t i = 0; i < v.size(); ++i) {
    ops[4 * i + 0] = v[i].send;
    ops[4 * i + 1] = v[i].peer;
    ops[4 * i + 2] = v[i].unit0;
    ops[4 * i + 3] = v[i].units;
  }
  return (int)v.size();
}

void tmg_destroy(tmg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);  // no kernel may outlive its buffers
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->comm) ncclCommDestroy(c->comm);
  for (void* p : c->allocs) cudaFree(p);
  for (auto& pb : c->pool) cudaFree(pb.first);
  if (c->h_state) cudaFreeHost(c->h_state);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int tmg_set_conductivity(tmg_ctx* c, const double* kappa, const tmg_patch* patches, int np) {
  if (!c || !kappa) return set_err(c, TMG_EARG, "tmg_set_conductivity: null argument");
  const int64_t n = host_cells(c);
  for (int64_t i = 0; i < n; ++i)
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
    UP(kappa, kappa);
  });
  if (rc) return rc;
  return finish_problem(c);
}

namespace {
// tmg_tree_gen's segments (7 doubles each: a, b, width), breadth-first.
// Plain IEEE double arithmetic in a fixed order; inputs.tree_segments
// restates it bit for bit.
std::vector<double> tree_segments(const tmg_tree_gen& t, double lx, double ly, double lz) {
  uint64_t st = t.seed ^ 0x9E3779B97F4A7C15ULL;
  auto uni = [&st]() {  // Lcg64::next_uniform (rng.hpp:17-25)
    st = 6364136223846793005ULL * st + 1442695040888963407ULL;
    return (double)(st >> 11) * 0x1.0p-53;
  };
  struct Node {
    double a[3], d[3];
    int level;
  };
  std::vector<Node> q;
  q.push_back(Node{{0.5 * lx, 0.5 * ly, 0.0}, {0.0, 0.0, 1.0}, 0});
  std::vector<double> seg;
  for (size_t n = 0; n < q.size(); ++n) {
    const Node nd = q[n];
    double len = t.length0, w = t.width0;
    for (int k = 0; k < nd.level; ++k) {
      len = len * t.lshrink;
      w = w * t.wshrink;
    }
    const double b[3] = {nd.a[0] + len * nd.d[0], nd.a[1] + len * nd.d[1], nd.a[2] + len * nd.d[2]};
    seg.insert(seg.end(), {nd.a[0], nd.a[1], nd.a[2], b[0], b[1], b[2], w});
    if (nd.level + 1 >= t.depth) continue;
    for (int c = 0; c < 2; ++c) {
      double v[3];
      for (int i = 0; i < 3; ++i) v[i] = nd.d[i] + t.spread * (uni() - 0.5);
      const double nrm = std::sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
      q.push_back(Node{{b[0], b[1], b[2]}, {v[0] / nrm, v[1] / nrm, v[2] / nrm}, nd.level + 1});
    }
  }
  return seg;
}

int set_design_common(tmg_ctx* c, double lo, double hi, int p, const tmg_patch* patches, int np,
                      double vf, int passes, int radius) {
  if (!(lo > 0.0) || !(hi > lo))  // material.cpp:11-12
    return set_err(c, TMG_ECONFIG, "MaterialModel: requires 0 < kappa_lo < kappa_hi");
  if (p < 1) return set_err(c, TMG_ECONFIG, "MaterialModel: penalization p must be >= 1");
  if (!(vf >= 0.0 && vf <= 1.0) || passes < 0 || radius < 0)
    return set_err(c, TMG_ECONFIG, "design generator: need 0 <= vf <= 1, passes, radius >= 0");
  int rc = validate_patches(c, patches, np);
  if (rc) return rc;
  c->patches.clear();
  for (int i = 0; i < np; ++i)
    c->patches.push_back(Patch{patches[i].face, patches[i].u0, patches[i].v0, patches[i].u1,
                               patches[i].v1, patches[i].value});
  return TMG_OK;
}

// generate (x-fastest, whole grid) with `gen`, distribute to the slabs, kappa.
// m_gen > 0: `gen` fills a larger field of m_gen cells of which the context's
// grid is the part from cell `offset` (a bottom slab of a bigger domain).
int generate_design(tmg_ctx* c, double lo, double hi, int p, double* rho_out,
                    const std::function<void(double* rho, double* f, void* scratch)>& gen,
                    int64_t m_gen = 0, int64_t offset = 0) {
  const int rc = guard(c, [&] {
    CK(cudaSetDevice(c->device));
    const tmg_grid& G = c->grid;
    const int64_t m_own = G.nx * G.ny * G.nz;  // the whole design (every rank generates it)
    const int64_t m = m_gen > 0 ? m_gen : m_own;
    double* rho = dalloc<double>(c, m);
    double* f = dalloc<double>(c, m);
    double* scratch = dalloc<double>(c, (int64_t)(gen_scratch_bytes(m) / sizeof(double)) + 1);
    gen(rho, f, scratch);
    CK(cudaGetLastError());
    rho += offset;
    for (Slab& s : c->slabs) {
      launch_to_brick(s.g, c->cb, rho + s.xoff, s.r, c->stream);
      launch_conductivity(s.g, c->cb, s.r, s.kappa, lo, hi, p, c->stream);
      CK(cudaGetLastError());
    }
    if (rho_out)
      CK(cudaMemcpyAsync(rho_out, rho, sizeof(double) * (size_t)m_own, cudaMemcpyDeviceToHost,
                         c->stream));
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, rho - offset);
    dfree(c, f);
    dfree(c, scratch);
  });
  if (rc) return rc;
  return finish_problem(c);
}
}  // namespace

int tmg_set_design_generated(tmg_ctx* c, const tmg_design_gen* gen, double lo, double hi, int p,
                             const tmg_patch* patches, int np, double* rho_out) {
  if (!c || !gen) return set_err(c, TMG_EARG, "tmg_set_design_generated: null argument");
  const int rc = set_design_common(c, lo, hi, p, patches, np, gen->vf, gen->passes, gen->radius);
  if (rc) return rc;
  const tmg_grid& G = c->grid;
  return generate_design(c, lo, hi, p, rho_out, [&](double* rho, double* f, void* scratch) {
    launch_box_filter_design(G.nx, G.ny, G.nz, gen->vf, gen->seed, gen->passes, gen->radius, rho,
                             f, scratch, c->stream);
  });
}

int tmg_set_design_frozen(tmg_ctx* c, double vstar, uint64_t seed, int passes, double lo,
                          double hi, int p, const tmg_patch* patches, int np, double* rho_out) {
  if (!c) return set_err(c, TMG_EARG, "tmg_set_design_frozen: null argument");
  const int rc = set_design_common(c, lo, hi, p, patches, np, vstar, passes, 0);
  if (rc) return rc;
  const tmg_grid& G = c->grid;
  return generate_design(c, lo, hi, p, rho_out, [&](double* rho, double* f, void* scratch) {
    launch_frozen_design(G.nx, G.ny, G.nz, vstar, seed, passes, rho, f, scratch, c->stream);
  });
}

int tmg_set_design_tree(tmg_ctx* c, const tmg_tree_gen* t, double lo, double hi, int p,
                        const tmg_patch* patches, int np, double* rho_out) {
  if (!c || !t) return set_err(c, TMG_EARG, "tmg_set_design_tree: null argument");
  if (t->depth < 1 || t->depth > 12 || !(t->length0 > 0.0) || !(t->width0 > 0.0) ||
      !(t->lshrink > 0.0) || !(t->wshrink > 0.0))
    return set_err(c, TMG_ECONFIG,
                   "tree generator: need 1 <= depth <= 12 and positive lengths, widths, shrinks");
  const int rc = set_design_common(c, lo, hi, p, patches, np, t->vf, t->passes, t->radius);
  if (rc) return rc;
  const tmg_grid& G = c->grid;
  const double dx = t->dom[0] > 0 ? t->dom[0] : G.lx, dy = t->dom[1] > 0 ? t->dom[1] : G.ly,
               dz = t->dom[2] > 0 ? t->dom[2] : G.lz;
  // whole-domain generation (global_n): the field, its filter and its top-k
  // threshold are those of the global design; the context keeps its slab
  int64_t gn[3] = {G.nx, G.ny, G.nz}, offset = 0;
  double ex[3] = {G.lx, G.ly, G.lz};
  if (t->global_n[0] > 0) {
    if (t->global_n[0] != G.nx || t->global_n[1] != G.ny || t->z0 < 0 ||
        t->z0 + G.nz > t->global_n[2] || !(t->dom[0] > 0 && t->dom[1] > 0 && t->dom[2] > 0))
      return set_err(c, TMG_ECONFIG,
                     "tree generator: the context must be the z-slab [z0, z0 + nz) of the "
                     "global_n grid over dom");
    for (int a = 0; a < 3; ++a) {
      gn[a] = t->global_n[a];
      ex[a] = t->dom[a];
    }
    offset = t->z0 * G.nx * G.ny;
  }
  const std::vector<double> seg = tree_segments(*t, dx, dy, dz);
  const int nseg = (int)(seg.size() / 7);
  return generate_design(
      c, lo, hi, p, rho_out,
      [&](double* rho, double* f, void* scratch) {
        double* dseg = dalloc<double>(c, (int64_t)seg.size());
        CK(cudaMemcpyAsync(dseg, seg.data(), sizeof(double) * seg.size(), cudaMemcpyHostToDevice,
                           c->stream));
        launch_tree_design(gn[0], gn[1], gn[2], ex[0], ex[1], ex[2], t->vf, t->seed, t->passes,
                           t->radius, dseg, nseg, t->amp, rho, f, scratch, c->stream);
        CK(cudaStreamSynchronize(c->stream));  // seg host vector outlives the copy
        dfree(c, dseg);
      },
      t->global_n[0] > 0 ? gn[0] * gn[1] * gn[2] : 0, offset);
}

int tmg_set_design(tmg_ctx* c, const double* rho, double lo, double hi, int p,
                   const tmg_patch* patches, int np) {
  if (!c || !rho) return set_err(c, TMG_EARG, "tmg_set_design: null argument");
  if (!(lo > 0.0) || !(hi > lo))  // material.cpp:11-12
    return set_err(c, TMG_ECONFIG, "MaterialModel: requires 0 < kappa_lo < kappa_hi");
  if (p < 1) return set_err(c, TMG_ECONFIG, "MaterialModel: penalization p must be >= 1");
  const int64_t n = host_cells(c);
  for (int64_t i = 0; i < n; ++i) {
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
    UP(rho, r);  // r as scratch for rho (brick layout)
    for (Slab& s : c->slabs) {
      launch_conductivity(s.g, c->cb, s.r, s.kappa, lo, hi, p, c->stream);
      CK(cudaGetLastError());
    }
  });
  if (rc) return rc;
  return finish_problem(c);
}

// interpolate_design's checks (grid.cpp:223-231); uploads the coarse field
int interp_prepare(tmg_ctx* c, const double* lo, const int64_t* nlo, double** dlo) {
  if (!c || !lo || !nlo) return set_err(c, TMG_EARG, "interpolate_design: null argument");
  const int64_t nhi[3] = {c->grid.nx, c->grid.ny, c->grid.nz};
  for (int a = 0; a < 3; ++a)
    if (nlo[a] <= 0 || nhi[a] % nlo[a] != 0)
      return set_err(c, TMG_ECONFIG, "interpolate_design: non-integer refinement factor");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    const int64_t m = nlo[0] * nlo[1] * nlo[2];
    *dlo = dalloc<double>(c, m);
    CK(cudaMemcpyAsync(*dlo, lo, sizeof(double) * (size_t)m, cudaMemcpyHostToDevice, c->stream));
  });
}

int tmg_set_x0_interpolated(tmg_ctx* c, const double* x_lo, const int64_t* n_lo) {
  double* dlo = nullptr;
  int rc = interp_prepare(c, x_lo, n_lo, &dlo);
  if (rc) return rc;
  rc = guard(c, [&] {
    for (Slab& s : c->slabs) {
      launch_interpolate(s.g, c->cb, dlo, n_lo, s.x, c->stream);
      CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(c->stream));
  });
  dfree(c, dlo);
  return rc;
}

int tmg_set_design_interpolated(tmg_ctx* c, const double* rho_lo, const int64_t* n_lo, double lo,
                                double hi, int p, const tmg_patch* patches, int np) {
  if (!(lo > 0.0) || !(hi > lo))  // material.cpp:11-12
    return set_err(c, TMG_ECONFIG, "MaterialModel: requires 0 < kappa_lo < kappa_hi");
  if (p < 1) return set_err(c, TMG_ECONFIG, "MaterialModel: penalization p must be >= 1");
  int rc = validate_patches(c, patches, np);
  if (rc) return rc;
  const int64_t m = n_lo ? n_lo[0] * n_lo[1] * n_lo[2] : 0;
  for (int64_t i = 0; rho_lo && i < m; ++i) {
    double r = 1.0;
    for (int k = 0; k < p; ++k) r *= rho_lo[i];
    if (!(lo + r * (hi - lo) > 0.0))
      return set_err(c, TMG_ECONFIG, "assemble_system: conductivity must be positive");
  }
  double* dlo = nullptr;
  rc = interp_prepare(c, rho_lo, n_lo, &dlo);
  if (rc) return rc;
  c->patches.clear();
  for (int i = 0; i < np; ++i)
    c->patches.push_back(Patch{patches[i].face, patches[i].u0, patches[i].v0, patches[i].u1,
                               patches[i].v1, patches[i].value});
  rc = guard(c, [&] {
    for (Slab& s : c->slabs) {
      launch_interpolate(s.g, c->cb, dlo, n_lo, s.r, c->stream);  // r as scratch for rho
      launch_conductivity(s.g, c->cb, s.r, s.kappa, lo, hi, p, c->stream);
      CK(cudaGetLastError());
    }
  });
  dfree(c, dlo);
  if (rc) return rc;
  return finish_problem(c);
}

int tmg_sensitivity(tmg_ctx* c, const double* rho, double kappa_lo, double kappa_hi, double f0,
                    int p, const double* t, const double* u, double* grad) {
  if (!c || !rho || !t || !u || !grad) return set_err(c, TMG_EARG, "sensitivity: null argument");
  if (!c->have_problem) return set_err(c, TMG_EARG, "sensitivity: no problem set");
  if (!(kappa_lo > 0.0) || !(kappa_hi > kappa_lo))  // material.cpp:11-12
    return set_err(c, TMG_ECONFIG, "MaterialModel: requires 0 < kappa_lo < kappa_hi");
  if (f0 < 0.0) return set_err(c, TMG_ECONFIG, "MaterialModel: f0 must be nonnegative");
  if (p < 1) return set_err(c, TMG_ECONFIG, "MaterialModel: penalization p must be >= 1");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    const int64_t C = cells_per_brick(c);
    UP(rho, r);
    UP(t, pbuf[0]);
    UP(u, pbuf[1]);
    exchange(c, [&](Slab& s) { return (void*)s.pbuf[0]; }, sizeof(double) * C, false);
    exchange(c, [&](Slab& s) { return (void*)s.pbuf[1]; }, sizeof(double) * C, false);
    for (Slab& s : c->slabs) {
      launch_sensitivity(s.g, c->cb, c->patches.data(), (int)c->patches.size(), c->grid.lx,
                         c->grid.ly, c->grid.lz, s.r, s.kappa, s.pbuf[0], s.pbuf[1], kappa_lo,
                         kappa_hi, f0, p, s.q, c->stream);
      CK(cudaGetLastError());
    }
    DOWN(q, grad);
  });
}

int tmg_simp_init(tmg_ctx* c, const tmg_simp_options* o, const tmg_mmg_options* mmg,
                  const double* rho0) {
  if (!c || !o || !mmg) return set_err(c, TMG_EARG, "tmg_simp_init: null argument");
  if (c->dist()) return set_err(c, TMG_ENOTSUP, "the SIMP loop runs on single-slab contexts");
  if (!c->have_problem)
    return set_err(c, TMG_EARG, "tmg_simp_init: set a problem (patches) first");
  if (!(o->volfrac > 0.0 && o->volfrac <= 1.0) || !(o->rmin >= 1.0) || !(o->move > 0.0))
    return set_err(c, TMG_ECONFIG, "simp: need 0 < volfrac <= 1, rmin >= 1, move > 0");
  if (!(o->kappa_lo > 0.0) || !(o->kappa_hi > o->kappa_lo) || o->p < 1)
    return set_err(c, TMG_ECONFIG, "MaterialModel: requires 0 < kappa_lo < kappa_hi, p >= 1");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    auto& S = c->simp;
    const int64_t M = c->M;
    const tmg_grid& G = c->grid;
    for (double** v : {&S.x, &S.xphys, &S.xnew, &S.dc, &S.dv, &S.W, &S.tmp, &S.T, &S.U})
      if (!*v) *v = dalloc<double>(c, M);
    if (!S.part) S.part = dalloc<double>(c, sum_partials_doubles());
    if (!S.scal) S.scal = dalloc<double>(c, 4);
    S.o = *o;
    S.mmg = *mmg;
    S.iter = 0;
    if (rho0)
      CK(cudaMemcpyAsync(S.x, rho0, sizeof(double) * (size_t)M, cudaMemcpyHostToDevice,
                         c->stream));
    else
      launch_fill(S.x, M, o->volfrac, c->stream);
    launch_density_filter(G.nx, G.ny, G.nz, o->rmin, nullptr, nullptr, S.W, 0, c->stream);
    launch_fill(S.tmp, M, 1.0 / (double)M, c->stream);  // d mean(x~) / d x~
    launch_density_filter(G.nx, G.ny, G.nz, o->rmin, S.tmp, S.W, S.dv, 2, c->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    S.on = true;
  });
}

int tmg_simp_step(tmg_ctx* c, tmg_simp_report* rep) {
  if (!c) return set_err(c, TMG_EARG, "null context");
  if (!c->simp.on) return set_err(c, TMG_EARG, "tmg_simp_step: call tmg_simp_init first");
  auto& S = c->simp;
  const auto t0 = std::chrono::steady_clock::now();
  tmg_simp_report r{};
  r.iteration = S.iter;
  const tmg_grid& G = c->grid;
  const int64_t M = c->M;
  auto host_scalar = [&](double* d) {
    double v = 0.0;
    CK(cudaMemcpyAsync(&v, d, sizeof v, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return v;
  };
  int rc = guard(c, [&] {
    CK(cudaSetDevice(c->device));
    Slab& s = c->slabs[0];
    // 1. physical densities and conductivity
    launch_density_filter(G.nx, G.ny, G.nz, S.o.rmin, S.x, S.W, S.xphys, 1, c->stream);
    launch_to_brick(s.g, c->cb, S.xphys, s.r, c->stream);
    launch_conductivity(s.g, c->cb, s.r, s.kappa, S.o.kappa_lo, S.o.kappa_hi, S.o.p, c->stream);
    CK(cudaGetLastError());
    launch_sum(S.xphys, M, S.part, S.scal, c->stream);
    r.volume = host_scalar(S.scal) / (double)M;
  });
  if (rc) return rc;
  if ((rc = finish_problem(c))) return rc;  // mask, faces, coefficients
  tmg_mmg_options mo = S.mmg;
  mo.warm_start = S.iter > 0;  // consecutive designs differ little
  if ((rc = tmg_setup(c, &mo))) return rc;
  r.setup_seconds = c->setup_seconds;
  rc = guard(c, [&] {
    Slab& s = c->slabs[0];
    const size_t bytes = sizeof(double) * (size_t)M;
    // 2. state LS1: b = f vol + Dirichlet lift (fvm.cpp:63-112)
    launch_fill(s.q, M, S.o.source, c->stream);
    launch_boundary(s.g, c->cb, c->patches.data(), (int)c->patches.size(), c->grid.lx,
                    c->grid.ly, c->grid.lz, s.kappa, s.q, s.dmask, s.b, nullptr, c->stream);
    if (S.iter > 0) CK(cudaMemcpyAsync(s.x, S.T, bytes, cudaMemcpyDeviceToDevice, c->stream));
    tmg_report a{};
    solve_device(c, S.o.rtol, S.o.maxit, S.iter > 0, &a, nullptr, nullptr);
    if (!a.converged) {
      set_err(c, TMG_ESOLVER, "simp: state solve did not converge (%d iterations)", a.iterations);
      throw Fail{TMG_ESOLVER};
    }
    r.ls1_iterations = a.iterations;
    r.ls1_seconds = a.solve_seconds;
    CK(cudaMemcpyAsync(S.T, s.x, bytes, cudaMemcpyDeviceToDevice, c->stream));
    launch_sum(S.T, M, S.part, S.scal, c->stream);
    r.cost = host_scalar(S.scal) / (double)M;
    // 3. adjoint LS2: rhs = 1/M (adjoint_rhs, optim.cpp:16-19)
    launch_fill(s.b, M, 1.0 / (double)M, c->stream);
    if (S.iter > 0) CK(cudaMemcpyAsync(s.x, S.U, bytes, cudaMemcpyDeviceToDevice, c->stream));
    solve_device(c, S.o.rtol, S.o.maxit, S.iter > 0, &a, nullptr, nullptr);
    if (!a.converged) {
      set_err(c, TMG_ESOLVER, "simp: adjoint solve did not converge (%d iterations)",
              a.iterations);
      throw Fail{TMG_ESOLVER};
    }
    r.ls2_iterations = a.iterations;
    r.ls2_seconds = a.solve_seconds;
    CK(cudaMemcpyAsync(S.U, s.x, bytes, cudaMemcpyDeviceToDevice, c->stream));
    // 4. sensitivity w.r.t. the physical densities (design-independent source);
    // the solves used s.r, so the densities go to brick layout again (S.xnew
    // is free until the OC update)
    launch_to_brick(s.g, c->cb, S.xphys, S.xnew, c->stream);
    launch_sensitivity(s.g, c->cb, c->patches.data(), (int)c->patches.size(), c->grid.lx,
                       c->grid.ly, c->grid.lz, S.xnew, s.kappa, S.T, S.U, S.o.kappa_lo,
                       S.o.kappa_hi, 0.0, S.o.p, s.q, c->stream);
    launch_from_brick(s.g, c->cb, s.q, S.tmp, c->stream);
    launch_density_filter(G.nx, G.ny, G.nz, S.o.rmin, S.tmp, S.W, S.dc, 2, c->stream);
    CK(cudaGetLastError());
    // 5. OC update: bisection (in log space) on the volume multiplier
    double lo = 1e-40, hi = 1e40;
    for (int it = 0; it < 200 && hi / lo > 1.0 + 1e-10; ++it) {
      const double mid = std::sqrt(lo * hi);
      launch_oc_candidate(S.x, S.dc, S.dv, mid, S.o.move, 0.0, M, S.xnew, c->stream);
      launch_density_filter(G.nx, G.ny, G.nz, S.o.rmin, S.xnew, S.W, S.tmp, 1, c->stream);
      launch_sum(S.tmp, M, S.part, S.scal, c->stream);
      if (host_scalar(S.scal) / (double)M > S.o.volfrac) lo = mid;
      else hi = mid;
    }
    launch_oc_candidate(S.x, S.dc, S.dv, hi, S.o.move, 0.0, M, S.xnew, c->stream);
    launch_maxdiff(S.xnew, S.x, M, S.part, S.scal, c->stream);
    r.change = host_scalar(S.scal);
    std::swap(S.x, S.xnew);
    CK(cudaGetLastError());
  });
  if (rc) return rc;
  ++S.iter;
  r.step_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (rep) *rep = r;
  return TMG_OK;
}

int tmg_simp_download(tmg_ctx* c, double* xphys, double* temperature) {
  if (!c || !c->simp.on) return set_err(c, TMG_EARG, "tmg_simp_download: no SIMP loop");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    auto& S = c->simp;
    const size_t bytes = sizeof(double) * (size_t)c->M;
    if (xphys) {
      launch_density_filter(c->grid.nx, c->grid.ny, c->grid.nz, S.o.rmin, S.x, S.W, S.tmp, 1,
                            c->stream);
      CK(cudaMemcpyAsync(xphys, S.tmp, bytes, cudaMemcpyDeviceToHost, c->stream));
    }
    if (temperature) {
      launch_from_brick(c->slabs[0].g, c->cb, S.T, S.xnew, c->stream);
      CK(cudaMemcpyAsync(temperature, S.xnew, bytes, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

// ------------------------------------------------ reference design loop (MMA)

int tmg_optim_init(tmg_ctx* c, const tmg_optim_options* o, const tmg_mmg_options* mmg,
                   const double* x0) {
  if (!c || !o || !mmg) return set_err(c, TMG_EARG, "tmg_optim_init: null argument");
  if (c->dist()) return set_err(c, TMG_ENOTSUP, "the design loop runs on single-slab contexts");
  if (!c->have_problem)
    return set_err(c, TMG_EARG, "tmg_optim_init: set a problem (patches) first");
  if (!(o->vstar > 0.0 && o->vstar <= 1.0))
    return set_err(c, TMG_ECONFIG, "optimize: vstar must lie in (0, 1]");
  if (!(o->kappa_lo > 0.0) || !(o->kappa_hi > o->kappa_lo))
    return set_err(c, TMG_ECONFIG, "MaterialModel: requires 0 < kappa_lo < kappa_hi");
  if (o->f0 < 0.0) return set_err(c, TMG_ECONFIG, "MaterialModel: f0 must be nonnegative");
  if (o->p < 1) return set_err(c, TMG_ECONFIG, "MaterialModel: penalization p must be >= 1");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    auto& O = c->opt;
    const int64_t M = c->M;
    for (double** v : {&O.x, &O.xp, &O.xp2, &O.xnew, &O.low, &O.upp, &O.grad, &O.xb, &O.T, &O.U})
      if (!*v) *v = dalloc<double>(c, M);
    if (!O.part) O.part = dalloc<double>(c, mma_partials_doubles());
    if (!O.sp) O.sp = dalloc<double>(c, sum_partials_doubles());
    if (!O.scal) O.scal = dalloc<double>(c, 8);
    if (!O.bar) O.bar = dalloc<unsigned int>(c, 2);
    CK(cudaMemsetAsync(O.bar, 0, 2 * sizeof(unsigned int), c->stream));
    O.o = *o;
    O.mmg = *mmg;
    O.iter = 0;
    O.have_T = false;
    if (x0)
      CK(cudaMemcpyAsync(O.x, x0, sizeof(double) * (size_t)M, cudaMemcpyHostToDevice,
                         c->stream));
    else
      launch_fill(O.x, M, o->vstar, c->stream);  // DesignField(grid, vstar)
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    O.on = true;
  });
}

namespace {
// solve_pair (optim.cpp:248-292) on the current design: conductivity, heat
// source, set-up, LS1 and (with_adjoint) LS2. Returns TMG_OK or an error code.
int optim_solve_pair(tmg_ctx* c, bool with_adjoint, tmg_iteration_log* L) {
  auto& O = c->opt;
  const int64_t M = c->M;
  int rc = guard(c, [&] {
    CK(cudaSetDevice(c->device));
    Slab& s = c->slabs[0];
    launch_to_brick(s.g, c->cb, O.x, O.xb, c->stream);
    launch_conductivity(s.g, c->cb, O.xb, s.kappa, O.o.kappa_lo, O.o.kappa_hi, O.o.p, c->stream);
    CK(cudaGetLastError());
  });
  if (rc) return rc;
  if ((rc = finish_problem(c))) return rc;
  tmg_mmg_options mo = O.mmg;
  mo.warm_start = O.o.warm_start && O.iter > 0;
  if ((rc = tmg_setup(c, &mo))) return rc;
  L->setup_seconds = c->setup_seconds;
  const bool warm = O.o.warm_start && O.have_T;
  return guard(c, [&] {
    Slab& s = c->slabs[0];
    const size_t bytes = sizeof(double) * (size_t)M;
    // LS1: b = f(x) vol + Dirichlet lift (assemble_system, fvm.cpp:63-112)
    launch_heat_source(s.g, c->cb, O.xb, s.q, O.o.f0, O.o.p, c->stream);
    launch_boundary(s.g, c->cb, c->patches.data(), (int)c->patches.size(), c->grid.lx,
                    c->grid.ly, c->grid.lz, s.kappa, s.q, s.dmask, s.b, nullptr, c->stream);
    if (warm) CK(cudaMemcpyAsync(s.x, O.T, bytes, cudaMemcpyDeviceToDevice, c->stream));
    tmg_report a{};
    solve_device(c, O.o.rtol, O.o.maxit, warm, &a, nullptr, nullptr);
    if (!a.converged) {
      set_err(c, TMG_ESOLVER, "state solve (LS1) did not converge within %d iterations",
              O.o.maxit);
      throw Fail{TMG_ESOLVER};
    }
    L->ls1_iters = a.iterations;
    L->ls1_seconds = a.solve_seconds;
    CK(cudaMemcpyAsync(O.T, s.x, bytes, cudaMemcpyDeviceToDevice, c->stream));
    launch_sum(O.T, M, O.sp, O.scal, c->stream);
    double sum = 0.0;
    CK(cudaMemcpyAsync(&sum, O.scal, sizeof sum, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    L->cost = sum / (double)M;  // mean_temperature (optim.cpp:10-14)
    if (!with_adjoint) return;
    // LS2: adjoint_rhs (optim.cpp:16-19)
    launch_fill(s.b, M, 1.0 / (double)M, c->stream);
    if (warm) CK(cudaMemcpyAsync(s.x, O.U, bytes, cudaMemcpyDeviceToDevice, c->stream));
    solve_device(c, O.o.rtol, O.o.maxit, warm, &a, nullptr, nullptr);
    if (!a.converged) {
      set_err(c, TMG_ESOLVER, "adjoint solve (LS2) did not converge within %d iterations",
              O.o.maxit);
      throw Fail{TMG_ESOLVER};
    }
    L->ls2_iters = a.iterations;
    L->ls2_seconds = a.solve_seconds;
    CK(cudaMemcpyAsync(O.U, s.x, bytes, cudaMemcpyDeviceToDevice, c->stream));
    O.have_T = true;
  });
}
}  // namespace

int tmg_optim_step(tmg_ctx* c, tmg_iteration_log* log) {
  if (!c) return set_err(c, TMG_EARG, "null context");
  if (!c->opt.on) return set_err(c, TMG_EARG, "tmg_optim_step: call tmg_optim_init first");
  auto& O = c->opt;
  const auto t0 = std::chrono::steady_clock::now();
  tmg_iteration_log L{};
  L.iter = O.iter + 1;
  const int64_t M = c->M;
  auto host = [&](const double* d, int k) {
    double v[8];
    CK(cudaMemcpyAsync(v, d, sizeof(double) * k, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return std::vector<double>(v, v + k);
  };
  int rc = guard(c, [&] {
    CK(cudaSetDevice(c->device));
    launch_sum(O.x, M, O.sp, O.scal, c->stream);
    L.volume = host(O.scal, 1)[0] / (double)M;  // DesignField::volume_fraction
  });
  if (rc) return rc;
  if ((rc = optim_solve_pair(c, true, &L))) return rc;
  rc = guard(c, [&] {
    Slab& s = c->slabs[0];
    // sensitivity (optim.cpp:21-84) with the design-dependent source
    launch_sensitivity(s.g, c->cb, c->patches.data(), (int)c->patches.size(), c->grid.lx,
                       c->grid.ly, c->grid.lz, O.xb, s.kappa, O.T, O.U, O.o.kappa_lo,
                       O.o.kappa_hi, O.o.f0, O.o.p, s.q, c->stream);
    launch_from_brick(s.g, c->cb, s.q, O.grad, c->stream);
    // MMA update with constraint volume - vstar, gradient 1/M (optim.cpp:308-318)
    const MmaParams mp{O.o.move_limit, O.o.asy_init, O.o.asy_incr, O.o.asy_decr, 0.0, 1.0,
                       1.0 / (double)M};
    launch_mma_asymptotes(O.x, O.xp, O.xp2, O.low, O.upp, M, O.iter, mp, c->stream);
    launch_mma_dual(O.x, O.grad, O.low, O.upp, M, L.volume - O.o.vstar, mp, O.part, O.bar,
                    O.scal, c->stream);
    CK(cudaGetLastError());
    const std::vector<double> d = host(O.scal, 3);
    if (d[1] != 0.0) {
      set_err(c, TMG_ESOLVER, "mma_update: multiplier bisection failed, bracket [%g, %g]",
              0.5 * d[2], d[2]);
      throw Fail{TMG_ESOLVER};
    }
    L.lambda = d[0];
    launch_mma_primal(O.x, O.grad, O.low, O.upp, M, O.scal, mp, O.xnew, O.part, O.scal + 3,
                      c->stream);
    CK(cudaGetLastError());
    L.dx_inf = host(O.scal + 3, 1)[0];
    // MmaState: x_prev2 <- x_prev, x_prev <- x; x <- x_new
    double* t = O.xp2;
    O.xp2 = O.xp;
    O.xp = O.x;
    O.x = O.xnew;
    O.xnew = t;
  });
  if (rc) return rc;
  ++O.iter;
  L.step_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (log) *log = L;
  return TMG_OK;
}

int tmg_optim_evaluate(tmg_ctx* c, tmg_iteration_log* log) {
  if (!c) return set_err(c, TMG_EARG, "null context");
  if (!c->opt.on) return set_err(c, TMG_EARG, "tmg_optim_evaluate: call tmg_optim_init first");
  tmg_iteration_log L{};
  L.iter = c->opt.iter;
  int rc = guard(c, [&] {
    CK(cudaSetDevice(c->device));
    launch_sum(c->opt.x, c->M, c->opt.sp, c->opt.scal, c->stream);
    double v = 0.0;
    CK(cudaMemcpyAsync(&v, c->opt.scal, sizeof v, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    L.volume = v / (double)c->M;
  });
  if (rc) return rc;
  if ((rc = optim_solve_pair(c, false, &L))) return rc;
  if (log) *log = L;
  return TMG_OK;
}

int tmg_optim_download(tmg_ctx* c, double* x, double* temperature) {
  if (!c || !c->opt.on) return set_err(c, TMG_EARG, "tmg_optim_download: no design loop");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    auto& O = c->opt;
    const size_t bytes = sizeof(double) * (size_t)c->M;
    if (x) CK(cudaMemcpyAsync(x, O.x, bytes, cudaMemcpyDeviceToHost, c->stream));
    if (temperature) {
      launch_from_brick(c->slabs[0].g, c->cb, O.T, O.xnew, c->stream);
      CK(cudaMemcpyAsync(temperature, O.xnew, bytes, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

int tmg_assemble_rhs(tmg_ctx* c, const double* source, double* rhs_out) {
  if (!c || !rhs_out) return set_err(c, TMG_EARG, "tmg_assemble_rhs: null argument");
  if (!c->have_problem) return set_err(c, TMG_EARG, "tmg_assemble_rhs: no problem set");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    if (source) UP(source, q);
    for (Slab& s : c->slabs) {
      launch_boundary(s.g, c->cb, c->patches.data(), (int)c->patches.size(), c->grid.lx,
                      c->grid.ly, c->grid.lz, s.kappa, source ? s.q : nullptr, s.dmask, s.z,
                      nullptr, c->stream);
      CK(cudaGetLastError());
    }
    DOWN(z, rhs_out);
  });
}

int tmg_setup(tmg_ctx* c, const tmg_mmg_options* o) {
  NvtxRange nvtx("tmg_setup");
  if (!c || !o) return set_err(c, TMG_EARG, "tmg_setup: null argument");
  if (!c->have_problem) return set_err(c, TMG_EARG, "tmg_setup: no problem set");
  const int kind = o->kind;
  const bool hier = kind == TMG_PRECOND_MMG || kind == TMG_PRECOND_TWO_GRID;
  const bool fine_bj = hier && o->fine_blocks == TMG_FINE_BLOCKS_CC;
  if (hier && o->fine_blocks != TMG_FINE_BLOCKS_COARSE_CELL && !fine_bj)
    return set_err(c, TMG_EARG, "fine_blocks must be TMG_FINE_BLOCKS_COARSE_CELL or _CC");
  const bool gen = c->cb == 0;  // generic brick shape (generic.cu)
  const bool want_cc = kind == TMG_PRECOND_BLOCK_JACOBI || fine_bj;
  // exact fine blocks by the generic box block Thomas (generic.cu): every
  // block of a generic shape, and the cc elements the tuned kernels of
  // block_jacobi.cu (8^3, 16^3, 32^3 cells) do not cover
  const int box_kind = (want_cc && (gen || !bj_supported((int)c->cb, c->g.sd))) ? 1
                       : (gen && hier) ? 0 : -1;
  const bool gen_boxes = box_kind >= 0;
  const int gen_kind = box_kind;
  if (gen_boxes && box_plane_cells(c->g, gen_kind) > 4096)
    return set_err(c, TMG_ENOTSUP,
                   "GPU fine blocks of this shape have z planes of %d cells (limit 4096); use "
                   "fine_blocks = coarse_cell or a finer hierarchy",
                   box_plane_cells(c->g, gen_kind));
  if (want_cc || gen_boxes) {
    // the exact per-block factors (E^5 doubles per element) must fit
    size_t fr = 0, tot = 0;
    if (cudaSetDevice(c->device) == cudaSuccess && cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
      double need = 0.0;
      for (const Slab& s : c->slabs)
        need += gen_boxes ? 8.0 * (double)(gen_kind ? s.g.neo : s.g.nbo) * (double)box_doubles(s.g, gen_kind)
                    : 8.0 * (double)s.g.neo * (double)bj_doubles_per_element((int)c->cb, c->g.sd);
      if (need > 0.9 * (double)(fr + c->bytes))
        return set_err(c, TMG_ENOTSUP,
                       "cc-element block factors need %.1f GB (device has %.1f GB); use "
                       "fine_blocks = coarse_cell",
                       need / 1e9, (double)tot / 1e9);
    }
  }
  if (kind < 0 || kind > 4) return set_err(c, TMG_ECONFIG, "make_preconditioner: unknown kind");
  if (hier) {
    const int64_t cells = cells_per_brick(c);
    if (o->num_local_basis > cells)
      return set_err(c, TMG_EARG, "local_spectral_basis: more eigenvectors than cells requested");
    if (o->num_local_basis < 1 || o->num_local_basis > max_lc())
      return set_err(c, TMG_ENOTSUP, "GPU path handles L_c = 1..%d (got %lld)", max_lc(),
                     (long long)o->num_local_basis);
    const int64_t q = (int64_t)c->g.sd * c->g.sd * c->g.sd * o->num_local_basis;
    if (kind == TMG_PRECOND_TWO_GRID && q > 256)
      return set_err(c, TMG_ENOTSUP, "GPU two_grid handles sd^3*L_c <= 256 (got %lld)",
                     (long long)q);
    if (kind == TMG_PRECOND_MMG && o->num_cc_basis > q)
      return set_err(c, TMG_EARG,
                     "coarse_coarse_basis: more eigenvectors than coarse basis functions");
    if (kind == TMG_PRECOND_MMG && o->num_cc_basis < 1)
      return set_err(c, TMG_EARG, "num_cc_basis must be >= 1");
    if (kind == TMG_PRECOND_MMG && q > 64 && !coarse_large_supported((int)q, (int)o->num_cc_basis))
      return set_err(c, TMG_ENOTSUP,
                     "GPU coarse level handles sd^3*L_c <= 64, or a multiple of 64 up to 4096 with "
                     "num_cc_basis <= 20 (got %lld, %lld)",
                     (long long)q, (long long)o->num_cc_basis);
    if (o->smoother_sweeps < 0 || o->smoother_sweeps > 64)
      return set_err(c, TMG_ECONFIG, "MmgOptions: smoother_sweeps must lie in [0, 64] (got %d)",
                     o->smoother_sweeps);
  }
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    free_setup(c);  // the current bases (if any) move to phi_keep
    // warm start: the last set-up's bases seed the local eigensolver
    std::vector<double*> phi_prev(c->slabs.size(), nullptr);
    const bool warm = hier && o->warm_start && c->lc_keep == (int)o->num_local_basis;
    for (size_t k = 0; k < c->slabs.size(); ++k) {
      phi_prev[k] = warm ? c->slabs[k].phi_keep : nullptr;
      if (!warm) dfree_null(c, c->slabs[k].phi_keep);
      c->slabs[k].phi_keep = nullptr;
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, c->stream));
    const int64_t C = cells_per_brick(c);
    for (Slab& s : c->slabs) CK(cudaMemsetAsync(s.d_status, 0, 4 * sizeof(int), c->stream));
    if (kind == TMG_PRECOND_JACOBI) {
      for (Slab& s : c->slabs) {
        s.dinv = owned<double>(c, s, C);
        launch_apply(s.g, c->cb, s.coef, nullptr, nullptr, s.dinv, c->stream);
        CK(cudaGetLastError());
      }
    } else if (kind == TMG_PRECOND_BLOCK_JACOBI && box_kind == 1) {
      const int64_t per = box_doubles(c->g, 1);
      for (Slab& s : c->slabs) {
        s.Gbj = owned_e<double>(c, s, per);
        s.ybj = owned<double>(c, s, C);
        double* w = dalloc<double>(c, box_factor_work_doubles(s.g, 1));
        launch_box_factor(s.g, 1, s.coef, s.Gbj + s.g.e0 * per, s.d_status, w, c->stream);
        CK(cudaGetLastError());
        dfree(c, w);
      }
    } else if (kind == TMG_PRECOND_BLOCK_JACOBI) {
      const int64_t per = bj_doubles_per_element(c->cb, c->g.sd);
      for (Slab& s : c->slabs) {
        s.Gbj = owned_e<double>(c, s, per);
        if (bj_apply_kernels((int)c->cb, c->g.sd) > 1) s.ybj = owned<double>(c, s, C);
        const int64_t wd = bj_factor_work_doubles((int)c->cb, c->g.sd, s.g.neo);
        double* w = wd ? dalloc<double>(c, wd) : nullptr;
        launch_bj_factor(s.g, (int)c->cb, s.coef, s.Gbj + s.g.e0 * per, s.d_status, w, c->stream);
        CK(cudaGetLastError());
        if (w) dfree(c, w);
      }
    } else if (hier) {
      c->lc = (int)o->num_local_basis;
      // two_grid: R_cc = I (build_two_grid, solver.cpp:401-420)
      c->lcc = kind == TMG_PRECOND_TWO_GRID
                   ? (int)(c->g.sd * c->g.sd * c->g.sd * o->num_local_basis)
                   : (int)o->num_cc_basis;
      c->g.lc = c->lc;
      c->g.lcc = c->lcc;
      const int64_t q = (int64_t)c->g.sd * c->g.sd * c->g.sd * c->lc;
      const int lc = c->lc, lcc = c->lcc;
      for (Slab& s : c->slabs) {
        s.g.lc = lc;
        s.g.lcc = lcc;
        s.phi = ghosted<double>(c, s, lc * C);
        s.evals = owned<double>(c, s, lc);
        s.eig_iters = owned<int>(c, s, 1);
        if (box_kind >= 0) {  // box factors of the cc elements or of the bricks
          if (box_kind == 1) s.Gbj = owned_e<double>(c, s, box_doubles(c->g, 1));
          else s.Gf = owned<double>(c, s, box_doubles(c->g, 0));
          s.ybj = owned<double>(c, s, C);
        } else if (fine_bj) {
          s.Gbj = owned_e<double>(c, s, bj_doubles_per_element(c->cb, c->g.sd));
          if (bj_apply_kernels((int)c->cb, c->g.sd) > 1) s.ybj = owned<double>(c, s, C);
        } else {
          plan_fine_factors(c, s);
          s.Gf = dalloc<double>(c, std::max<int64_t>(s.nslots, 1) * thomas_doubles_per_brick(c->cb));
        }
        if (fine_bj || o->smoother_sweeps != 1 || gen) {  // unfused V-cycles
          s.r2 = ghosted<double>(c, s, C);
          s.t2 = ghosted<double>(c, s, C);
        }
        s.Ac = owned<double>(c, s, 7 * lc * lc);
        s.Bc = owned<double>(c, s, lc * lc);
        s.Rcc = ghosted_e<double>(c, s, lcc * q);
        s.cc_evals = owned_e<double>(c, s, lcc);
        s.Winv = owned_e<double>(c, s, q * q);
        for (double** v : {&s.rc, &s.rc0, &s.ec, &s.rc1, &s.tc}) {
          *v = ghosted<double>(c, s, lc);
          CK(cudaMemsetAsync(*v + s.bs0 * lc, 0, sizeof(double) * (size_t)(s.nbs * lc), c->stream));
        }
      }
      c->n_cc = c->g.ncc * lcc;
      c->rcc = dalloc<double>(c, c->n_cc);
      c->ecc = dalloc<double>(c, c->n_cc);
      // TMG_SETUP_PROFILE=1: per-phase device times on stderr (diagnostics only)
      const bool sprof = getenv("TMG_SETUP_PROFILE") != nullptr;
      cudaEvent_t ph[12];
      int nph = 0;
      const char* phname[12];
      auto mark = [&](const char* name) {
        nvtxMarkA(name);  // NVTX: set-up phase `name` enqueued
        if (!sprof) return;
        CK(cudaEventCreate(&ph[nph]));
        CK(cudaEventRecord(ph[nph], c->stream));
        phname[nph++] = name;
      };
      mark("alloc");
      const double tol = o->eig_tol > 0 ? o->eig_tol : 1e-9;  // residual / ||B|| (DESIGN.md §4 set-up)
      const int degree = o->eig_degree > 0 ? o->eig_degree : 32;
      const int max_outer = o->eig_max_outer > 0 ? o->eig_max_outer : 60;
      for (size_t k = 0; k < c->slabs.size(); ++k) {
        Slab& s = c->slabs[k];
        if (gen) {
          const int64_t wd = g_local_basis_scratch_doubles(s.g);
          double* w = wd ? dalloc<double>(c, wd) : nullptr;
          launch_g_local_basis(s.g, s.kappa, phi_prev[k], s.phi, s.evals, s.eig_iters, tol,
                               degree, max_outer, w, c->stream);
          if (w) dfree(c, w);  // stream-ordered reuse only
        } else {
          // bricks of one conductivity inside get their bases in closed form
          // (separable modes, k_local_basis_uniform); the eigensolver runs on
          // the others. TMG_EIG_SHARE=0: every brick through the eigensolver
          const char* es = getenv("TMG_EIG_SHARE");
          const bool share = !(es && es[0] == '0');
          std::vector<int> flag((size_t)s.g.nbo, 0);
          int* dflag = dalloc<int>(c, s.g.nbo);
          if (share) {
            launch_uniform_inside(s.g, c->cb, s.kappa, dflag, c->stream);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(flag.data(), dflag, sizeof(int) * flag.size(),
                               cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
          }
          std::vector<int64_t> list;
          for (int64_t i = 0; i < s.g.nbo; ++i)
            if (!flag[(size_t)i]) list.push_back(s.g.b0 + i);
          int64_t* dlist = dalloc<int64_t>(c, (int64_t)list.size());
          CK(cudaMemcpyAsync(dlist, list.data(), sizeof(int64_t) * list.size(),
                             cudaMemcpyHostToDevice, c->stream));
          launch_local_basis(s.g, c->cb, s.kappa, phi_prev[k], s.phi, s.evals, s.eig_iters, tol,
                             degree, max_outer, dlist, (int64_t)list.size(), c->stream);
          if (share)
            launch_local_basis_uniform(s.g, c->cb, s.kappa, dflag, s.phi, s.evals, s.eig_iters,
                                       c->stream);
          CK(cudaGetLastError());
          CK(cudaStreamSynchronize(c->stream));  // list lives on the host stack
          dfree(c, dlist);
          dfree(c, dflag);
        }
      }
      CK(cudaGetLastError());
      for (double*& pp : phi_prev) dfree_null(c, pp);  // stream-ordered reuse only
      XCH(phi, sizeof(double) * lc * C, false);
      for (Slab& s : c->slabs) {  // after the exchange: ghost bricks' faces too
        if (gen) break;           // read only by the templated boundary-form kernels
        s.phif = ghosted<double>(c, s, 6 * lc * c->cb * c->cb);
        launch_phi_faces(s.g, c->cb, s.phi, s.phif, s.bs0, s.nbs, c->stream);
      }
      CK(cudaGetLastError());
      mark("local_basis");
      for (Slab& s : c->slabs) {
        if (gen) launch_g_coarse_blocks(s.g, s.kappa, s.dmask, s.coef, s.phi, s.Ac, s.Bc, c->stream);
        else launch_coarse_blocks(s.g, c->cb, s.kappa, s.dmask, s.phi, s.Ac, s.Bc, c->stream);
      }
      CK(cudaGetLastError());
      mark("coarse_blocks");
      int* cc_iters = nullptr;
      if (sprof && q > 64) {
        cc_iters = dalloc<int>(c, 1);
        CK(cudaMemsetAsync(cc_iters, 0, sizeof(int), c->stream));
      }
      double* large_work = nullptr;
      if (q > 64) {
        int64_t wd = 0;
        for (Slab& s : c->slabs)
          wd = std::max(wd, coarse_large_work_doubles((int)q, s.g.neo, lcc));
        if (wd) large_work = dalloc<double>(c, wd);
      }
      for (Slab& s : c->slabs) {
        if (kind == TMG_PRECOND_TWO_GRID) launch_cc_identity(s.g, s.Rcc, s.cc_evals, c->stream);
        else if (q <= 64) launch_cc_basis(s.g, s.Ac, s.Bc, s.Rcc, s.cc_evals, c->stream);
        else  // Winv's storage holds the shifted inverses until the smoother overwrites it
          launch_cc_basis_large(s.g, s.Ac, s.Bc, s.Winv, large_work, s.Rcc, s.cc_evals,
                                s.d_status + 3, cc_iters, 1e-10, 100, c->stream);
      }
      if (cc_iters) {
        int it = 0;
        CK(cudaMemcpyAsync(&it, cc_iters, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        fprintf(stderr, "[setup] cc subspace iterations (max over elements): %d\n", it);
        dfree(c, cc_iters);
      }
      CK(cudaGetLastError());
      XCH(Rcc, sizeof(double) * lcc * q, true);
      mark("cc_basis");
      for (Slab& s : c->slabs) {
        if (q <= 64) launch_coarse_smoother(s.g, s.Ac, s.Winv, s.d_status + 1, c->stream);
        else launch_coarse_smoother_large(s.g, s.Ac, s.Winv, large_work, s.d_status + 1, c->stream);
      }
      dfree_null(c, large_work);
      CK(cudaGetLastError());
      mark("coarse_smoother");
      for (Slab& s : c->slabs) {
        if (box_kind >= 0) {
          const int bk = box_kind;
          const int64_t per = box_doubles(s.g, bk);
          double* G = bk ? s.Gbj + s.g.e0 * per : s.Gf + s.g.b0 * per;
          double* w = dalloc<double>(c, box_factor_work_doubles(s.g, bk));
          launch_box_factor(s.g, bk, s.coef, G, s.d_status, w, c->stream);
          dfree(c, w);
        } else if (fine_bj) {
          const int64_t per = bj_doubles_per_element(c->cb, c->g.sd);
          const int64_t wd = bj_factor_work_doubles((int)c->cb, c->g.sd, s.g.neo);
          double* w = wd ? dalloc<double>(c, wd) : nullptr;
          launch_bj_factor(s.g, (int)c->cb, s.coef, s.Gbj + s.g.e0 * per, s.d_status, w, c->stream);
          if (w) dfree(c, w);
        } else {
          launch_thomas_factor(s.g, c->cb, s.kappa, s.dmask, s.flist, s.nslots, s.Gf, s.d_status,
                               c->stream);
        }
      }
      CK(cudaGetLastError());
      mark("thomas_factor");
      // A_cc. Several cc-element z-planes and a large n_cc (or
      // TMG_ACC_PLANES=1): block Thomas over the planes (acc_planes.cu);
      // otherwise the dense inverse (replicated row blocks when partitioned).
      // Partitioned contexts assemble their own planes, all-gather the plane
      // blocks and couplings, and every rank factors and applies the whole
      // (replicated) plane solve after the r_cc all-gather.
      // Default by a per-V-cycle cost model (5 TB/s streaming, 6 us per
      // dependent plane step): the plane solve streams 2 ncz symmetric P x P
      // tiles in sequence; the dense inverse streams its symmetric tiles
      // (single slab) or each rank's n_cc / N full rows. A dense inverse
      // above 40 GB is not built. TMG_ACC_PLANES=0/1 overrides.
      const char* ap = getenv("TMG_ACC_PLANES");
      const double bw = 5e12, step = 6e-6, ncd = (double)c->n_cc;
      const double Pd = (double)(c->g.ncx * c->g.ncy * lcc);
      const double t_planes = 2.0 * (double)c->g.ncz * (Pd * Pd * 4.0 / bw + step);
      const double t_dense = (c->dist() ? ncd * ncd * 8.0 / (double)c->total : ncd * ncd * 4.0) / bw;
      const bool planes = c->g.ncz >= 2 && (ap ? ap[0] == '1'
                                                   : (t_planes < t_dense || ncd * ncd * 8.0 > 40e9));
      double* work = nullptr;
      if (planes) {
        GridParams g0 = c->slabs[0].g;  // global dims; the planes factor covers all elements
        g0.ncz = c->g.ncz;
        g0.ncc = c->g.ncc;
        const int64_t P = g0.ncx * g0.ncy * lcc;
        // partitioned contexts: every slab keeps only its row block of the
        // plane inverses (launch_acc_rows_solve; TMG_ACC_ROWS=0/1 overrides
        // the default of >= 4 slabs)
        const char* arow = getenv("TMG_ACC_ROWS");
        const bool rows = c->dist() && c->total > 1 && P % c->total == 0 &&
                          (arow ? arow[0] == '1' : c->total >= 4);
        double* Gd = dalloc<double>(c, g0.ncz * P * P);
        const int64_t ts = sym_tiles_doubles(P);
        c->accP = dalloc<double>(c, acc_planes_doubles(g0) - (rows ? g0.ncz * ts : 0));
        double* T = rows ? nullptr : c->accP;
        double* C = c->accP + (rows ? 0 : g0.ncz * ts);
        double* wv = C + g0.ncc * lcc * lcc;
        for (size_t k = 0; k < c->slabs.size(); ++k)
          launch_acc_assemble_planes(c->slabs[k].g, c->slabs[k].Ac, c->slabs[k].Rcc, Gd, C, c->stream,
                                     k == 0);
        CK(cudaGetLastError());
        if (c->nccl()) {
          const Slab& s = c->slabs[0];
          const int64_t nxy = g0.ncx * g0.ncy, k0 = s.g.e0 / nxy, nk = s.g.neo / nxy;
          NK(ncclAllGather(Gd + k0 * P * P, Gd, (size_t)(nk * P * P), ncclDouble, c->comm, c->stream));
          NK(ncclAllGather(C + s.g.e0 * lcc * lcc, C, (size_t)(s.g.neo * lcc * lcc), ncclDouble, c->comm,
                           c->stream));
        }
        mark("acc_assemble");
        work = dalloc<double>(c, dense_inverse_work_doubles(P));
        acc_planes_factor(g0, Gd, C, T, work, c->slabs[0].d_status + 2, c->stream);
        CK(cudaGetLastError());
        if (rows) {  // each slab's rows of every dense plane inverse
          const int64_t nr = P / c->total;
          for (Slab& s : c->slabs) {
            s.accRows = dalloc<double>(c, g0.ncz * nr * P);
            for (int64_t k = 0; k < g0.ncz; ++k)
              CK(cudaMemcpyAsync(s.accRows + k * nr * P, Gd + k * P * P + (int64_t)s.id * nr * P,
                                 sizeof(double) * (size_t)(nr * P), cudaMemcpyDeviceToDevice,
                                 c->stream));
          }
        }
        mark("acc_planes");
        c->symvP = dalloc<double>(c, sym_partials_doubles(P));
        c->planes = AccPlanesRef{T, C, wv};
        c->acc_planes = true;
        c->acc_rows = rows;
        CK(cudaStreamSynchronize(c->stream));
        dfree(c, Gd);
      } else {
        // every slab assembles its rows of the one dense matrix
        double* Acc = dalloc<double>(c, c->n_cc * c->n_cc);
        for (Slab& s : c->slabs) launch_acc_assemble(s.g, s.Ac, s.Rcc, Acc, c->stream);
        CK(cudaGetLastError());
        if (c->nccl()) {
          const Slab& s = c->slabs[0];
          const int64_t rows = s.g.neo * lcc;
          NK(ncclAllGather(Acc + s.g.e0 * lcc * c->n_cc, Acc, (size_t)(rows * c->n_cc),
                           ncclDouble, c->comm, c->stream));
        }
        mark("acc_assemble");
        work = dalloc<double>(c, dense_inverse_work_doubles(c->n_cc));
        dense_spd_inverse(Acc, c->n_cc, work, c->slabs[0].d_status + 2, c->stream);
        CK(cudaGetLastError());
        mark("acc_inverse");
        if (!c->dist()) {
          c->AccT = dalloc<double>(c, sym_tiles_doubles(c->n_cc));
          c->symvP = dalloc<double>(c, sym_partials_doubles(c->n_cc));
          pack_sym_tiles(Acc, c->n_cc, c->AccT, c->stream);
          CK(cudaGetLastError());
          mark("pack_tiles");
          CK(cudaStreamSynchronize(c->stream));
          dfree(c, Acc);
        } else {
          c->Ainv = Acc;  // row blocks applied per slab (launch_gemv_rows)
        }
      }
      CK(cudaStreamSynchronize(c->stream));
      for (int i = 1; i < nph; ++i) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, ph[i - 1], ph[i]));
        fprintf(stderr, "[setup] %-16s %9.3f ms\n", phname[i], t);
      }
      for (int i = 0; i < nph; ++i) cudaEventDestroy(ph[i]);
      dfree(c, work);
    }
    CK(cudaEventRecord(e1, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaGetLastError());
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    c->setup_seconds = 1e-3 * ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (Slab& s : c->slabs) {
      int status[4];
      CK(cudaMemcpy(status, s.d_status, sizeof status, cudaMemcpyDeviceToHost));
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
    }
    c->kind = kind;
    c->fine_bj = fine_bj ? 1 : 0;
    c->box_kind = box_kind;
    c->nu = hier ? o->smoother_sweeps : 1;
    c->have_setup = true;
    build_graph(c, 4);
  });
}

int tmg_upload_rhs(tmg_ctx* c, const double* b) {
  if (!c || !b) return set_err(c, TMG_EARG, "tmg_upload_rhs: null argument");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    UP(b, b);
  });
}

int tmg_upload_x0(tmg_ctx* c, const double* x0) {
  if (!c || !x0) return set_err(c, TMG_EARG, "tmg_upload_x0: null argument");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    UP(x0, x);
  });
}

int tmg_solve_resident(tmg_ctx* c, double rtol, int maxit, int use_x0, tmg_report* rep) {
  NvtxRange nvtx("tmg_solve_resident");
  if (!c) return set_err(c, TMG_EARG, "null context");
  if (maxit < 0) return set_err(c, TMG_EARG, "pcg: negative max_iterations");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    solve_device(c, rtol, maxit, use_x0, rep, nullptr, nullptr);
  });
}

int tmg_solve_resident_ex(tmg_ctx* c, double rtol, int maxit, int use_x0, int flags,
                          tmg_report* rep) {
  NvtxRange nvtx("tmg_solve_resident");
  if (!c) return set_err(c, TMG_EARG, "null context");
  if (maxit < 0) return set_err(c, TMG_EARG, "pcg: negative max_iterations");
  tmg_report local{};
  const int rc = guard(c, [&] {
    CK(cudaSetDevice(c->device));
    solve_device(c, rtol, maxit, use_x0, &local, nullptr, nullptr);
    if (!(flags & TMG_SOLVE_TRUE_RESIDUAL) || !local.converged || local.status == kStatusZeroRhs)
      return;
    // Residual replacement. A use_x0 solve with max_iterations = 0 runs only
    // the init kernel: r = b - A x exactly as pcg() forms it for x0
    // (solver.cpp:515-521), i.e. the TRUE residual of the resident x.
    int total = local.iterations;
    double secs = local.solve_seconds, prev = 0.0;
    for (int k = 0;; ++k) {
      tmg_report chk{};
      solve_device(c, rtol, 0, 1, &chk, nullptr, nullptr);
      secs += chk.solve_seconds;
      const double tr = chk.final_relative_residual;
      local.final_relative_residual = tr;
      if (tr <= rtol) {
        local.converged = 1;
        local.status = kStatusConverged;
        break;
      }
      // no progress: the FP64 floor eps |A||x| / |b| of the problem
      // is above rtol; further restarts cannot go lower
      if ((k > 0 && tr > 0.5 * prev) || k == 4 || total >= maxit) {
        local.converged = 0;
        local.status = (k > 0 && tr > 0.5 * prev) ? kStatusFloor : kStatusMaxIt;
        break;
      }
      prev = tr;
      tmg_report r2{};
      solve_device(c, rtol, maxit - total, 1, &r2, nullptr, nullptr);
      total += r2.iterations;
      secs += r2.solve_seconds;
      local.restarts = k + 1;
      if (!r2.converged) {  // max iterations inside a restart
        local.converged = 0;
        local.status = r2.status;
        local.final_relative_residual = r2.final_relative_residual;
        break;
      }
    }
    local.iterations = total;
    local.solve_seconds = secs;
  });
  if (rep) *rep = local;
  return rc;
}

int tmg_apply_operator_abs(tmg_ctx* c, const double* x, double* y) {
  if (!c || !x || !y) return set_err(c, TMG_EARG, "tmg_apply_operator_abs: null argument");
  if (!c->have_problem) return set_err(c, TMG_EARG, "apply: no problem set");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    UP(x, p);
    XCH(p, sizeof(double) * cells_per_brick(c), false);
    for (Slab& s : c->slabs) {
      launch_apply_abs(s.g, c->cb, s.coef, s.p, s.q, c->stream);
      CK(cudaGetLastError());
    }
    DOWN(q, y);
  });
}

int tmg_download_solution(tmg_ctx* c, double* x) {
  if (!c || !x) return set_err(c, TMG_EARG, "tmg_download_solution: null argument");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    DOWN(x, x);
  });
}

int tmg_pcg(tmg_ctx* c, const double* b, const double* x0, double rtol, int maxit, double* x_out,
            double* history, tmg_report* rep) {
  NvtxRange nvtx("tmg_pcg");
  if (!c || !b || !x_out) return set_err(c, TMG_EARG, "pcg: null argument");
  if (maxit < 0) return set_err(c, TMG_EARG, "pcg: negative max_iterations");
  tmg_report local{};
  const int rc = guard(c, [&] {
    CK(cudaSetDevice(c->device));
    UP(b, b);
    if (x0) UP(x0, x);
    solve_device(c, rtol, maxit, x0 ? 1 : 0, &local, nullptr, nullptr);
    DOWN(x, x_out);
    if (history && local.iterations > 0)
      CK(cudaMemcpy(history, c->slabs[0].history, sizeof(double) * (size_t)local.iterations,
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
    UP(x, p);
    XCH(p, sizeof(double) * cells_per_brick(c), false);
    for (Slab& s : c->slabs) {
      launch_apply(s.g, c->cb, s.coef, s.p, s.q, nullptr, c->stream);
      CK(cudaGetLastError());
    }
    DOWN(q, y);
  });
}

int tmg_apply_preconditioner(tmg_ctx* c, const double* rin, double* zout) {
  if (!c || !rin || !zout) return set_err(c, TMG_EARG, "Preconditioner::apply: null argument");
  if (!c->have_setup) return set_err(c, TMG_EARG, "apply: no preconditioner set up");
  return guard(c, [&] {
    CK(cudaSetDevice(c->device));
    ensure_history(c, 1);
    init_states(c, 0.0, 1);
    UP(rin, r);
    enqueue_precond_init(c);
    CK(cudaGetLastError());
    DOWN(z, zout);
  });
}

int tmg_get_sizes(tmg_ctx* c, int64_t* s) {
  if (!c || !s) return set_err(c, TMG_EARG, "null argument");
  s[0] = c->M;
  s[1] = c->g.nb;
  s[2] = c->g.nb * c->lc;
  s[3] = c->g.ncc;
  s[4] = c->g.ncc * c->lcc;
  s[5] = cells_per_brick(c);
  return TMG_OK;
}

int tmg_get_fine_factor_slots(tmg_ctx* c, int64_t* slots, int64_t* bricks) {
  if (!c || !slots || !bricks) return set_err(c, TMG_EARG, "null argument");
  *slots = 0;
  *bricks = 0;
  for (const Slab& s : c->slabs) {
    *slots += s.nslots;
    *bricks += s.g.nbo;
  }
  return TMG_OK;
}

int tmg_get_local_bases(tmg_ctx* c, double* phi, double* evals, int* iters) {
  if (!c || !c->have_setup || !hierarchical(c))
    return set_err(c, TMG_EARG, "no MMG hierarchy set up");
  if (!single(c)) return set_err(c, TMG_ENOTSUP, "hierarchy getters need a single-slab context");
  return guard(c, [&] {
    const Slab& s = c->slabs[0];
    const int64_t C = cells_per_brick(c);
    if (phi)
      CK(cudaMemcpy(phi, s.phi, sizeof(double) * (size_t)(c->g.nb * c->lc * C),
                    cudaMemcpyDeviceToHost));
    if (evals)
      CK(cudaMemcpy(evals, s.evals, sizeof(double) * (size_t)(c->g.nb * c->lc),
                    cudaMemcpyDeviceToHost));
    if (iters)
      CK(cudaMemcpy(iters, s.eig_iters, sizeof(int) * (size_t)c->g.nb, cudaMemcpyDeviceToHost));
  });
}

int tmg_get_coarse_operator(tmg_ctx* c, double* ac) {
  if (!c || !c->have_setup || !hierarchical(c) || !ac)
    return set_err(c, TMG_EARG, "no MMG hierarchy set up");
  if (!single(c)) return set_err(c, TMG_ENOTSUP, "hierarchy getters need a single-slab context");
  return guard(c, [&] {
    const GridParams& g = c->g;
    const int L = c->lc;
    std::vector<double> blk((size_t)(g.nb * 7 * L * L));
    CK(cudaMemcpy(blk.data(), c->slabs[0].Ac, sizeof(double) * blk.size(),
                  cudaMemcpyDeviceToHost));
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
  if (!c || !c->have_setup || !hierarchical(c) || !rcc)
    return set_err(c, TMG_EARG, "no MMG hierarchy set up");
  if (!single(c)) return set_err(c, TMG_ENOTSUP, "hierarchy getters need a single-slab context");
  return guard(c, [&] {
    const GridParams& g = c->g;
    const int64_t q = (int64_t)g.sd * g.sd * g.sd * c->lc, nc = g.nb * c->lc;
    std::vector<double> R((size_t)(g.ncc * c->lcc * q));
    CK(cudaMemcpy(R.data(), c->slabs[0].Rcc, sizeof(double) * R.size(), cudaMemcpyDeviceToHost));
    std::fill(rcc, rcc + g.ncc * c->lcc * nc, 0.0);
    for (int64_t e = 0; e < g.ncc; ++e) {
      const int64_t ei = e % g.ncx, ej = (e / g.ncx) % g.ncy, ek = e / (g.ncx * g.ncy);
      for (int64_t ch = 0; ch < (int64_t)g.sd * g.sd * g.sd; ++ch) {
        const int64_t di = ch % g.sd, dj = (ch / g.sd) % g.sd, dk = ch / (g.sd * g.sd);
        const int64_t I = (ei * g.sd + di) + g.nbx * ((ej * g.sd + dj) + g.nby * (ek * g.sd + dk));
        for (int k = 0; k < c->lcc; ++k)
          for (int a = 0; a < c->lc; ++a)
            rcc[(e * c->lcc + k) * nc + I * c->lc + a] =
                R[(size_t)((e * c->lcc + k) * q + ch * c->lc + a)];
      }
    }
  });
}

int tmg_profile_solve(tmg_ctx* c, double rtol, int maxit, double* ms_total, int* count) {
  if (!c || !ms_total || !count) return set_err(c, TMG_EARG, "null argument");
  if (!single(c))
    return set_err(c, TMG_ENOTSUP, "per-kernel profiling needs a single-slab context");
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
