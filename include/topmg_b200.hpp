// topmg_b200.hpp — header-only C++ drop-in for the reference's solver
// interface (proj/core/include/topmg/solver.hpp), over the C ABI
// topmg_b200.h. Include it from code that already includes the reference's
// "topmg/solver.hpp" and link libtopmg_b200.so; see INTEGRATION.md.
//
//   auto m = topmg_b200::make_preconditioner(PrecondKind::Mmg, sys, hgrid, opts);
//   PcgResult r = topmg_b200::pcg(sys.matrix, sys.rhs, *m, {1e-8, 10000});
//
// topmg_b200::pcg runs the whole PCG on the GPU (same stopping rule, report
// and exceptions as topmg::pcg, solver.cpp:483-575). The preconditioner object
// is also a plain topmg::Preconditioner: apply() runs one device V-cycle with
// host copies, so the reference's own topmg::pcg accepts it unchanged.
#pragma once

#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "topmg/solver.hpp"
#include "topmg_b200.h"

namespace topmg_b200 {

inline void check(int rc, const tmg_ctx* c) {
  if (rc == TMG_OK) return;
  const std::string msg = tmg_last_error(c);
  switch (rc) {
    case TMG_ECONFIG: throw topmg::ConfigError(msg);
    case TMG_ESOLVER: throw topmg::SolverError(msg);
    case TMG_EARG: throw std::invalid_argument(msg);
    default: throw std::runtime_error("topmg_b200: " + msg);
  }
}

// A GPU-resident operator + preconditioner for one assembled system.
class GpuMmgPreconditioner final : public topmg::Preconditioner {
 public:
  // make_preconditioner (solver.cpp:462-481) for all five kinds. The operator
  // is rebuilt matrix-free from system.kappa and system.boundary
  // (fvm.hpp:20-26); system.matrix is not copied to the device. fine_blocks
  // selects the Mmg / TwoGrid fine smoother partition: the default
  // TMG_FINE_BLOCKS_CC is the reference's own (build_mmg's fine_blocks_by_cc,
  // solver.cpp:353-361; cc elements of 8^3, 16^3 or 32^3 cells), so this
  // factory is a faithful drop-in for topmg::make_preconditioner;
  // TMG_FINE_BLOCKS_COARSE_CELL opts into the fast GPU partition (one block
  // per coarse cell; fewer bytes per V-cycle, a few more
  // iterations: INTEGRATION.md).
  GpuMmgPreconditioner(topmg::PrecondKind kind, const topmg::AssembledSystem& system,
                       const topmg::HierarchicalGrid& hgrid, const topmg::MmgOptions& opts = {},
                       int device = 0, int fine_blocks = TMG_FINE_BLOCKS_CC)
      : kind_(kind), n_(system.grid.num_cells()) {
    tmg_grid g{};
    g.nx = system.grid.nx;
    g.ny = system.grid.ny;
    g.nz = system.grid.nz;
    g.lx = system.grid.lx;
    g.ly = system.grid.ly;
    g.lz = system.grid.lz;
    g.ncc[0] = hgrid.ncc[0];
    g.ncc[1] = hgrid.ncc[1];
    g.ncc[2] = hgrid.ncc[2];
    g.sd = hgrid.sd;
    tmg_ctx* c = nullptr;
    check(tmg_create(&g, device, &c), nullptr);
    ctx_.reset(c);
    std::vector<tmg_patch> patches;
    for (const auto& p : system.boundary.patches)
      patches.push_back({static_cast<int>(p.face), p.u0, p.v0, p.u1, p.v1, p.value});
    check(tmg_set_conductivity(ctx_.get(), system.kappa.data(), patches.data(),
                               static_cast<int>(patches.size())),
          ctx_.get());
    tmg_mmg_options o{};
    o.kind = static_cast<int>(kind);
    o.num_local_basis = opts.num_local_basis;
    o.num_cc_basis = opts.num_cc_basis;
    o.smoother_sweeps = opts.smoother_sweeps;
    o.fine_blocks = fine_blocks;
    check(tmg_setup(ctx_.get(), &o), ctx_.get());
  }

  // Preconditioner::apply (solver.hpp:28): one V-cycle on the device.
  void apply(std::span<const double> r, std::span<double> z) const override {
    if (static_cast<topmg::index_t>(r.size()) != n_ || static_cast<topmg::index_t>(z.size()) != n_)
      throw std::invalid_argument("GpuMmgPreconditioner: size mismatch");
    check(tmg_apply_preconditioner(ctx_.get(), r.data(), z.data()), ctx_.get());
  }
  topmg::index_t size() const override { return n_; }

  tmg_ctx* context() const { return ctx_.get(); }
  topmg::PrecondKind kind() const { return kind_; }

 private:
  struct Deleter {
    void operator()(tmg_ctx* c) const { tmg_destroy(c); }
  };
  std::unique_ptr<tmg_ctx, Deleter> ctx_;
  topmg::PrecondKind kind_;
  topmg::index_t n_;
};

inline std::unique_ptr<topmg::Preconditioner> make_preconditioner(
    topmg::PrecondKind kind, const topmg::AssembledSystem& system,
    const topmg::HierarchicalGrid& hgrid, const topmg::MmgOptions& opts = {}, int device = 0,
    int fine_blocks = TMG_FINE_BLOCKS_CC) {
  return std::make_unique<GpuMmgPreconditioner>(kind, system, hgrid, opts, device, fine_blocks);
}

// topmg::pcg (solver.cpp:483-575) with the whole iteration on the device. `a`
// must be the system the preconditioner was built from (checked by size).
inline topmg::PcgResult pcg(const topmg::SparseOperator& a, const std::vector<double>& b,
                            const topmg::Preconditioner& m, const topmg::PcgOptions& opts = {},
                            const std::vector<double>& x0 = {}) {
  const auto* g = dynamic_cast<const GpuMmgPreconditioner*>(&m);
  if (!g) throw std::invalid_argument("topmg_b200::pcg: preconditioner was not built on the GPU");
  const topmg::index_t n = a.rows();
  if (a.cols() != n) throw std::invalid_argument("pcg: operator must be square");
  if (static_cast<topmg::index_t>(b.size()) != n) throw std::invalid_argument("pcg: rhs size mismatch");
  if (!x0.empty() && static_cast<topmg::index_t>(x0.size()) != n)
    throw std::invalid_argument("pcg: initial guess size mismatch");
  if (g->size() != n) throw std::invalid_argument("pcg: preconditioner size mismatch");
  topmg::PcgResult res;
  res.x.assign(static_cast<std::size_t>(n), 0.0);
  std::vector<double> hist(static_cast<std::size_t>(opts.max_iterations > 0 ? opts.max_iterations : 1));
  tmg_report rep{};
  check(tmg_pcg(g->context(), b.data(), x0.empty() ? nullptr : x0.data(), opts.rtol,
                opts.max_iterations, res.x.data(), hist.data(), &rep),
        g->context());
  res.report.preconditioner = topmg::to_string(g->kind());
  res.report.iterations = rep.iterations;
  res.report.converged = rep.converged != 0;
  res.report.residual_history.assign(hist.begin(), hist.begin() + rep.iterations);
  res.report.setup_seconds = rep.setup_seconds;
  res.report.solve_seconds = rep.solve_seconds;
  return res;
}

}  // namespace topmg_b200
