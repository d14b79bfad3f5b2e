// Integration check of include/topmg_b200.hpp inside the reference's own code
// base: assemble with the reference (fvm.cpp), build the GPU preconditioner
// through the drop-in, then solve (1) with the reference's topmg::pcg using
// the GPU V-cycle as a plain Preconditioner and (2) with topmg_b200::pcg
// (device-resident), and compare against the reference's own MMG solve with
// the same block partition. Built by oracle/build_ref.sh (test
// infrastructure); run by tests/test_gpu_parity.py on the GPU box.
#include <cmath>
#include <cstdio>

#include "topmg/fvm.hpp"
#include "topmg/material.hpp"
#include "topmg/rng.hpp"
#include "topmg/solver.hpp"
#include "topmg_b200.hpp"

using namespace topmg;

int main() {
  const index_t n = 16;
  const GridSpec grid(n, n, n);
  const HierarchicalGrid h = build_hierarchy(grid, {2, 2, 2}, 2);
  const DesignField design = frozen_bench_design(grid, 0.3, 20240501);
  const MaterialModel mat(1e-3, 1.0, 1.0, 3);
  const std::vector<double> kappa = conductivity(design, mat);
  const AssembledSystem sys = assemble_system(grid, kappa, std::vector<double>(n * n * n, 1.0),
                                              BoundarySpec::bottom_center_patch(1, 1, 0.2, 0.0));
  const PcgOptions opts{1e-8, 1000};

  bool ok = true;
  auto rel = [](const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
      num += (a[i] - b[i]) * (a[i] - b[i]);
      den += b[i] * b[i];
    }
    return std::sqrt(num / den);
  };
  auto check = [&](const char* what, const PcgResult& ref, const Preconditioner& gpu) {
    const PcgResult via_ref_pcg = topmg::pcg(sys.matrix, sys.rhs, gpu, opts);  // reference loop
    const PcgResult device = topmg_b200::pcg(sys.matrix, sys.rhs, gpu, opts);  // device loop
    std::printf("%s: reference %d it; topmg::pcg + GPU V-cycle %d it, rel %.3e; "
                "topmg_b200::pcg %d it, rel %.3e (%s)\n",
                what, ref.report.iterations, via_ref_pcg.report.iterations,
                rel(via_ref_pcg.x, ref.x), device.report.iterations, rel(device.x, ref.x),
                device.report.preconditioner.c_str());
    ok = ok && via_ref_pcg.report.converged && device.report.converged && ref.report.converged;
    ok = ok && std::abs(via_ref_pcg.report.iterations - ref.report.iterations) <= 1;
    ok = ok && std::abs(device.report.iterations - ref.report.iterations) <= 1;
    ok = ok && rel(via_ref_pcg.x, ref.x) < 1e-6 && rel(device.x, ref.x) < 1e-6;
  };

  // (1) the drop-in's defaults against the reference's own factory defaults
  // (make_preconditioner -> build_mmg / build_two_grid, fine_blocks_by_cc)
  for (const PrecondKind kind : {PrecondKind::Mmg, PrecondKind::TwoGrid}) {
    const auto ref_m = topmg::make_preconditioner(kind, sys, h);
    const PcgResult ref = topmg::pcg(sys.matrix, sys.rhs, *ref_m, opts);
    const auto gpu = topmg_b200::make_preconditioner(kind, sys, h);
    check(kind == PrecondKind::Mmg ? "mmg (defaults)" : "two_grid (defaults)", ref, *gpu);
  }

  // (2) the opt-in coarse-cell fine blocks against the reference built with
  // the same partition through its public build_hierarchy_operators
  CoarseSpaces cs = build_coarse_spaces(h, kappa, 4, 8);
  std::vector<std::vector<index_t>> fine, coarse;
  for (index_t e = 0; e < h.num_coarse(); ++e) fine.push_back(h.cells_of_coarse(e));
  for (index_t e = 0; e < h.num_coarse_coarse(); ++e) {
    std::vector<index_t> rows;
    for (index_t c : h.coarse_children(e))
      for (index_t j = 0; j < 4; ++j) rows.push_back(c * 4 + j);
    coarse.push_back(rows);
  }
  MultiscaleHierarchy ref_m = build_hierarchy_operators(
      sys.matrix, std::move(cs.restriction_c), std::move(cs.restriction_cc), fine, coarse, 1);
  const PcgResult ref = topmg::pcg(sys.matrix, sys.rhs, ref_m, opts);
  auto gpu = topmg_b200::make_preconditioner(PrecondKind::Mmg, sys, h, {}, 0,
                                             TMG_FINE_BLOCKS_COARSE_CELL);
  check("mmg (coarse-cell fine blocks)", ref, *gpu);

  // the exceptions of the reference surface through the adapter
  try {
    topmg_b200::pcg(sys.matrix, std::vector<double>(3, 1.0), *gpu, opts);
    ok = false;
  } catch (const std::invalid_argument&) {
  }
  std::printf(ok ? "ADAPTER OK\n" : "ADAPTER FAILED\n");
  return ok ? 0 : 1;
}
