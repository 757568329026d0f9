// Drop-in check: the reference's own solve_range_space (pdeopt, CPU FETI-DP; built from
// /root/reference/proj/src against the Eigen-API shim, oracle/_ref) and the seam
// solve_range_space_gpu (control_gpu.cpp -> libfetigpu.so) on the SAME pdeopt::ControlProblem
// and FactorSolverConfig.  Prints one JSON line; exit 0 iff y, u, lambda agree to relative
// L2 <= 1e-8 and the iteration counts to +-2 (north_star), and both reject phi <= 0.
//
//   seam_check <n> <s> <phi> <thermal|sine> <augment 0|1>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "control_gpu.hpp"
#include "fetigpu.h"

using namespace pdeopt;

static double rel(const Vec& a, const Vec& b) { return (a - b).norm() / std::max(b.norm(), 1e-300); }

int main(int argc, char** argv) {
  if (argc != 6) {
    std::fprintf(stderr, "usage: seam_check n s phi thermal|sine augment\n");
    return 2;
  }
  const int n = std::atoi(argv[1]), s = std::atoi(argv[2]);
  const double phi = std::atof(argv[3]);
  const bool sine = std::strcmp(argv[4], "sine") == 0;
  ControlProblem p = make_thermal_problem(n, phi);  // control.cpp:24-34
  if (sine) {  // BASELINE.json's seeded sine-mode target, y_c = 0 (the library's generator)
    fetigpu_desc d{};
    d.n_x = d.n_y = n;
    d.len_x = d.len_y = 1.0;
    if (fetigpu_target_sine(&d, 0ull, 8, 8, p.target_state.data()) != FETIGPU_OK) return 3;
    p.boundary_values = Vec::Zero(p.m());
  }
  FactorSolverConfig cfg;
  cfg.method = FactorMethod::FetiDp;
  cfg.tol = 1e-10;
  cfg.feti.s_x = cfg.feti.s_y = s;
  cfg.feti.augment = std::atoi(argv[5]) != 0;
  cfg.feti.tol = 1e-10;
  cfg.feti.max_iter = 2000;
  const RangeSpaceResult ref = solve_range_space(p, cfg);
  const RangeSpaceResult gpu = solve_range_space_gpu(p, cfg);
  const double ey = rel(gpu.solution.y, ref.solution.y), eu = rel(gpu.solution.u, ref.solution.u),
               el = rel(gpu.solution.lambda, ref.solution.lambda);
  const int dp = std::abs(gpu.plus_stats.iterations - ref.plus_stats.iterations);
  const int dm = std::abs(gpu.minus_stats.iterations - ref.minus_stats.iterations);
  bool contract_ok = true;
  for (int which = 0; which < 2; ++which) {
    ControlProblem bad = p;
    bad.phi = -1.0;
    try {
      if (which == 0) (void)solve_range_space(bad, cfg);
      else (void)solve_range_space_gpu(bad, cfg);
      contract_ok = false;
    } catch (const ContractError&) {
    }
  }
  const bool ok = ey <= 1e-8 && eu <= 1e-8 && el <= 1e-8 && dp <= 2 && dm <= 2 && gpu.converged && ref.converged &&
                  contract_ok;
  std::printf(
      "{\"n\": %d, \"s\": %d, \"phi\": %g, \"target\": \"%s\", \"augment\": %d, \"rel_y\": %.3e, \"rel_u\": %.3e, "
      "\"rel_lambda\": %.3e, \"iters_ref\": [%d, %d], \"iters_gpu\": [%d, %d], \"contract_errors\": %s, \"ok\": %s}\n",
      n, s, phi, argv[4], cfg.feti.augment ? 1 : 0, ey, eu, el, ref.plus_stats.iterations, ref.minus_stats.iterations,
      gpu.plus_stats.iterations, gpu.minus_stats.iterations, contract_ok ? "true" : "false", ok ? "true" : "false");
  return ok ? 0 : 1;
}
