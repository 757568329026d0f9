// The reference-side drop-in, compiled here against the REAL pdeopt
// headers (/root/reference/proj/include, with the Eigen-API shim oracle/ref_shim standing in
// for Eigen) and linked against libfetigpu.so:
//
//   RangeSpaceResult solve_range_space_gpu(const ControlProblem&, const FactorSolverConfig&)
//
// has solve_range_space's contract (control.hpp:149-152, control.cpp:297-334) for
// FactorMethod::FetiDp, with the two complex FETI-DP(H) solves, V a, V^-1 and the primal
// recovery on the B200 (fetigpu_create + fetigpu_schur_solve, include/fetigpu.h).  A
// maintainer adds `FetiDpGpu` to FactorMethod (control.hpp:97) and dispatches to this
// function at the top of solve_range_space; that one-line header change is the only edit
// this TU needs in the reference.
#include "control_gpu.hpp"

#include "fetigpu.h"

namespace pdeopt {
namespace {

fetigpu_desc make_desc(const ControlProblem& p, const FactorSolverConfig& cfg) {
  fetigpu_desc d{};
  d.n_x = p.mesh.n_x;
  d.n_y = p.mesh.n_y;
  d.len_x = p.mesh.len_x;
  d.len_y = p.mesh.len_y;
  d.physics = p.physics.kind == PhysicsKind::Heat ? 0 : 1;
  d.young = p.physics.material.young_modulus;
  d.poisson = p.physics.material.poisson_ratio;
  d.s_x = cfg.feti.s_x;
  d.s_y = cfg.feti.s_y;
  d.phi = p.phi;                                      // c = -i/sqrt(phi), control.cpp:116
  d.tol = cfg.tol < 1e-12 ? cfg.feti.tol : cfg.tol;  // the tolerance rule of control.cpp:172
  d.max_iter = cfg.feti.max_iter;
  d.augment = cfg.feti.augment ? 1 : 0;
  d.device = 0;
  return d;
}

void check(int rc) {
  if (rc == FETIGPU_OK) return;
  if (rc == FETIGPU_CONTRACT) throw ContractError(fetigpu_last_error());
  throw NumericalError(fetigpu_last_error());
}

SolveStats to_stats(const fetigpu_feti_stats& s) {
  SolveStats out;
  out.iterations = s.iterations;
  out.relative_residual = s.relative_residual;
  out.converged = s.converged != 0;
  out.wall_time = s.solve_seconds;
  return out;
}

}  // namespace

RangeSpaceResult solve_range_space_gpu(const ControlProblem& problem, const FactorSolverConfig& cfg) {
  problem.validate();
  const fetigpu_desc d = make_desc(problem, cfg);
  fetigpu_ctx* ctx = nullptr;
  check(fetigpu_create(&d, &ctx));  // partition + assembly + factorization of K + cV, once
  RangeSpaceResult out;
  out.solution.y.resize(problem.n());
  out.solution.u.resize(problem.n());
  out.solution.lambda.resize(problem.n());
  fetigpu_schur_stats st{};
  const int rc = fetigpu_schur_solve(ctx, problem.target_state.data(),
                                     problem.m() > 0 ? problem.boundary_values.data() : nullptr,
                                     out.solution.y.data(), out.solution.u.data(), out.solution.lambda.data(), &st);
  fetigpu_destroy(ctx);
  check(rc);
  out.plus_stats = to_stats(st.plus);
  out.minus_stats = to_stats(st.minus);
  out.solution.imag_leak = st.imag_leak;
  out.imag_leak_warning = st.imag_leak_warning != 0;
  out.converged = st.converged != 0;
  out.factor_setup_seconds = st.factor_setup_seconds;
  return out;
}

}  // namespace pdeopt
