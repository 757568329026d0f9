// oracle/_ref driver: a thin extern "C" layer over the UNMODIFIED reference sources
// (/root/reference/proj/src/{mesh,fem,mmio,feti,control}.cpp), compiled in place against the
// Eigen-API shim in oracle/ref_shim/ (the image has no Eigen).  TEST INFRASTRUCTURE ONLY:
// tests/ and bench.py's reference arm load it as the checker / CPU baseline; the product
// never does.  Nothing here re-implements reference arithmetic — every entry calls the
// reference's own public API:
//   ref_schur_solve  -> pdeopt::solve_range_space(problem, {FetiDp, ...})   control.cpp:297-334
//   ref_feti_*       -> pdeopt::FetiSolver<Complex> (ctor, solve, apply_dual_operator,
//                       apply_dirichlet_preconditioner)                       feti.cpp:377-717
// The problem is the reference's make_thermal_problem (control.cpp:24-34) or
// make_cantilever_problem (control.cpp:36-46); a caller-supplied target ybar (BASELINE's
// seeded sine-mode target) replaces the reference's own target, with y_c = 0 unless given.
#include <complex>
#include <cstring>
#include <memory>
#include <string>

#include "pdeopt/control.hpp"
#include "pdeopt/feti.hpp"

using namespace pdeopt;

namespace {
thread_local std::string g_err;

template <class F> int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const ContractError& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

ControlProblem make_problem(int kind, int n, double phi, const double* ybar, const double* yc) {
  ControlProblem p = kind == 0 ? make_thermal_problem(n, phi) : make_cantilever_problem(n, phi);
  if (ybar) {
    for (int i = 0; i < p.n(); ++i) p.target_state[i] = ybar[i];
    p.boundary_values = Vec::Zero(p.m());
    if (yc)
      for (int i = 0; i < p.m(); ++i) p.boundary_values[i] = yc[i];
  }
  p.validate();
  return p;
}

// The two factor solvers of solve_range_space (control.cpp:302-304), set up once and reused:
// the reference's per_solve_seconds regime (experiments.cpp:264-265).
struct PairHandle {
  ControlProblem problem;
  std::unique_ptr<ComplexFactorSolver> plus, minus;
};

struct FetiHandle {
  ControlProblem problem;
  std::shared_ptr<const FetiPartition> part;
  std::unique_ptr<ComplexFetiSolver> solver;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// n_free (state dofs) and m (constrained dofs) of the reference problem.
int ref_problem_size(int kind, int n, int* n_free, int* m) {
  return guarded([&] {
    const ControlProblem p = kind == 0 ? make_thermal_problem(n, 1.0) : make_cantilever_problem(n, 1.0);
    *n_free = p.n();
    *m = p.m();
  });
}

// The reference's own target / boundary values (for its thermal / cantilever problem).
int ref_problem_data(int kind, int n, double* ybar, double* yc) {
  return guarded([&] {
    const ControlProblem p = kind == 0 ? make_thermal_problem(n, 1.0) : make_cantilever_problem(n, 1.0);
    for (int i = 0; i < p.n(); ++i) ybar[i] = p.target_state[i];
    for (int i = 0; i < p.m(); ++i) yc[i] = p.boundary_values[i];
  });
}

// stats: [0] its+, [1] its-, [2] conv+, [3] conv-, [4] relres+, [5] relres-, [6] imag_leak,
//        [7] factor_setup_seconds, [8] wall seconds of solve_range_space, [9] imag_leak_warning
int ref_schur_solve(int kind, int n, int s_x, int s_y, double phi, const double* ybar, const double* yc, double tol,
                    int max_iter, int augment, int threads, double* y, double* u, double* lam, double* stats) {
  return guarded([&] {
    const ControlProblem p = make_problem(kind, n, phi, ybar, yc);
    FactorSolverConfig cfg;
    cfg.method = FactorMethod::FetiDp;
    cfg.tol = tol;
    cfg.max_iter = max_iter;
    cfg.feti.s_x = s_x;
    cfg.feti.s_y = s_y;
    cfg.feti.augment = augment != 0;
    cfg.feti.tol = tol;
    cfg.feti.max_iter = max_iter;
    cfg.feti.threads = threads;
    detail::WallTimer t;
    const RangeSpaceResult r = solve_range_space(p, cfg);
    const double wall = t.seconds();
    for (int i = 0; i < p.n(); ++i) {
      y[i] = r.solution.y[i];
      u[i] = r.solution.u[i];
      lam[i] = r.solution.lambda[i];
    }
    stats[0] = r.plus_stats.iterations;
    stats[1] = r.minus_stats.iterations;
    stats[2] = r.plus_stats.converged;
    stats[3] = r.minus_stats.converged;
    stats[4] = r.plus_stats.relative_residual;
    stats[5] = r.minus_stats.relative_residual;
    stats[6] = r.solution.imag_leak;
    stats[7] = r.factor_setup_seconds;
    stats[8] = wall;
    stats[9] = r.imag_leak_warning;
  });
}

// Setup of solve_range_space's two ComplexFactorSolver(FetiDp) (control.cpp:297-304), timed.
int ref_pair_create(int kind, int n, int s_x, int s_y, double phi, double tol, int max_iter, int augment, int threads,
                    void** out, double* setup_seconds) {
  return guarded([&] {
    auto h = std::make_unique<PairHandle>();
    h->problem = kind == 0 ? make_thermal_problem(n, phi) : make_cantilever_problem(n, phi);
    FactorSolverConfig cfg;
    cfg.method = FactorMethod::FetiDp;
    cfg.tol = tol;
    cfg.max_iter = max_iter;
    cfg.feti.s_x = s_x;
    cfg.feti.s_y = s_y;
    cfg.feti.augment = augment != 0;
    cfg.feti.tol = tol;
    cfg.feti.max_iter = max_iter;
    cfg.feti.threads = threads;
    const SchurFactors factors = build_complex_factors(h->problem);
    detail::WallTimer t;
    h->plus = std::make_unique<ComplexFactorSolver>(h->problem, factors.c, cfg);
    h->minus = std::make_unique<ComplexFactorSolver>(h->problem, -factors.c, cfg);
    *setup_seconds = t.seconds();
    *out = h.release();
  });
}

void ref_pair_destroy(void* h) { delete static_cast<PairHandle*>(h); }

// The dual part of solve_range_space (control.cpp:306-320) for a target ybar (y_c = 0) with
// the factors reused: rhs = K ybar, a = (K + cV)^-1 rhs, t = (K - cV)^-1 V a, lambda = Re t.
// stats: [0] its+, [1] its-, [2] converged (both), [3] per_solve_seconds = wall time of the
// two factor solves (experiments.cpp:265), [4] wall seconds of the whole call.
int ref_pair_solve(void* hv, const double* ybar, double* lam, double* stats) {
  return guarded([&] {
    auto* h = static_cast<PairHandle*>(hv);
    detail::WallTimer t;
    ControlProblem& p = h->problem;
    for (int i = 0; i < p.n(); ++i) p.target_state[i] = ybar[i];
    p.boundary_values = Vec::Zero(p.m());
    const Vec rhs = p.schur_rhs();
    const CVec crhs = rhs.cast<Complex>();
    auto [a, sp] = h->plus->solve(crhs);
    CVec va(a.size());
    p.ops.V.apply(a, va);
    auto [tv, sm] = h->minus->solve(va);
    for (int i = 0; i < p.n(); ++i) lam[i] = tv[i].real();
    stats[0] = sp.iterations;
    stats[1] = sm.iterations;
    stats[2] = sp.converged && sm.converged;
    stats[3] = sp.wall_time + sm.wall_time;
    stats[4] = t.seconds();
  });
}

// A persistent FetiSolver<Complex> on A = stiffness_coeff K + (mass_re + i mass_im) V.
int ref_feti_create(int kind, int n, int s_x, int s_y, double stiffness_coeff, double mass_re, double mass_im,
                    double tol, int max_iter, int augment, int threads, void** out) {
  return guarded([&] {
    auto h = std::make_unique<FetiHandle>();
    h->problem = kind == 0 ? make_thermal_problem(n, 1.0) : make_cantilever_problem(n, 1.0);
    h->part = std::make_shared<const FetiPartition>(
        partition_structured(h->problem.mesh, h->problem.physics, h->problem.ops, s_x, s_y));
    OperatorSpec spec;
    spec.stiffness_coeff = stiffness_coeff;
    spec.mass_coeff = Complex(mass_re, mass_im);
    FetiConfig fc;
    fc.s_x = s_x;
    fc.s_y = s_y;
    fc.augment = augment != 0;
    fc.tol = tol;
    fc.max_iter = max_iter;
    fc.threads = threads;
    h->solver = std::make_unique<ComplexFetiSolver>(h->problem.mesh, h->problem.physics, h->problem.ops, h->part, spec, fc);
    *out = h.release();
  });
}

void ref_feti_destroy(void* h) { delete static_cast<FetiHandle*>(h); }

// sizes: [0] n_free, [1] n_lambda, [2] coarse_dim, [3] n_subdomains
int ref_feti_sizes(void* hv, int* sizes) {
  return guarded([&] {
    auto* h = static_cast<FetiHandle*>(hv);
    sizes[0] = h->part->n_free;
    sizes[1] = h->solver->n_lambda();
    sizes[2] = h->solver->coarse_dim();
    sizes[3] = h->part->n_subdomains();
  });
}

// stats: [0] iterations, [1] relres, [2] converged, [3] primal_residual, [4] interface_jump,
//        [5] solve seconds
int ref_feti_solve(void* hv, const double* rhs_c128, double* x_c128, double* stats) {
  return guarded([&] {
    auto* h = static_cast<FetiHandle*>(hv);
    const int n = h->part->n_free;
    CVec rhs(n);
    std::memcpy(rhs.data(), rhs_c128, sizeof(Complex) * n);
    auto [x, st] = h->solver->solve(rhs);
    std::memcpy(x_c128, x.data(), sizeof(Complex) * n);
    stats[0] = st.dual.iterations;
    stats[1] = st.dual.relative_residual;
    stats[2] = st.dual.converged;
    stats[3] = st.primal_residual;
    stats[4] = st.interface_jump;
    stats[5] = st.solve_seconds;
  });
}

// which: 0 = dual operator F (feti.cpp:581-594), 1 = Dirichlet preconditioner (597-627),
//        2 = augmentation projection (572-578)
int ref_feti_apply(void* hv, int which, const double* in_c128, double* out_c128) {
  return guarded([&] {
    auto* h = static_cast<FetiHandle*>(hv);
    const int m = h->solver->n_lambda();
    CVec v(m);
    std::memcpy(v.data(), in_c128, sizeof(Complex) * m);
    CVec r;
    if (which == 0) r = h->solver->apply_dual_operator(v);
    else if (which == 1) r = h->solver->apply_dirichlet_preconditioner(v);
    else {
      r = v;
      h->solver->project_out_augmentation(r);
    }
    std::memcpy(out_c128, r.data(), sizeof(Complex) * m);
  });
}

}  // extern "C"
