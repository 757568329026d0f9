// Declaration a maintainer adds next to solve_range_space in pdeopt/control.hpp.
#pragma once

#include "pdeopt/control.hpp"

namespace pdeopt {

/// solve_range_space(problem, cfg) for cfg.method == FetiDp, on the B200 (libfetigpu.so).
RangeSpaceResult solve_range_space_gpu(const ControlProblem& problem, const FactorSolverConfig& cfg);

}  // namespace pdeopt
