"""Phase timings of config-2 Schur solves (FETIGPU_PHASE_TIMES=1: CUDA events at named points
of every FETI solve, printed per solve; the first creation also prints the setup stages)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FETIGPU_PHASE_TIMES"] = "1"
import paper_1312_5653_b200 as F  # noqa: E402

p = F.make_seeded_problem(1024, 1e-4, seed=0)
s = F.SchurSolver(p, 32, 32, tol=1e-10, max_iter=2000)
for k in range(3):
    s.solve()
s.close()
