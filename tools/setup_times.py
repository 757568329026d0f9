"""Setup-stage timings of the config-2 context (FETIGPU_PHASE_TIMES=1 prints them): three
consecutive creations (the first also pays CUDA's lazy module loading)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FETIGPU_PHASE_TIMES"] = "1"
import paper_1312_5653_b200 as F  # noqa: E402

p = F.make_seeded_problem(1024, 1e-4, seed=0)
for k in range(3):
    t0 = time.perf_counter()
    s = F.SchurSolver(p, 32, 32, tol=1e-10, max_iter=2000)
    print(f"create {k}: {time.perf_counter() - t0:.3f} s", file=sys.stderr, flush=True)
    s.close()
