"""One config-2 range-space Schur solve after one warm-up solve (for ncu launch lists).
Usage: python tools/profile_step.py [n] [s] [phi]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_5653_b200 as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
s = int(sys.argv[2]) if len(sys.argv) > 2 else 32
phi = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
p = F.make_seeded_problem(n, phi, seed=0)
solver = F.SchurSolver(p, s, s, tol=1e-10, max_iter=2000)
print("setup launches", solver.launch_count(reset=True), flush=True)
solver.solve()
print("warm-up solve launches", solver.launch_count(reset=True), flush=True)
t0 = time.perf_counter()
out = solver.solve()
print("solve launches", solver.launch_count(reset=True), "iters", out["plus_stats"]["iterations"],
      out["minus_stats"]["iterations"], "wall ms", 1e3 * (time.perf_counter() - t0), flush=True)
solver.close()
