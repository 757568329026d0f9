"""Config 3 (2048^2, 64x64 subdomains, phi 1e-6) on one GPU: setup, solve rate, spans."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_5653_b200 as F  # noqa: E402

p = F.make_seeded_problem(2048, 1e-6, seed=0)
t0 = time.perf_counter()
sv = F.SchurSolver(p, 64, 64, tol=1e-10, max_iter=2000)
print("setup s", time.perf_counter() - t0, flush=True)
sv.solve()
t0 = time.perf_counter()
k = 5
for _ in range(k):
    out = sv.solve()
dt = (time.perf_counter() - t0) / k
print("solves/s", 1.0 / dt, "iters", out["plus_stats"]["iterations"], out["minus_stats"]["iterations"],
      "spans", sv.step_spans(), flush=True)
