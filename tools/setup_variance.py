"""Setup time of config 2 over repeated context creations, for two max_iter values (the Krylov
bases are (max_iter + 1) vectors each): python tools/setup_variance.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_5653_b200 as F  # noqa: E402

p = F.make_seeded_problem(1024, 1e-4, seed=0)
for mi in (2000, 200, 2000, 200):
    ts = []
    for k in range(6):
        t0 = time.perf_counter()
        s = F.SchurSolver(p, 32, 32, tol=1e-10, max_iter=mi)
        ts.append(time.perf_counter() - t0)
        s.close()
    print(mi, " ".join(f"{t:.3f}" for t in ts), flush=True)
