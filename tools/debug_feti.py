import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1312_5653_b200 as F
p = F.make_seeded_problem(256, 1e-4)
solver = F.SchurSolver(p, 8, 8, tol=1e-10)
print("created", flush=True)
x, st = solver.feti_solve(np.ones(p.n, dtype=complex))
print("feti ok", st, flush=True)
