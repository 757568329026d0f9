import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1312_5653_b200 as F
n, s, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
p = F.make_seeded_problem(n, 1e-4)
solver = F.SchurSolver(p, s, s, tol=1e-10)
for r in range(reps):
    out = solver.solve()
    print(r, out["plus_stats"]["iterations"], flush=True)
print("done", flush=True)
