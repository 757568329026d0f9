"""How often would selective reorthogonalisation skip CGS pass 2?  Runs config-2 FETI solves
in eager mode and records, per Arnoldi step, ratio = |w - V h1| / |w| from the pass-1 dots
(h1 = V^H w, |w|^2) read back after each step.  python tools/cgs_ratio.py [n s phi]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FETIGPU_EAGER"] = "1"
os.environ["FETIGPU_CGS_RATIO"] = "1"
import paper_1312_5653_b200 as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
s = int(sys.argv[2]) if len(sys.argv) > 2 else 32
phi = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
p = F.make_seeded_problem(n, phi)
sv = F.SchurSolver(p, s, s, tol=1e-10, max_iter=2000)
out = sv.solve()
print("iterations", out["plus_stats"]["iterations"], out["minus_stats"]["iterations"])
