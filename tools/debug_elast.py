"""Plane-strain parity probe: FETI solve, Schur lambda and recovery vs the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_5653_b200 as F  # noqa: E402
from oracle import oracle as O  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


n_x, n_y, s_x, s_y, phi = 48, 32, 6, 4, 1e-4
p = F.make_problem(n_x, n_y, phi, physics=1, len_x=1.5, len_y=1.0, young=1.0, poisson=0.3)
op = O.Problem(n_x, n_y, len_x=1.5, len_y=1.0, physics=1, young=1.0, poisson=0.3)
K, V = op.dense(0), op.dense(1)
rng = np.random.default_rng(3)
ybar = rng.standard_normal(p.n)
sv = F.SchurSolver(p, s_x, s_y, tol=1e-10, max_iter=2000)
c = -1j / np.sqrt(phi)
A = K + c * V
rhs = rng.standard_normal(p.n) + 0j
x, st = sv.feti_solve(rhs)
xd = np.linalg.solve(A, rhs)
print("feti x vs dense", rel(x, xd), st)
out = sv.solve(ybar, None)
S = K @ np.linalg.solve(V, K) + V / phi
lam_d = np.linalg.solve(S, K @ ybar)
print("lambda vs dense", rel(out["lambda"], lam_d))
y_from_gpu_lam = ybar - np.linalg.solve(V, K @ out["lambda"])
print("y(gpu lambda) vs gpu y", rel(out["y"], y_from_gpu_lam))
print("V^-1 check: first entries", out["y"][:4], y_from_gpu_lam[:4])
