"""Effective GB/s of the two packed-GEMV classes when called back to back (profile events):
small meshes keep the operator L2-resident, config 2 streams it from HBM.
python tools/gemv_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_5653_b200 as F  # noqa: E402

for n, s in ((256, 8), (512, 16), (768, 24), (1024, 32)):
    p = F.make_seeded_problem(n, 1e-4)
    sv = F.SchurSolver(p, s, s, tol=1e-10, max_iter=100)
    nl = F.partition_info(p, s, s)["n_lambda"]
    lam = np.random.default_rng(0).standard_normal(nl) + 1j * np.random.default_rng(1).standard_normal(nl)
    for _ in range(3):
        sv.apply_dirichlet_preconditioner(lam)
        sv.apply_dual_operator(lam)
    sv.profile(True)
    sv.profile_read(reset=True)
    for _ in range(20):
        sv.apply_dirichlet_preconditioner(lam)
    pr = sv.profile_read(reset=True)
    for _ in range(20):
        sv.apply_dual_operator(lam)
    du = sv.profile_read(reset=True)
    sv.profile(False)
    for name, prof, k in (("precond", pr, "precond_gemv"), ("dual", du, "dual_gemv")):
        b = sv.class_bytes(k)
        us = 1000 * prof[k]["ms"] / prof[k]["launches"]
        print(f"n={n} S={s * s} {name:8s} {b / 1e6:8.1f} MB {us:8.2f} us {b / us / 1e3:8.1f} GB/s", flush=True)
    sv.close()
