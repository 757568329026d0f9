"""Config-4/5 driver: setup phase times, Schur solves/s, per-class kernel times.
python tools/run3d.py [--config 4|5] [--n N] [--s S] [--solves K]"""
import argparse, json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1312_5653_b200 import box

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--s", type=int, default=0)
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--phi", type=float, default=0.0)
a = ap.parse_args()
if a.config == 4:
    n, s, phi, phys = a.n or 128, a.s or 8, a.phi or 1e-6, 0
else:
    n, s, phi, phys = a.n or 64, a.s or 4, a.phi or 1e-4, 1
p = box.make_box_problem(n, phi=phi, physics=phys, young=1.0, poisson=0.3, seed=0)
print("info", box.box_partition_info(p, s), flush=True)
t = time.time()
solver = box.BoxSchurSolver(p, s, tol=1e-10, max_iter=2000)
print("setup %.2f s" % (time.time() - t), solver.setup_times(), flush=True)
for k in range(a.solves):
    solver.profile(True)
    t = time.time()
    r = solver.solve(p.target_state)
    dt = time.time() - t
    prof = solver.profile_read()
    solver.profile(False)
    print("solve %d: %.3f s  its %d/%d conv %s leak %.2e relres %.2e/%.2e prim %.2e" % (
        k, dt, r["plus_stats"]["iterations"], r["minus_stats"]["iterations"], r["converged"], r["imag_leak"],
        r["plus_stats"]["relative_residual"], r["minus_stats"]["relative_residual"], r["plus_stats"]["primal_residual"]), flush=True)
    print("  classes", json.dumps({k2: (round(v["ms"], 2), v["launches"]) for k2, v in prof.items()}), flush=True)
for kl in ("precond_gemv", "dual_gemv"):
    b = solver.class_bytes(kl)
    print(kl, "bytes/launch %.3f GB" % (b / 1e9), "avg ms %.3f" % (prof[kl]["ms"] / max(prof[kl]["launches"], 1) * 2),
          "GB/s %.0f" % (b / (prof[kl]["ms"] / max(prof[kl]["launches"], 1) * 2) / 1e6))
