"""Generates tests/golden/config3_ref_digest.npz: digests of the REFERENCE's dual solve at
BASELINE config 3's full size (2048^2 Q1 heat, 64x64 subdomains of 32x32, phi = 1e-6, seeded
sine target seed 0, y_c = 0, tol 1e-10, augment = false): oracle/_ref's two
ComplexFactorSolver(FetiDp) (control.cpp:302-304) and the dual part of solve_range_space
(control.cpp:306-320): lambda = Re t, u = lambda / phi.  (The reference's recovery of y
factors V by a sparse Cholesky every call, which the shim's banded Cholesky cannot do at
4.2M dofs in reasonable time; y is pinned by the oracle digest config3_digest.npz and the KKT
equations in tests/test_gpu_fullsize.py.)  Kept: norms, 4096 sampled entries, 32 random
projections of lambda and u, and the iteration counts.  ~10 min on 8 cores:
    python tests/golden/make_config3_ref_digest.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import refbind as R  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config3_ref_digest.npz")
N, S, PHI = 2048, 64, 1e-6
NSAMPLE, NPROJ = 4096, 32


def main():
    import paper_1312_5653_b200 as F  # host-side seeded target (no GPU needed)

    ybar = F.make_seeded_problem(N, PHI, seed=0).target_state
    t0 = time.time()
    pair = R.FactorPair(N, S, S, PHI, tol=1e-10, max_iter=2000, threads=os.cpu_count() or 1)
    t1 = time.time()
    lam, st = pair.solve(ybar)
    t2 = time.time()
    idx = np.sort(np.random.default_rng(12345).choice(lam.size, NSAMPLE, replace=False))
    rng = np.random.default_rng(2024)
    proj = [rng.standard_normal(lam.size) for _ in range(NPROJ)]
    d = {"ybar_norm": np.linalg.norm(ybar), "sample_index": idx, "iters": np.array(st["iterations"])}
    for k, v in (("lambda", lam), ("u", lam / PHI)):
        d[f"{k}_norm"] = np.linalg.norm(v)
        d[f"{k}_sample"] = v[idx]
        d[f"{k}_proj"] = np.array([p @ v for p in proj])
    np.savez_compressed(OUT, **d)
    print(f"config 3: setup {t1 - t0:.0f} s, dual solve {t2 - t1:.0f} s, iterations {st['iterations']}", flush=True)


if __name__ == "__main__":
    main()
