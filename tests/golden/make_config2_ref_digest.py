"""Generates tests/golden/config2_ref_digest.npz: digests of the REFERENCE's own range-space
Schur solve (oracle/_ref: the unmodified pdeopt sources built against the Eigen-API shim,
pdeopt::solve_range_space with FactorMethod::FetiDp) at BASELINE config 2's full size --
1024^2 Q1 heat, 32x32 subdomains of 32x32 elements, seeded sine target (seed 0), y_c = 0,
tol 1e-10, augment = false -- for every phi of the sweep {1e-2, 1e-4, 1e-6, 1e-8}.

The full vectors (3 x 1M doubles per phi) are too large to commit, so each phi keeps
  * the 2-norms of y, u, lambda,
  * 4096 entries at seeded positions,
  * 32 projections onto seeded N(0,1) vectors: for a difference d, the projections are
    N(0, |d|^2) draws, so sqrt(mean((P a - P b)^2)) estimates |a - b| -- a relative-L2
    check of the whole vector (tests/test_gpu_fullsize.py),
  * the iteration counts of both factor solves.
The CPU oracle (oracle/feti_oracle.cpp) is run on the same inputs and its full-vector
relative differences to the reference are recorded (and must be <= 1e-8).

~9 min per phi on 8 cores (the reference factors V by a sparse Cholesky every call).
Run here:  python tests/golden/make_config2_ref_digest.py [phi ...]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from oracle import refbind as R  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config2_ref_digest.npz")
N, S, TOL, MAX_ITER = 1024, 32, 1e-10, 2000
PHIS = (1e-2, 1e-4, 1e-6, 1e-8)
NSAMPLE, NPROJ = 4096, 32


def sample_index(n):
    return np.sort(np.random.default_rng(12345).choice(n, NSAMPLE, replace=False))


def projections(v, nproj=NPROJ):
    rng = np.random.default_rng(2024)
    return np.array([rng.standard_normal(v.size) @ v for _ in range(nproj)])


def digest(prefix, r, d):
    idx = sample_index(r["y"].size)
    for k in ("y", "u", "lambda"):
        d[f"{prefix}_{k}_norm"] = np.linalg.norm(r[k])
        d[f"{prefix}_{k}_sample"] = r[k][idx]
        d[f"{prefix}_{k}_proj"] = projections(r[k])
    d[f"{prefix}_iters"] = np.array([r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]])


def main():
    import paper_1312_5653_b200 as F  # host-side seeded target (no GPU needed)

    phis = [float(a) for a in sys.argv[1:]] or list(PHIS)
    d = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    ybar = F.make_seeded_problem(N, 1e-4, seed=0).target_state
    d["ybar_norm"] = np.linalg.norm(ybar)
    d["sample_index"] = sample_index(ybar.size)
    op = O.Problem(N)
    for phi in phis:
        tag = f"p{int(round(-np.log10(phi)))}"
        t0 = time.time()
        r = R.schur_solve(N, S, S, phi, ybar, tol=TOL, max_iter=MAX_ITER, threads=8)
        t_ref = time.time() - t0
        digest(tag, r, d)
        t0 = time.time()
        o = op.schur_solve(S, S, phi, ybar, None, tol=TOL, max_iter=MAX_ITER, threads=8)
        t_orc = time.time() - t0
        errs = [np.linalg.norm(o[k] - r[k]) / np.linalg.norm(r[k]) for k in ("y", "u", "lambda")]
        d[f"{tag}_oracle_rel"] = np.array(errs)
        d[f"{tag}_oracle_iters"] = np.array([o["plus_stats"]["iterations"], o["minus_stats"]["iterations"]])
        print(f"phi={phi:g}: reference {t_ref:.0f} s its {d[tag + '_iters']}, oracle {t_orc:.0f} s its "
              f"{d[tag + '_oracle_iters']}, oracle-vs-reference rel (y,u,lam) {errs}", flush=True)
        assert max(errs) <= 1e-8
        np.savez_compressed(OUT, **d)


if __name__ == "__main__":
    main()
