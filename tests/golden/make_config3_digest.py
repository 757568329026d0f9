"""Generate tests/golden/config3_digest.npz: a digest of the oracle's config-3 solve.

Config 3 of BASELINE.json (2048^2 Q1 heat, 64x64 subdomains, phi = 1e-6, sine target seed 0)
has 4.2M unknowns per vector, too large to commit and too slow for the oracle inside a test
(~170 s on 16 cores).  The digest keeps 4096 seeded sample entries plus the 2-norms of y, u,
lambda and the iteration counts; tests/test_gpu_fullsize.py compares the GPU solve with it.

Run (CPU, this container): python tests/golden/make_config3_digest.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

N, S, PHI, SEED, N_SAMPLES = 2048, 64, 1e-6, 0, 4096


def sample_index(n_free):
    return np.sort(np.random.default_rng(20261020).choice(n_free, N_SAMPLES, replace=False))


def main():
    t = time.time()
    p = O.Problem(N)
    ybar = p.target_sine(SEED)
    out = p.schur_solve(S, S, PHI, ybar, None, tol=1e-10, max_iter=2000, threads=os.cpu_count())
    idx = sample_index(len(ybar))
    np.savez_compressed(
        os.path.join(os.path.dirname(os.path.abspath(__file__)), "config3_digest.npz"),
        idx=idx, y=out["y"][idx], u=out["u"][idx], lam=out["lambda"][idx],
        norms=np.array([np.linalg.norm(out[k]) for k in ("y", "u", "lambda")]),
        iters=np.array([out["plus_stats"]["iterations"], out["minus_stats"]["iterations"]]),
        ybar_norm=np.linalg.norm(ybar))
    print("config3 digest written", time.time() - t, "s")


if __name__ == "__main__":
    main()
