"""Generates tests/golden/config45_digest.npz: digests of the CPU oracle's range-space Schur
solve (oracle/feti_oracle.cpp, the 3D restatement; the reference itself is 2D only) at
BASELINE configs 4 and 5 at FULL size:

  config 4: 128^3 Q1 heat, 8x8x8 subdomains of 16^3, phi = 1e-6, sine target seed 0 (mmax 6)
  config 5: 64^3 Q1 linear elasticity (E = 1, nu = 0.3, clamped x = 0), 4x4x4 subdomains of
            16^3, phi = 1e-4, sine target seed 0 (mmax 6)

tol 1e-10, augment = false.  The oracle factors the subdomain blocks by symmetric band LDL^T
here (orc_set_band_ldlt: a third of the pivoted band LU's memory -- the LU needs ~74 GB at
config 4; agrees with it to rounding, tests/test_oracle3d.py) so both configs fit in 62 GB.

Per config the digest keeps the norms of y, u, lambda, 4096 entries at seeded positions,
32 projections onto seeded N(0,1) vectors (sqrt(mean((P a - P b)^2)) estimates |a - b|),
and both iteration counts.  Run here (CPU, ~10-20 min per config on 8 cores):
    python tests/golden/make_3d_digest.py [4] [5]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config45_digest.npz")
CFG = {4: dict(n=128, s=8, phi=1e-6, physics=0), 5: dict(n=64, s=4, phi=1e-4, physics=1)}
NSAMPLE, NPROJ = 4096, 32


def sample_index(n):
    return np.sort(np.random.default_rng(12345).choice(n, NSAMPLE, replace=False))


def projections(v, nproj=NPROJ):
    rng = np.random.default_rng(2024)
    return np.array([rng.standard_normal(v.size) @ v for _ in range(nproj)])


def main():
    configs = [int(a) for a in sys.argv[1:]] or [4, 5]
    d = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    th = os.cpu_count() or 1
    O.set_band_ldlt(True)
    for c in configs:
        cfg = CFG[c]
        p = O.Problem(cfg["n"], cfg["n"], n_z=cfg["n"], physics=cfg["physics"], young=1.0, poisson=0.3)
        ybar = p.target_sine(0, mmax=6)
        t0 = time.time()
        pair = O.SchurPair(p, cfg["s"], cfg["s"], cfg["phi"], tol=1e-10, max_iter=2000, threads=th, s_z=cfg["s"],
                           setup_threads=th)
        t1 = time.time()
        r = pair.run(ybar)
        t2 = time.time()
        del pair
        tag = f"c{c}"
        idx = sample_index(p.n)
        d[f"{tag}_ybar_norm"] = np.linalg.norm(ybar)
        d[f"{tag}_sample_index"] = idx
        for k in ("y", "u", "lambda"):
            d[f"{tag}_{k}_norm"] = np.linalg.norm(r[k])
            d[f"{tag}_{k}_sample"] = r[k][idx]
            d[f"{tag}_{k}_proj"] = projections(r[k])
        d[f"{tag}_iters"] = np.array([r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]])
        print(f"config {c}: n = {p.n}, setup {t1 - t0:.0f} s, solve {t2 - t1:.0f} s, iterations {d[tag + '_iters']}",
              flush=True)
        np.savez_compressed(OUT, **d)


if __name__ == "__main__":
    main()
