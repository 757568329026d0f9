"""Generate tests/golden/golden3d.npz: full oracle solutions (oracle/feti_oracle.cpp, the 3D
restatement) at the SUBDOMAIN SIZES of BASELINE.json configs 4-5 on smaller cubes.

The full config-4/5 oracle runs do not fit this container's memory (the restated Eigen
SparseLU keeps 2 kl + ku + 1 band rows per factor: ~74 GB for config 4's 2 x 512 A_rr
factors), so the full-size GPU solves are checked by size-independent KKT residuals
(tests/test_gpu3d.py) and these fixtures pin the GPU path at the exact subdomain shapes:
  heat48: 48^3 heat, 3^3 subdomains of 16^3 (the centre one is config 4's interior class),
          phi = 1e-6, sine target seed 0 (l, m, n ~ U{1..6})
  elast32: 32^3 elasticity (E = 1, nu = 0.3, clamped x = 0), 2^3 subdomains of 16^3
          (config 5's subdomain size), phi = 1e-4, sine target seed 0
Run (CPU, this container, a few minutes): python tests/golden/make_3d_golden.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

CASES = {"heat48": dict(n=48, s=3, phi=1e-6, physics=0), "elast32": dict(n=32, s=2, phi=1e-4, physics=1)}


def main():
    out = {}
    th = os.cpu_count() or 1
    for name, c in CASES.items():
        t = time.time()
        p = O.Problem(c["n"], c["n"], n_z=c["n"], physics=c["physics"], young=1.0, poisson=0.3)
        ybar = p.target_sine(0, mmax=6)
        pair = O.SchurPair(p, c["s"], c["s"], c["phi"], tol=1e-10, max_iter=2000, threads=th, s_z=c["s"],
                           setup_threads=th)
        r = pair.run(ybar)
        for k in ("y", "u", "lambda"):
            out[f"{name}_{k}"] = r[k]
        out[f"{name}_iters"] = np.array([r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]])
        out[f"{name}_ybar_norm"] = np.linalg.norm(ybar)
        print(name, "iterations", out[f"{name}_iters"], f"{time.time() - t:.0f} s", flush=True)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden3d.npz"), **out)


if __name__ == "__main__":
    main()
