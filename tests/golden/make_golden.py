"""Regenerates tests/golden/*.npz from the CPU oracle (oracle/feti_oracle.cpp).

The reference ships no golden vectors and cannot be built here (no Eigen); these
fixtures freeze the oracle's outputs after it was pinned against the reference's
known-answer tests and scipy direct solves (tests/test_oracle.py), so later changes to
either the oracle or the GPU path are caught at full precision.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def main():
    out = {}
    # BASELINE config 1: 64x64, 4x4 subdomains, phi = 1e-4, tol 1e-10, seeds 0..2
    p = O.Problem(64)
    for seed in (0, 1, 2):
        r = p.schur_solve(4, 4, 1e-4, p.target_sine(seed), None, tol=1e-10, max_iter=2000, threads=4)
        out[f"cfg1_s{seed}_lambda"] = r["lambda"]
        out[f"cfg1_s{seed}_iters"] = np.array([r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]])
        a, m, n = O.sine_modes(seed)
        out[f"sine_s{seed}_a"], out[f"sine_s{seed}_m"], out[f"sine_s{seed}_n"] = a, m, n
    # reference thermal problem (fem.cpp:194-220, nonzero y_c), n = 16, 2x2, phi = 2e-5
    q = O.Problem(16)
    r = q.schur_solve(2, 2, 2e-5, q.target_thermal(), q.boundary_thermal(), tol=1e-12, max_iter=2000)
    out["thermal16_y"], out["thermal16_u"], out["thermal16_lambda"] = r["y"], r["u"], r["lambda"]
    out["thermal16_iters"] = np.array([r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]])
    np.savez_compressed(os.path.join(HERE, "oracle_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "oracle_golden.npz"), sorted(out))


if __name__ == "__main__":
    main()
