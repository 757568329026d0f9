"""Full BASELINE sizes on the GPU.

* config 2 (1024^2, 32x32 subdomains): against the CPU oracle (~30-60 s of CPU time).
* config 3 (2048^2, 64x64 subdomains, 4.2M dofs): the oracle is too slow for a test, so
  the solution is checked through size-independent properties: the two KKT equations
  (control.cpp:56-59) with the exact Q1 operators built by Kronecker products in scipy
      K y + K_c y_c - V u = 0,      V (y - ybar) + K lambda = 0,      u = lambda / phi,
  and determinism / conjugate symmetry of the iteration counts.  The first residual is
  the Schur residual K ybar - S lambda; relative to |K ybar| it inherits the conditioning
  of K -/+ i beta V at the FETI tolerance 1e-10 (calibrated on the oracle: ~2e-10 at
  phi <= 1e-6, ~2e-8 at 1e-4, ~1e-5 at 1e-2), hence the phi-dependent bound.
"""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def q1_operators(n):
    """Interior-node Q1 stiffness/mass on the unit square, Dirichlet on the whole boundary:
    K = K1 (x) M1 + M1 (x) K1, V = M1 (x) M1 with 1-D P1 matrices (tensor-product Q1)."""
    h = 1.0 / n
    m = n - 1
    e = np.ones(m)
    K1 = sp.diags([-e[:-1], 2 * e, -e[:-1]], [-1, 0, 1]) / h
    M1 = sp.diags([e[:-1], 4 * e, e[:-1]], [-1, 0, 1]) * (h / 6.0)
    K = (sp.kron(M1, K1) + sp.kron(K1, M1)).tocsr()
    V = sp.kron(M1, M1).tocsr()
    return K, V


def test_q1_kronecker_operators_match_oracle(oracle_mod):
    K, V = q1_operators(16)
    p = oracle_mod.Problem(16)
    assert np.abs(K.toarray() - p.dense(0)).max() <= 1e-14
    assert np.abs(V.toarray() - p.dense(1)).max() <= 1e-17


def test_config2_matches_oracle(fetigpu, oracle_mod):
    n, s, phi = 1024, 32, 1e-4
    p = fetigpu.make_seeded_problem(n, phi, seed=0)
    solver = fetigpu.SchurSolver(p, s, s, tol=1e-10, max_iter=2000)
    out = solver.solve()
    solver.close()
    import os

    ref = oracle_mod.Problem(n).schur_solve(s, s, phi, p.target_state, None, tol=1e-10, max_iter=2000,
                                            threads=os.cpu_count() or 1)
    assert out["converged"] and ref["converged"]
    for k in ("y", "u", "lambda"):
        assert rel(out[k], ref[k]) <= 1e-8, k
    assert abs(out["plus_stats"]["iterations"] - ref["plus_stats"]["iterations"]) <= 2
    assert abs(out["minus_stats"]["iterations"] - ref["minus_stats"]["iterations"]) <= 2


# calibrated on the oracle at 1024^2, seed 1 (the GPU reproduces the same values):
# 1.83e-4 at phi = 1e-2, 6.1e-8 at phi = 1e-8 (K -/+ i beta V conditioning at FETI tol 1e-10)
# and on the oracle at 2048^2, 64x64, phi = 1e-6, seed 0: 1.216e-4, 26 / 26 iterations
# (orc_schur run for 166 s on 16 cores; the bound grows with the mesh, h^-2 conditioning)
SCHUR_RES_BOUND = {(1024, 1e-2): 1e-3, (1024, 1e-8): 5e-7, (2048, 1e-6): 5e-4}
CONFIG3_ORACLE_ITERS = 26


def check_kkt(out, ybar, phi, n):
    K, V = q1_operators(n)
    r1 = K @ out["y"] - V @ out["u"]
    r2 = V @ (out["y"] - ybar) + K @ out["lambda"]
    assert np.linalg.norm(r1) <= SCHUR_RES_BOUND[(n, phi)] * np.linalg.norm(K @ ybar)
    # r2 vanishes by construction (primal recovery); bound it by the rounding scale |K||lambda|
    assert np.linalg.norm(r2) <= 1e-12 * np.linalg.norm(abs(K) @ abs(out["lambda"]))
    assert np.allclose(out["u"] * phi, out["lambda"], rtol=1e-14, atol=0)


@pytest.mark.parametrize("phi", [1e-2, 1e-8])
def test_config2_phi_sweep_kkt_residuals(fetigpu, phi):
    n, s = 1024, 32
    p = fetigpu.make_seeded_problem(n, phi, seed=1)
    solver = fetigpu.SchurSolver(p, s, s, tol=1e-10, max_iter=2000)
    out = solver.solve()
    solver.close()
    assert out["converged"]
    check_kkt(out, p.target_state, phi, n)
    assert abs(out["plus_stats"]["iterations"] - out["minus_stats"]["iterations"]) <= 2


def test_config3_kkt_residuals_and_determinism(fetigpu):
    n, s, phi = 2048, 64, 1e-6
    p = fetigpu.make_seeded_problem(n, phi, seed=0)
    solver = fetigpu.SchurSolver(p, s, s, tol=1e-10, max_iter=2000)
    a = solver.solve()
    b = solver.solve()
    solver.close()
    assert a["converged"]
    for k in ("y", "u", "lambda"):
        assert np.array_equal(a[k], b[k])
    check_kkt(a, p.target_state, phi, n)
    assert abs(a["plus_stats"]["iterations"] - CONFIG3_ORACLE_ITERS) <= 2
    assert abs(a["minus_stats"]["iterations"] - CONFIG3_ORACLE_ITERS) <= 2
