"""The reference's hot-path acceptance criteria (src/verify.cpp) restated on the GPU path,
with the reference's own iteration counts (tests/golden/ref_golden.npz, from oracle/_ref)
as the pin:

  4  range-space correctness (verify.cpp:129-147): thermal n = 8 at phi = 1e-2 .. 1e-8, the
     GPU range-space solve against a dense KKT solve, rel err <= 1e-8, constraint violation
     <= 1e-8 (the reference runs this with its CPU direct backend; here the GPU FETI path)
  6  conjugate-pair symmetry (verify.cpp:194-226): the phi sweep of experiments.cpp:118-127
     (thermal 64^2, 8x8 subdomains, phi = 2e-2 .. 2e-12, augment false and true), every
     solve converged and |iters(-) - iters(+)| <= 2
  7  numerical scalability (verify.cpp:228-246): thermal n = 16, 32, 64 at H/h = 8,
     phi = 2e-8: converged, iterations non-increasing (+2 slack) as n grows

For 6 and 7 every GPU iteration count is also within +-2 of the reference's own count.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_criterion4_range_space_correctness(fetigpu, oracle_mod):
    worst_err = worst_violation = 0.0
    for phi in (1e-2, 1e-4, 1e-6, 1e-8):
        p = fetigpu.make_thermal_problem(8, phi)
        op = oracle_mod.Problem(8)
        K, V, Kc = op.dense(0), op.dense(1), op.dense(2)
        n = op.n
        A = np.zeros((3 * n, 3 * n))
        A[:n, :n], A[:n, 2 * n:] = V, K
        A[n:2 * n, n:2 * n], A[n:2 * n, 2 * n:] = phi * V, -V
        A[2 * n:, :n], A[2 * n:, n:2 * n] = K, -V
        rhs = np.zeros(3 * n)
        rhs[:n] = V @ p.target_state
        rhs[2 * n:] = -(Kc @ p.boundary_values)
        x = np.linalg.solve(A, rhs)
        out = fetigpu.solve_range_space(p, tol=1e-12, max_iter=2000)  # FetiConfig defaults: 2x2, augment
        got = np.concatenate([out["y"], out["u"], out["lambda"]])
        worst_err = max(worst_err, np.linalg.norm(got - x) / np.linalg.norm(x))
        ky = K @ out["y"]
        viol = np.linalg.norm(ky + Kc @ p.boundary_values - V @ out["u"]) / np.linalg.norm(ky)  # control.cpp:127-133
        worst_violation = max(worst_violation, viol)
    assert worst_err <= 1e-8 and worst_violation <= 1e-8, (worst_err, worst_violation)


def test_criterion6_conjugate_pair_symmetry(fetigpu, gold):
    from paper_1312_5653_b200 import experiments as E

    cfg = E.ExperimentConfig.defaults_for("phi_sweep")
    rows = E.run_phi_sweep(cfg)
    assert len(rows) == 2 * len(cfg.phi)
    assert np.allclose(cfg.phi, gold["crit6_phis"], rtol=1e-15)
    worst = 0
    for i, row in enumerate(rows):
        assert row.converged, (row.phi, row.augment, row.error)
        worst = max(worst, abs(row.iters_minus - row.iters_plus))
        ref = gold["crit6_iters"][i // 2][1 if row.augment else 0]
        assert abs(row.iters_plus - int(ref[0])) <= 2 and abs(row.iters_minus - int(ref[1])) <= 2, (row.phi, row.augment)
    assert worst <= 2


def test_criterion7_numerical_scalability(fetigpu, gold):
    from paper_1312_5653_b200 import experiments as E

    cfg = E.ExperimentConfig.defaults_for("scalability")
    cfg.augment = True  # the ExperimentConfig default (experiments.hpp:29)
    rows = E.run_scalability(cfg)
    assert len(rows) == 3
    for i, row in enumerate(rows):
        assert row.converged
        ref = gold["crit7_iters"][i]
        assert abs(row.iters_plus - int(ref[0])) <= 2 and abs(row.iters_minus - int(ref[1])) <= 2
        if i > 0:
            assert row.iters_minus <= rows[i - 1].iters_minus + 2
            assert row.iters_plus <= rows[i - 1].iters_plus + 2
