"""Pins the CPU oracle to the REFERENCE ITSELF.

oracle/_ref is the unmodified reference (/root/reference/proj/src/{mesh,fem,mmio,feti,
control}.cpp) compiled in place against the Eigen-API shim in oracle/ref_shim/ (the image
has no Eigen, proj/CMakeLists.txt:15), plus the reference's own doctest unit tests and its
acceptance runner (oracle/Makefile `ref`).  These CPU tests check
  1. the shimmed build passes the reference's own unit tests (tests/test_*.cpp: 105 of 107
     cases; the two dense-condition-number cases of test_mesh_fem.cpp only exercise the
     shim's Jacobi eigensolver for 95 s and are run by `oracle/_ref/unit_tests` alone),
  2. the committed fixtures tests/golden/ref_golden.npz (written by make_ref_golden.py from
     the reference's solve_range_space / FetiSolver) are what the reference produces,
  3. the oracle (the C++ restatement every other CPU/GPU test uses as the checker) equals
     the reference on every fixture: y, u, lambda to 1e-10 relative, iterations equal.
The GPU path is compared with the same fixtures in tests/test_gpu_ref.py.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import refbind as R

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "ref_golden.npz")
REF_BIN = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "unit_tests")

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built and reference sources absent")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def gold():
    R.lib()
    return np.load(GOLD)


def test_reference_unit_tests_pass_with_shim():
    R.lib()  # builds oracle/_ref if needed
    if not os.path.exists(REF_BIN):
        pytest.skip("reference unit-test binary not built")
    out = subprocess.run([REF_BIN, "-tce=condition number"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    summary = out.stdout.strip().splitlines()[-1]
    assert "105 passed | 0 failed" in summary, summary


def test_reference_reproduces_fixtures(gold):
    r = R.schur_solve(64, 4, 4, 1e-4, gold["cfg1_s0_ybar"])
    for k in ("y", "u", "lambda"):
        assert rel(r[k], gold[f"cfg1_s0_{k}"]) <= 1e-13, k
    assert [r["plus_stats"]["iterations"], r["minus_stats"]["iterations"]] == list(gold["cfg1_s0_iters"])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_oracle_matches_reference_config1(oracle_mod, gold, seed):
    """BASELINE config 1 (64^2, 4x4, phi = 1e-4, seeded sine target, y_c = 0)."""
    ybar = gold[f"cfg1_s{seed}_ybar"]
    p = oracle_mod.Problem(64)
    assert np.array_equal(p.target_sine(seed), ybar)  # the shared seeded-target generator
    o = p.schur_solve(4, 4, 1e-4, ybar, None, tol=1e-10, max_iter=2000)
    for k in ("y", "u", "lambda"):
        assert rel(o[k], gold[f"cfg1_s{seed}_{k}"]) <= 1e-10, k
    assert [o["plus_stats"]["iterations"], o["minus_stats"]["iterations"]] == list(gold[f"cfg1_s{seed}_iters"])


@pytest.mark.parametrize("e", [2, 4, 6, 8])
def test_oracle_matches_reference_phi_sweep(oracle_mod, gold, e):
    """Config 2's phi sweep on 128^2 with config 2's 32x32-element subdomains."""
    o = oracle_mod.Problem(128).schur_solve(4, 4, 10.0 ** (-e), gold["sweep_ybar"], None, tol=1e-10, max_iter=2000,
                                            threads=4)
    assert rel(o["y"], gold[f"sweep_p{e}_y"]) <= 1e-10
    assert rel(o["lambda"], gold[f"sweep_p{e}_lambda"]) <= 1e-10
    assert [o["plus_stats"]["iterations"], o["minus_stats"]["iterations"]] == list(gold[f"sweep_p{e}_iters"])


def test_oracle_matches_reference_thermal_and_augmented(oracle_mod, gold):
    """The reference's own thermal problem (non-zero y_c) and edge-RBM augmentation."""
    p = oracle_mod.Problem(32)
    o = p.schur_solve(4, 4, 1e-4, p.target_thermal(), p.boundary_thermal(), tol=1e-10, max_iter=2000)
    for k in ("y", "u", "lambda"):
        assert rel(o[k], gold[f"thermal32_{k}"]) <= 1e-10, k
    assert [o["plus_stats"]["iterations"], o["minus_stats"]["iterations"]] == list(gold["thermal32_iters"])
    o = oracle_mod.Problem(64).schur_solve(4, 4, 1e-4, gold["cfg1_s0_ybar"], None, tol=1e-10, max_iter=2000,
                                           augment=True)
    for k in ("y", "u", "lambda"):
        assert rel(o[k], gold[f"aug_cfg1_{k}"]) <= 1e-10, k
    assert [o["plus_stats"]["iterations"], o["minus_stats"]["iterations"]] == list(gold["aug_cfg1_iters"])


def test_oracle_matches_reference_cantilever(oracle_mod, gold):
    """Plane-strain rubber cantilever (control.cpp:36-46), 24x8 mesh, 6x2 subdomains.  The
    state y = ybar - V^-1 K lambda cancels ~7 digits here (|y| = 5e-7 |ybar|: the target is
    nearly reachable), so y is compared against the size of ybar; u and lambda to 1e-10."""
    p = oracle_mod.Problem(24, 8, len_x=3.0, len_y=1.0, physics=1, young=20.7e6, poisson=0.45)
    o = p.schur_solve(6, 2, 1e-4, gold["cant8_ybar"], np.zeros(p.m), tol=1e-10, max_iter=2000)
    for k in ("u", "lambda"):
        assert rel(o[k], gold[f"cant8_{k}"]) <= 1e-10, k
    assert np.linalg.norm(o["y"] - gold["cant8_y"]) <= 1e-10 * np.linalg.norm(gold["cant8_ybar"])
    assert [o["plus_stats"]["iterations"], o["minus_stats"]["iterations"]] == list(gold["cant8_iters"])


def test_oracle_matches_reference_operators_and_feti(oracle_mod, gold):
    c = -1j / np.sqrt(1e-4)
    for tag, coeff in (("p", c), ("m", -c)):
        f = oracle_mod.Feti(oracle_mod.Problem(64), 4, 4, coeff)
        rng = np.random.default_rng(7)
        lam = rng.uniform(-1, 1, f.n_lambda) + 1j * rng.uniform(-1, 1, f.n_lambda)
        assert rel(f.apply_dual_operator(lam), gold[f"ops_cfg1_{tag}_dual"]) <= 1e-12
        assert rel(f.apply_dirichlet_preconditioner(lam), gold[f"ops_cfg1_{tag}_precond"]) <= 1e-12
    c = -1j / np.sqrt(2e-8)
    for aug in (1, 0):
        x, st = oracle_mod.Feti(oracle_mod.Problem(16), 2, 2, c, augment=bool(aug)).solve(gold["feti16_rhs"])
        assert rel(x, gold[f"feti16_aug{aug}_x"]) <= 1e-9
        assert st["iterations"] == int(gold[f"feti16_aug{aug}_iters"][0])


def test_reference_contract_errors():
    """ContractError / NumericalError propagate through the reference driver (csr.hpp:26-36)."""
    with pytest.raises(R.ContractError):
        R.schur_solve(16, 2, 2, -1.0, np.zeros(R.problem_size(R.HEAT, 16)[0]))
    with pytest.raises(R.ContractError):
        R.schur_solve(16, 3, 3, 1e-4, np.zeros(R.problem_size(R.HEAT, 16)[0]))
