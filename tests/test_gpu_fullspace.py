"""Full-space KKT method on the GPU, restating test_control.cpp:290-362 with
the B200 FETI-DP inner solves in place of the reference's DirectLu inner backend."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def dense_kkt(oracle_mod, p):
    op = oracle_mod.Problem(p.n_x)
    K, V, Kc = op.dense(0), op.dense(1), op.dense(2)
    n = p.n
    A = np.zeros((3 * n, 3 * n))
    A[:n, :n], A[:n, 2 * n:] = V, K
    A[n:2 * n, n:2 * n], A[n:2 * n, 2 * n:] = p.phi * V, -V
    A[2 * n:, :n], A[2 * n:, n:2 * n] = K, -V
    b = np.concatenate([V @ p.target_state, np.zeros(n), -(Kc @ p.boundary_values)])
    x = np.linalg.solve(A, b)
    return x[:n], x[n:2 * n], x[2 * n:]


@pytest.mark.parametrize("phi", [2e-2, 2e-5])
def test_exact_schur_preconditioner_converges_in_3(fetigpu, oracle_mod, phi):  # test_control.cpp:290-303
    p = fetigpu.make_thermal_problem(8, phi)
    out = fetigpu.solve_full_space(p, precond="sc", outer="gmres", tol=1e-10, inner_tol=1e-12)
    assert out["stats"]["converged"]
    assert out["stats"]["iterations"] <= 3
    y, u, lam = dense_kkt(oracle_mod, p)
    assert rel(out["y"], y) <= 1e-8 and rel(out["u"], u) <= 1e-8 and rel(out["lambda"], lam) <= 1e-8


def test_unpreconditioned_minres(fetigpu, oracle_mod):  # test_control.cpp:305-320
    p = fetigpu.make_thermal_problem(8, 2e-5)
    out = fetigpu.solve_full_space(p, precond="none", outer="minres", tol=1e-10, max_iter=20000)
    assert out["stats"]["converged"]
    y, _, _ = dense_kkt(oracle_mod, p)
    assert rel(out["y"], y) <= 1e-4


def test_pearson_wathen_iterations_flat_in_phi(fetigpu):  # test_control.cpp:322-340
    iters = []
    for phi in (1e-2, 1e-5, 1e-8):
        p = fetigpu.make_thermal_problem(8, phi)
        out = fetigpu.solve_full_space(p, precond="sp", outer="minres", tol=1e-7)
        assert out["stats"]["converged"]
        assert out["stats"]["iterations"] <= 20
        iters.append(out["stats"]["iterations"])
    assert max(iters) - min(iters) <= 3


def test_exact_schur_with_minres_rejected(fetigpu):  # test_control.cpp:342-348
    p = fetigpu.make_thermal_problem(4, 1e-3)
    with pytest.raises(ValueError):
        fetigpu.solve_full_space(p, precond="sc", outer="minres")


@pytest.mark.parametrize("phi", [1e-2, 1e-5, 1e-8])
def test_range_and_full_space_agree(fetigpu, phi):  # test_control.cpp:350-362
    p = fetigpu.make_thermal_problem(8, phi)
    rs = fetigpu.solve_range_space(p)
    fs = fetigpu.solve_full_space(p, precond="sc", outer="gmres", tol=1e-12)
    assert np.linalg.norm(rs["y"] - fs["y"]) <= 1e-7 * (1.0 + np.linalg.norm(fs["y"]))
    assert np.linalg.norm(rs["u"] - fs["u"]) <= 1e-7 * (1.0 + np.linalg.norm(fs["u"]))


def test_full_space_config1_mesh(fetigpu, oracle_mod):
    """BASELINE config-1 mesh (64^2, 4x4 subdomains, seeded target): sc + GMRES and sp + MINRES
    both reproduce the range-space solution."""
    p = fetigpu.make_seeded_problem(64, 1e-4, seed=0)
    ref = oracle_mod.Problem(64).schur_solve(4, 4, 1e-4, p.target_state, None, tol=1e-12, max_iter=2000, threads=4)
    sc = fetigpu.solve_full_space(p, precond="sc", outer="gmres", tol=1e-11, s_x=4, s_y=4, augment=False)
    sp = fetigpu.solve_full_space(p, precond="sp", outer="minres", tol=1e-10, s_x=4, s_y=4, augment=False)
    assert sc["stats"]["converged"] and sp["stats"]["converged"]
    for out in (sc, sp):
        assert rel(out["y"], ref["y"]) <= 1e-7
        assert rel(out["lambda"], ref["lambda"]) <= 1e-6
