"""Pins the CPU oracle (oracle/feti_oracle.cpp) before it is trusted as the checker.

The reference ships no golden vectors; its own known-answer tests
and direct-solver equivalences are re-expressed here against independent numpy/scipy
direct solves:
  test_mesh_fem.cpp:108-150, test_feti.cpp:51-106, 280-351, test_krylov.cpp:153-198,
  test_control.cpp:152-163, verify.cpp:150-191.
"""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ------------------------------------------------------------------ mesh / FEM
def test_heat_element_mass_exact(oracle_mod):  # test_mesh_fem.cpp:108-119
    p = oracle_mod.Problem(10, 10, 3.0, 3.0)  # h = 0.3
    ke, me = p.element_matrices()
    expected = np.array([[4, 2, 1, 2], [2, 4, 2, 1], [1, 2, 4, 2], [2, 1, 2, 4]]) * 0.3 * 0.3 / 36.0
    assert np.abs(me - expected).max() <= 1e-15


def test_heat_element_stiffness(oracle_mod):  # test_mesh_fem.cpp:121-126
    ke, _ = oracle_mod.Problem(4).element_matrices()
    assert np.abs(ke.sum(axis=1)).max() <= 1e-14
    assert ke[0, 0] == pytest.approx(2.0 / 3.0)
    assert ke[0, 2] == pytest.approx(-1.0 / 3.0)


def test_assembled_operators_invariants(oracle_mod):  # test_mesh_fem.cpp:128-142
    p = oracle_mod.Problem(4)
    assert (p.n, p.m) == (9, 16)
    K, V = p.dense(0), p.dense(1)
    assert np.array_equal(K, K.T) and np.array_equal(V, V.T)
    assert p.mass_entry_sum == pytest.approx(1.0, rel=1e-14)
    assert np.linalg.eigvalsh(K)[0] > 0 and np.linalg.eigvalsh(V)[0] > 0


def test_stiffness_row_sums_vanish(oracle_mod):  # test_mesh_fem.cpp:144-150
    p = oracle_mod.Problem(6)
    rs = p.dense(0) @ np.ones(p.n) + p.dense(2) @ np.ones(p.m)
    assert np.abs(rs).max() <= 1e-13


# ------------------------------------------------------------------ partition
def test_partition_2x2_n8(oracle_mod):  # test_feti.cpp:51-68
    info = oracle_mod.Problem(8).partition_info(2, 2)
    assert info["n_subdomains"] == 4 and info["n_corner_dofs"] == 1
    assert info["n_lambda"] == 12 and info["n_edges"] == 4


def test_partition_rejects(oracle_mod):  # test_feti.cpp:70-77
    p = oracle_mod.Problem(6)
    for sx, sy in ((4, 2), (6, 6), (1, 1)):
        with pytest.raises(ValueError):
            p.partition_info(sx, sy)


def test_partition_1x2_has_no_corners(oracle_mod):  # test_feti.cpp:249-251
    assert oracle_mod.Problem(8).partition_info(1, 2)["n_corner_dofs"] == 0


def test_partition_geometry_law(oracle_mod):  # test_feti.cpp:101-106
    assert oracle_mod.Problem(128).partition_info(32, 32)["ex"] == 4


@pytest.mark.parametrize("n,s,expect", [(64, 4, (16, 9, 360, 24)), (1024, 32, (1024, 961, 61504, 1984))])
def test_partition_sizes_appendix_a(oracle_mod, n, s, expect):
    info = oracle_mod.Problem(n).partition_info(s, s)
    assert (info["n_subdomains"], info["n_corner_dofs"], info["n_lambda"], info["n_edges"]) == expect


# ------------------------------------------------------------------ GMRES
def random_complex_symmetric(n, rng):  # test_helpers.hpp:29-40
    a = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    a = np.triu(a) + np.triu(a, 1).T
    return a + (4 + 2j) * np.eye(n)


def test_gmres_dense_lu(oracle_mod):  # test_krylov.cpp:153-165
    rng = np.random.default_rng(99)
    a = random_complex_symmetric(20, rng)
    b = rng.uniform(-1, 1, 20) + 1j * rng.uniform(-1, 1, 20)
    x, st = oracle_mod.gmres_dense(a, b, tol=1e-12)
    assert st["converged"]
    assert rel(x, np.linalg.solve(a, b)) <= 1e-10


def test_gmres_conjugate_systems(oracle_mod):  # test_krylov.cpp:167-191
    rng = np.random.default_rng(2024)
    a = random_complex_symmetric(16, rng)
    b = rng.uniform(-1, 1, 16) + 1j * rng.uniform(-1, 1, 16)
    x1, s1 = oracle_mod.gmres_dense(a, b, tol=1e-11)
    x2, s2 = oracle_mod.gmres_dense(a.conj(), b.conj(), tol=1e-11)
    assert s1["iterations"] == s2["iterations"]
    assert np.allclose(s1["history"], s2["history"], rtol=1e-12, atol=1e-12)
    assert np.linalg.norm(x1 - x2.conj()) <= 1e-12 * (1 + np.linalg.norm(x1))


def test_gmres_zero_rhs(oracle_mod):  # test_krylov.cpp:193-200
    x, st = oracle_mod.gmres_dense(np.eye(4), np.zeros(4, dtype=complex))
    assert st["converged"] and st["iterations"] == 0 and np.linalg.norm(x) == 0.0


# ------------------------------------------------------------------ FETI
def test_feti_real_poisson_matches_cholesky(oracle_mod):  # test_feti.cpp:280-298 (augment=false)
    p = oracle_mod.Problem(8)
    K, Kc = p.dense(0), p.dense(2)
    rhs = K @ p.target_thermal() + Kc @ p.boundary_thermal()
    x, st = oracle_mod.Feti(p, 2, 2, 0.0, tol=1e-10).solve(rhs.astype(complex))
    assert st["converged"]
    xd = np.linalg.solve(K, rhs)
    assert rel(x.real, xd) <= 1e-9 and np.abs(x.imag).max() == 0.0
    assert st["interface_jump"] <= 1e-9 * np.abs(x).max()
    assert st["primal_residual"] <= 1e-9


def test_feti_zero_rhs(oracle_mod):  # test_feti.cpp:300-307
    p = oracle_mod.Problem(8)
    x, st = oracle_mod.Feti(p, 2, 2, 0.0).solve(np.zeros(p.n, dtype=complex))
    assert np.linalg.norm(x) == 0.0 and st["iterations"] == 0


def test_feti_complex_factors_match_direct(oracle_mod):  # test_feti.cpp:309-332
    p = oracle_mod.Problem(16)
    phi = 2e-8
    c = -1j / np.sqrt(phi)
    rng = np.random.default_rng(29)
    rhs = rng.uniform(-1, 1, p.n).astype(complex)
    K, V = p.dense(0), p.dense(1)
    for coeff in (c, -c):
        x, st = oracle_mod.Feti(p, 2, 2, coeff, tol=1e-10).solve(rhs)
        assert st["converged"]
        assert rel(x, np.linalg.solve(K + coeff * V, rhs)) <= 1e-8


def test_feti_conjugate_pair_iterations(oracle_mod):  # test_feti.cpp:334-351
    p = oracle_mod.Problem(16)
    c = -1j / np.sqrt(2e-6)
    rng = np.random.default_rng(31)
    rhs = rng.uniform(-1, 1, p.n).astype(complex)
    its = [oracle_mod.Feti(p, 2, 2, coeff, tol=1e-10).solve(rhs)[1]["iterations"] for coeff in (c, -c)]
    assert abs(its[0] - its[1]) <= 2


def test_feti_criterion5(oracle_mod):  # verify.cpp:150-191
    n, phi = 32, 2e-8
    p = oracle_mod.Problem(n)
    K, V, Kc = p.dense(0), p.dense(1), p.dense(2)
    rhs = K @ p.target_thermal() + Kc @ p.boundary_thermal()
    c = -1j / np.sqrt(phi)
    for coeff in (0.0, c, -c):
        x, st = oracle_mod.Feti(p, 4, 4, coeff, tol=1e-10).solve(rhs.astype(complex))
        assert st["converged"]
        assert rel(x, np.linalg.solve(K + coeff * V, rhs)) <= 1e-8
        assert st["interface_jump"] <= 1e-8 * np.abs(x).max()


# ------------------------------------------------------------------ range space
def kkt_solve_sparse(p, phi, ybar, yc):
    K = sp.csr_matrix(p.dense(0)) if p.n < 2000 else None
    return K


def test_range_space_matches_dense_kkt(oracle_mod):  # test_control.cpp:152-163
    n, phi = 8, 2e-5
    p = oracle_mod.Problem(n)
    ybar, yc = p.target_thermal(), p.boundary_thermal()
    out = p.schur_solve(2, 2, phi, ybar, yc, tol=1e-12)
    K, V, Kc = p.dense(0), p.dense(1), p.dense(2)
    m = p.n
    A = np.block([[V, np.zeros((m, m)), K], [np.zeros((m, m)), phi * V, -V], [K, -V, np.zeros((m, m))]])
    rhs = np.concatenate([V @ ybar, np.zeros(m), -(Kc @ yc)])
    x = np.linalg.solve(A, rhs)
    assert out["converged"]
    assert rel(out["y"], x[:m]) <= 1e-8
    assert rel(out["u"], x[m:2 * m]) <= 1e-8
    assert rel(out["lambda"], x[2 * m:]) <= 1e-8
    viol = np.linalg.norm(K @ out["y"] + Kc @ yc - V @ out["u"]) / np.linalg.norm(K @ out["y"])
    assert viol <= 1e-8


def test_config1_schur_matches_sparse_direct(oracle_mod):
    """BASELINE config 1 (64x64, 4x4, phi=1e-4, seed 0) against a scipy sparse KKT solve."""
    n, phi = 64, 1e-4
    p = oracle_mod.Problem(n)
    ybar = p.target_sine(0)
    out = p.schur_solve(4, 4, phi, ybar, None, tol=1e-10, threads=4)
    K, V = sp.csr_matrix(p.dense(0)), sp.csr_matrix(p.dense(1))
    # exact Schur solve: (K V^-1 K + V/phi) lambda = K ybar
    S = K @ spla.splu(V.tocsc()).solve(K.toarray()) + V.toarray() / phi
    lam = np.linalg.solve(S, K @ ybar)
    assert out["converged"]
    assert rel(out["lambda"], lam) <= 1e-8
    assert rel(out["u"], lam / phi) <= 1e-8
    y = ybar - spla.spsolve(V.tocsc(), K @ lam)
    assert rel(out["y"], y) <= 1e-8
