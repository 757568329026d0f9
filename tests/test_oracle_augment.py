"""Oracle pins for the edge-RBM augmentation (feti.cpp:171-242, 394-454,
516-556, 572-578, 655-662), restating the reference's own known-answer tests."""
import numpy as np
import pytest


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def thermal(oracle_mod, n):
    return oracle_mod.Problem(n)


def elastic(oracle_mod, n):  # elastic_setup (test_feti.cpp:32-40): 3n x n on [0,3]x[0,1], rubber
    return oracle_mod.Problem(3 * n, n, len_x=3.0, len_y=1.0, physics=1, young=20.7e6, poisson=0.45)


def test_augmented_coarse_dimension(oracle_mod):  # test_feti.cpp:164-178 (column counts)
    # heat 8x8, 2x2: 4 edges -> 4 columns, 1 corner dof
    p = thermal(oracle_mod, 8)
    f = oracle_mod.Feti(p, 2, 2, 0.0, augment=True)
    assert p.partition_info(2, 2)["n_edges"] == 4
    assert f.coarse_dim == p.partition_info(2, 2)["n_corner_dofs"] + 4
    # plane strain elastic_setup(8, 2, 2): 4 edges x (tx, ty, rot) = 12 columns
    e = elastic(oracle_mod, 8)
    fe = oracle_mod.Feti(e, 2, 2, 0.0, augment=True)
    assert e.partition_info(2, 2)["n_edges"] == 4
    assert fe.coarse_dim == e.partition_info(2, 2)["n_corner_dofs"] + 12
    assert oracle_mod.Feti(p, 2, 2, 0.0).coarse_dim == p.partition_info(2, 2)["n_corner_dofs"]


def test_augmented_real_poisson_matches_direct(oracle_mod):  # test_feti.cpp:280-298 (both branches)
    p = thermal(oracle_mod, 8)
    K = p.dense(0)
    rhs = np.random.default_rng(5).standard_normal(p.n)
    x_ref = np.linalg.solve(K, rhs)
    for aug in (False, True):
        f = oracle_mod.Feti(p, 2, 2, 0.0, tol=1e-10, augment=aug)
        x, st = f.solve(rhs + 0j)
        assert st["converged"]
        assert rel(x.real, x_ref) <= 1e-9
        assert st["primal_residual"] <= 1e-9


def test_augmented_complex_factors_match_direct(oracle_mod):  # test_feti.cpp:309-332 (augment = true)
    p = thermal(oracle_mod, 16)
    phi = 2e-8
    c = -1j / np.sqrt(phi)
    K, V = p.dense(0), p.dense(1)
    rhs = np.random.default_rng(29).standard_normal(p.n) + 0j
    for coeff in (c, -c):
        f = oracle_mod.Feti(p, 2, 2, coeff, tol=1e-10, augment=True)
        x, st = f.solve(rhs)
        assert st["converged"]
        assert rel(x, np.linalg.solve(K + coeff * V, rhs)) <= 1e-8


def test_augmented_elasticity_helps(oracle_mod):  # test_feti.cpp:369-389
    e = elastic(oracle_mod, 8)
    K = e.dense(0)
    rhs = np.random.default_rng(41).standard_normal(e.n) + 0j
    plain = oracle_mod.Feti(e, 3, 2, 0.0, tol=1e-9, max_iter=2000)
    augm = oracle_mod.Feti(e, 3, 2, 0.0, tol=1e-9, max_iter=2000, augment=True)
    x1, s1 = plain.solve(rhs)
    x2, s2 = augm.solve(rhs)
    ref = np.linalg.solve(K, rhs.real)
    assert s1["converged"] and s2["converged"]
    assert rel(x1.real, ref) <= 1e-7 and rel(x2.real, ref) <= 1e-7
    assert s2["iterations"] <= s1["iterations"]


def test_augmented_spans_interface_h_over_h_2(oracle_mod):  # test_feti.cpp:407-425
    p = thermal(oracle_mod, 16)
    K = p.dense(0)
    rhs = np.random.default_rng(53).standard_normal(p.n) + 0j
    f = oracle_mod.Feti(p, 8, 8, 0.0, tol=1e-10, augment=True)
    x, st = f.solve(rhs)
    assert st["converged"] and st["iterations"] == 0
    assert rel(x.real, np.linalg.solve(K, rhs.real)) <= 1e-9
    assert st["primal_residual"] <= 1e-9


def test_augmented_range_space_matches_dense_kkt(oracle_mod):
    n, phi = 16, 2e-6
    p = thermal(oracle_mod, n)
    K, V = p.dense(0), p.dense(1)
    ybar = p.target_sine(0)
    S = K @ np.linalg.solve(V, K) + V / phi
    lam = np.linalg.solve(S, K @ ybar)
    y = ybar - np.linalg.solve(V, K @ lam)
    a = p.schur_solve(2, 2, phi, ybar, None, tol=1e-11, augment=False)
    b = p.schur_solve(2, 2, phi, ybar, None, tol=1e-11, augment=True)
    for r in (a, b):
        assert r["converged"]
        assert rel(r["lambda"], lam) <= 1e-7 and rel(r["y"], y) <= 1e-7
    assert b["plus_stats"]["iterations"] <= a["plus_stats"]["iterations"]


@pytest.mark.parametrize("n,s", [(16, 2), (32, 4)])
def test_augmented_dual_space_is_projected(oracle_mod, n, s):
    """The augmented solve equals the plain one (both exact) on heat and plane strain."""
    for prob in (thermal(oracle_mod, n), elastic(oracle_mod, n // 2)):
        rhs = np.random.default_rng(7).standard_normal(prob.n) + 0j
        x0, s0 = oracle_mod.Feti(prob, s, s, 0.0, tol=1e-11, max_iter=2000).solve(rhs)
        x1, s1 = oracle_mod.Feti(prob, s, s, 0.0, tol=1e-11, max_iter=2000, augment=True).solve(rhs)
        assert s0["converged"] and s1["converged"]
        assert rel(x1, x0) <= 1e-8


def test_rotation_mode_needs_two_edge_nodes(oracle_mod):  # feti.cpp:219-222
    e = elastic(oracle_mod, 4)  # 12 x 4, 2x2: vertical edges hold one node -> zero rotation column
    with pytest.raises(oracle_mod.NumericalError):
        oracle_mod.Feti(e, 2, 2, 0.0, augment=True)
