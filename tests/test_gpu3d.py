"""3D extension (BASELINE.json configs 4-5): the sm_100a path against the CPU oracle.

CPU part: the C++ host core's 3D partition and seeded target agree with the oracle's
restatement (oracle/feti_oracle.cpp partition_structured3d, orc_target_sine3).
GPU part (-m gpu): FETI-DP solves, operator applications and range-space Schur solves on
the device equal the oracle's on the same seeded inputs (relative L2 <= 1e-8, iteration
counts within +-2 — the north_star bar), for heat and linear elasticity.
"""
import numpy as np
import pytest


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


CASES = [  # physics, n, s
    (0, 8, 2),
    (0, 12, 3),
    (0, 16, 2),
    (1, 8, 2),
    (1, 12, 3),
]


@pytest.mark.parametrize("physics,n,s", CASES + [(0, 48, 3), (1, 24, 2)])
def test_host_partition3d_matches_oracle(fetigpu, oracle_mod, physics, n, s):
    from paper_1312_5653_b200 import box

    p = box.make_box_problem(n, phi=1e-4, physics=physics, young=1.0, poisson=0.3, seed=3)
    info = box.box_partition_info(p, s)
    q = oracle_mod.Problem(n, n, n_z=n, physics=physics, young=1.0, poisson=0.3)
    ref = q.partition_info(s, s, s)
    assert (info["n"], info["m"]) == (q.n, q.m)
    for k in ("n_subdomains", "n_corner_dofs", "n_lambda", "ex", "ey", "ez"):
        assert info[k] == ref[k], k
    sizes = q.partition_sizes(s, s, s)
    assert info["NB"] == sizes[:, 2].max() and info["NC"] == max(sizes[:, 3].max(), 1)
    assert info["NI"] == max(32, -(-sizes[:, 1].max() // 32) * 32)
    assert np.array_equal(p.target_state, q.target_sine(3, mmax=6))


def test_config4_config5_sizes(fetigpu):
    from paper_1312_5653_b200 import box

    i4 = box.box_partition_info(box.BoxProblem(128, 128, 128, 1e-6), 8)
    assert (i4["n"], i4["n_subdomains"], i4["n_corner_dofs"], i4["NB"], i4["NC"]) == (127 ** 3, 512, 343, 1530, 8)
    i5 = box.box_partition_info(box.BoxProblem(64, 64, 64, 1e-4, physics=1, young=1.0, poisson=0.3), 4)
    assert (i5["n"], i5["n_subdomains"], i5["n_corner_dofs"]) == (3 * 64 * 65 * 65, 64, 288)


@pytest.mark.gpu
@pytest.mark.parametrize("physics,n,s", CASES)
def test_gpu3d_feti_solve_matches_oracle(fetigpu, oracle_mod, physics, n, s):
    from paper_1312_5653_b200 import box

    phi = 1e-4
    c = -1j / np.sqrt(phi)
    p = box.make_box_problem(n, phi=phi, physics=physics, young=1.0, poisson=0.3, seed=1)
    q = oracle_mod.Problem(n, n, n_z=n, physics=physics, young=1.0, poisson=0.3)
    rng = np.random.default_rng(n + 10 * physics)
    rhs = rng.standard_normal(p.n) + 1j * rng.standard_normal(p.n)
    solver = box.BoxSchurSolver(p, s, tol=1e-10, max_iter=500)
    try:
        x, st = solver.feti_solve(rhs)
        F = oracle_mod.Feti(q, s, s, c, s_z=s, tol=1e-10, max_iter=500)
        xr, sr = F.solve(rhs)
        assert st["converged"] and sr["converged"]
        assert rel(x, xr) <= 1e-8
        assert abs(st["iterations"] - sr["iterations"]) <= 2
        assert st["primal_residual"] <= 1e-8
        # conjugate factor through conjugate reuse
        xm, stm = solver.feti_solve(np.conj(rhs), sign=-1)
        assert rel(xm, np.conj(x)) <= 1e-12 and stm["iterations"] == st["iterations"]
        # operator parity (apply_dual_operator / apply_dirichlet_preconditioner)
        lam = rng.standard_normal(F.n_lambda) + 1j * rng.standard_normal(F.n_lambda)
        assert rel(solver.apply_dual_operator(lam), F.apply_dual_operator(lam)) <= 1e-11
        assert rel(solver.apply_dirichlet_preconditioner(lam), F.apply_dirichlet_preconditioner(lam)) <= 1e-11
    finally:
        solver.close()


@pytest.mark.gpu
@pytest.mark.parametrize("physics,n,s,phi", [(0, 12, 3, 1e-6), (0, 16, 2, 1e-4), (1, 8, 2, 1e-4), (1, 12, 3, 1e-2)])
def test_gpu3d_schur_solve_matches_oracle(fetigpu, oracle_mod, physics, n, s, phi):
    from paper_1312_5653_b200 import box

    p = box.make_box_problem(n, phi=phi, physics=physics, young=1.0, poisson=0.3, seed=2)
    q = oracle_mod.Problem(n, n, n_z=n, physics=physics, young=1.0, poisson=0.3)
    r = box.solve_range_space_3d(p, s, tol=1e-10, max_iter=500)
    o = q.schur_solve(s, s, phi, p.target_state, s_z=s, tol=1e-10, max_iter=500)
    assert r["converged"] and o["converged"]
    for k in ("y", "u", "lambda"):
        assert rel(r[k], o[k]) <= 1e-8, k
    assert abs(r["plus_stats"]["iterations"] - o["plus_stats"]["iterations"]) <= 2
    assert abs(r["minus_stats"]["iterations"] - o["minus_stats"]["iterations"]) <= 2
    assert r["imag_leak"] <= 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("physics", [0, 1])
def test_gpu3d_schur_solve_with_dirichlet_data(fetigpu, oracle_mod, physics):
    """Non-zero constrained data y_c: rhs = K ybar + K_c y_c (control.cpp:15)."""
    from paper_1312_5653_b200 import box

    n, s, phi = 12, 3, 1e-4
    p = box.make_box_problem(n, phi=phi, physics=physics, young=1.0, poisson=0.3, seed=4)
    q = oracle_mod.Problem(n, n, n_z=n, physics=physics, young=1.0, poisson=0.3)
    yc = np.random.default_rng(7).standard_normal(q.m)
    solver = box.BoxSchurSolver(p, s, tol=1e-10, max_iter=500)
    try:
        r = solver.solve(p.target_state, yc)
    finally:
        solver.close()
    o = q.schur_solve(s, s, phi, p.target_state, yc, s_z=s, tol=1e-10, max_iter=500)
    for k in ("y", "u", "lambda"):
        assert rel(r[k], o[k]) <= 1e-8, k


@pytest.mark.gpu
@pytest.mark.parametrize("physics,mass_coeff", [(0, 100.0), (1, 10.0 + 5.0j)])
def test_gpu3d_feti_solve_mass_coeff(fetigpu, oracle_mod, physics, mass_coeff):
    """feti_solve with an explicit mass coefficient (python feti_solve, bindings.cpp:158-185),
    e.g. the real Pearson-Wathen factor K + V / sqrt(phi)."""
    from paper_1312_5653_b200 import box

    n, s = 12, 3
    p = box.make_box_problem(n, phi=1e-4, physics=physics, young=1.0, poisson=0.3, seed=6)
    q = oracle_mod.Problem(n, n, n_z=n, physics=physics, young=1.0, poisson=0.3)
    rhs = np.random.default_rng(11).standard_normal(p.n).astype(complex)
    x, st = box.feti_solve_3d(p, mass_coeff, rhs, s, tol=1e-10, max_iter=500)
    xr, sr = oracle_mod.Feti(q, s, s, mass_coeff, s_z=s, tol=1e-10, max_iter=500).solve(rhs)
    assert st["converged"] and sr["converged"]
    assert rel(x, xr) <= 1e-8
    assert abs(st["iterations"] - sr["iterations"]) <= 2


@pytest.mark.gpu
@pytest.mark.parametrize("physics,grid", [(0, (1, 1, 2)), (0, (2, 1, 1)), (1, (2, 1, 1)), (0, (3, 2, 1))])
def test_gpu3d_anisotropic_subdomain_grids(fetigpu, oracle_mod, physics, grid):
    """Slab partitions (1 x 1 x 2 heat: no corner at all, the coarse problem is empty) and
    anisotropic subdomain grids against the oracle."""
    from paper_1312_5653_b200 import box

    n, phi = 12, 1e-4
    sx, sy, sz = grid
    p = box.make_box_problem(n, phi=phi, physics=physics, young=1.0, poisson=0.3, seed=8)
    q = oracle_mod.Problem(n, n, n_z=n, physics=physics, young=1.0, poisson=0.3)
    solver = box.BoxSchurSolver(p, sx, sy, sz, tol=1e-10, max_iter=500)
    try:
        r = solver.solve()
        nc = solver.coarse_dim
    finally:
        solver.close()
    o = q.schur_solve(sx, sy, phi, p.target_state, s_z=sz, tol=1e-10, max_iter=500)
    if grid == (1, 1, 2) and physics == 0:
        assert nc == 0
    for k in ("y", "u", "lambda"):
        assert rel(r[k], o[k]) <= 1e-8, k
    assert abs(r["plus_stats"]["iterations"] - o["plus_stats"]["iterations"]) <= 2


@pytest.mark.gpu
def test_gpu3d_zero_rhs_and_contracts(fetigpu):
    from paper_1312_5653_b200 import ContractError, box

    p = box.make_box_problem(8, phi=1e-4)
    solver = box.BoxSchurSolver(p, 2)
    try:
        x, st = solver.feti_solve(np.zeros(p.n, dtype=complex))
        assert st["iterations"] == 0 and st["converged"] and not np.any(x)
        with pytest.raises(ContractError):
            solver.solve(np.zeros(p.n + 1))
    finally:
        solver.close()
    with pytest.raises(ContractError):
        box.BoxSchurSolver(box.make_box_problem(8, phi=1e-4), 3)  # 3 does not divide 8


# ---------------------------------------------------------------------------------------
# The BASELINE subdomain shapes (16^3 elements per subdomain) against committed oracle
# fixtures (tests/golden/make_3d_golden.py), and the full config-4/5 sizes through
# size-independent properties.
GOLDEN = {"heat48": dict(n=48, s=3, phi=1e-6, physics=0), "elast32": dict(n=32, s=2, phi=1e-4, physics=1)}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_gpu3d_config_subdomain_size_matches_golden(fetigpu, name):
    import os

    from paper_1312_5653_b200 import box

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden3d.npz"))
    c = GOLDEN[name]
    p = box.make_box_problem(c["n"], phi=c["phi"], physics=c["physics"], young=1.0, poisson=0.3, seed=0)
    assert abs(np.linalg.norm(p.target_state) - float(g[f"{name}_ybar_norm"])) <= 1e-12 * float(g[f"{name}_ybar_norm"])
    r = box.solve_range_space_3d(p, c["s"], tol=1e-10, max_iter=2000)
    assert r["converged"]
    for k in ("y", "u", "lambda"):
        assert rel(r[k], g[f"{name}_{k}"]) <= 1e-8, k
    its = g[f"{name}_iters"]
    assert abs(r["plus_stats"]["iterations"] - int(its[0])) <= 2
    assert abs(r["minus_stats"]["iterations"] - int(its[1])) <= 2


def kkt_residuals(oracle_mod, cfg, r, ybar):
    """State equation K y - V u (relative to |K ybar|; equals the Schur residual
    K ybar - S lambda) and adjoint equation V (y - ybar) + K lambda (relative to |K lambda|),
    with the exact operators assembled by the oracle (control.cpp:56-59)."""
    q = oracle_mod.Problem(cfg["n"], cfg["n"], n_z=cfg["n"], physics=cfg["physics"], young=1.0, poisson=0.3)
    ky = q.apply(0, r["y"])
    vu = q.apply(1, r["u"])
    kyb = q.apply(0, ybar)
    kl = q.apply(0, r["lambda"])
    vd = q.apply(1, r["y"] - ybar)
    return np.linalg.norm(ky - vu) / np.linalg.norm(kyb), np.linalg.norm(vd + kl) / np.linalg.norm(kl)


FULL = {4: dict(n=128, s=8, phi=1e-6, physics=0, state_tol=1e-8),
        5: dict(n=64, s=4, phi=1e-4, physics=1, state_tol=1e-6)}


def projections(v, nproj):
    """The digest's projections onto seeded N(0,1) vectors (tests/golden/make_3d_digest.py)."""
    g = np.random.default_rng(2024)
    return np.array([g.standard_normal(v.size) @ v for _ in range(nproj)])


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("config", [4, 5])
def test_gpu3d_full_config_properties(fetigpu, oracle_mod, config):
    from paper_1312_5653_b200 import box

    c = FULL[config]
    p = box.make_box_problem(c["n"], phi=c["phi"], physics=c["physics"], young=1.0, poisson=0.3, seed=0)
    solver = box.BoxSchurSolver(p, c["s"], tol=1e-10, max_iter=2000)
    try:
        r = solver.solve()
        r2 = solver.solve()
    finally:
        solver.close()
    assert r["converged"] and r["imag_leak"] <= 1e-6
    assert r["plus_stats"]["iterations"] == r["minus_stats"]["iterations"]  # conjugate pair
    for k in ("y", "u", "lambda"):  # deterministic: fixed-order reductions, no atomics
        assert np.array_equal(r[k], r2[k]), k
    state, adjoint = kkt_residuals(oracle_mod, c, r, p.target_state)
    assert state <= c["state_tol"], state
    assert adjoint <= 1e-10, adjoint
    # parity at full size: the oracle's own config-4/5 solve (tests/golden/make_3d_digest.py;
    # norms, 4096 sampled entries, 32 random projections = a relative-L2 estimate of the
    # whole difference, iteration counts +-2)
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "config45_digest.npz")
    d = np.load(path)
    tag = f"c{config}"
    assert abs(np.linalg.norm(p.target_state) - float(d[f"{tag}_ybar_norm"])) <= 1e-12 * float(d[f"{tag}_ybar_norm"])
    idx = d[f"{tag}_sample_index"]
    for k in ("y", "u", "lambda"):
        norm = float(d[f"{tag}_{k}_norm"])
        assert abs(np.linalg.norm(r[k]) - norm) <= 1e-8 * norm, k
        assert rel(r[k][idx], d[f"{tag}_{k}_sample"]) <= 1e-8, k
        pd = projections(r[k], d[f"{tag}_{k}_proj"].size) - d[f"{tag}_{k}_proj"]
        assert np.sqrt(np.mean(pd ** 2)) <= 1e-8 * norm, k
    its = d[f"{tag}_iters"]
    assert abs(r["plus_stats"]["iterations"] - int(its[0])) <= 2
    assert abs(r["minus_stats"]["iterations"] - int(its[1])) <= 2


@pytest.mark.gpu
def test_gpu3d_nonconvergence_is_not_an_error(fetigpu, oracle_mod):
    """max_iter reached: converged = false, iterations = max_iter, the same iterate and
    relative residual as the oracle (krylov.hpp:97-100)."""
    from paper_1312_5653_b200 import box

    n, s, phi = 12, 3, 1e-4
    p = box.make_box_problem(n, phi=phi, seed=1)
    rhs = np.random.default_rng(9).standard_normal(p.n).astype(complex)
    x, st = box.feti_solve_3d(p, -1j / np.sqrt(phi), rhs, s, tol=1e-12, max_iter=3)
    xr, sr = oracle_mod.Feti(oracle_mod.Problem(n, n, n_z=n), s, s, -1j / np.sqrt(phi), s_z=s, tol=1e-12,
                             max_iter=3).solve(rhs)
    assert not st["converged"] and st["iterations"] == 3
    assert not sr["converged"] and sr["iterations"] == 3
    assert abs(st["relative_residual"] - sr["relative_residual"]) <= 1e-6 * sr["relative_residual"]
    assert rel(x, xr) <= 1e-8


@pytest.mark.gpu
@pytest.mark.parametrize("switch", ["FETIGPU3D_NO_FDM", "FETIGPU_NO_STENCIL"])
def test_gpu3d_fast_paths_agree_with_plain_paths(fetigpu, monkeypatch, switch):
    """3D heat: the separable interior solve (FETIGPU3D_NO_FDM keeps the block-band
    substitution) and the 27-point stencil global applies (FETIGPU_NO_STENCIL keeps the
    element-by-element apply) against the plain paths: same iterations, equal to rounding."""
    from paper_1312_5653_b200 import box

    p = box.make_box_problem(16, phi=1e-4, seed=2)
    out = []
    for plain in (False, True):
        if plain:
            monkeypatch.setenv(switch, "1")
        s = box.BoxSchurSolver(p, 2, tol=1e-10, max_iter=500)
        out.append(s.solve())
        s.close()
    a, b = out
    for side in ("plus_stats", "minus_stats"):
        assert a[side]["iterations"] == b[side]["iterations"]
    for k in ("y", "u", "lambda"):
        assert np.linalg.norm(a[k] - b[k]) <= 1e-11 * np.linalg.norm(b[k]), k
