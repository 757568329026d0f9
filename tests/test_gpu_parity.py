"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle and dense
direct solves.  Re-expresses the reference's hot-path tests:
test_feti.cpp:300-351, test_control.cpp:141-163, verify.cpp:150-191, test_smoke.py:48-58.

Tolerances: north_star parity is relative L2 <= 1e-8 in u, y, lambda at the same Krylov
tolerance with iteration counts within +-2; operator applications agree to 1e-12.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def dense_kkt_solution(orc_problem, phi, ybar, yc):
    K, V, Kc = orc_problem.dense(0), orc_problem.dense(1), orc_problem.dense(2)
    n = orc_problem.n
    A = np.zeros((3 * n, 3 * n))
    A[:n, :n] = V
    A[:n, 2 * n:] = K
    A[n:2 * n, n:2 * n] = phi * V
    A[n:2 * n, 2 * n:] = -V
    A[2 * n:, :n] = K
    A[2 * n:, n:2 * n] = -V
    rhs = np.zeros(3 * n)
    rhs[:n] = V @ ybar
    if yc is not None and len(yc):
        rhs[2 * n:] = -(Kc @ yc)
    x = np.linalg.solve(A, rhs)
    return x[:n], x[n:2 * n], x[2 * n:]


@pytest.mark.parametrize("n,s", [(16, 2), (32, 4), (64, 4)])
@pytest.mark.parametrize("phi", [2e-8, 1e-4])
def test_operators_match_oracle(fetigpu, oracle_mod, n, s, phi):
    """apply_dual_operator / apply_dirichlet_preconditioner (feti.cpp:581-627)."""
    p = fetigpu.make_seeded_problem(n, phi)
    c = -1j / np.sqrt(phi)
    gpu = fetigpu.SchurSolver(p, s, s, tol=1e-10)
    ref = oracle_mod.Feti(oracle_mod.Problem(n), s, s, c)
    assert gpu.n_lambda == ref.n_lambda
    rng = np.random.default_rng(7)
    lam = rng.uniform(-1, 1, ref.n_lambda) + 1j * rng.uniform(-1, 1, ref.n_lambda)
    for sign, coeff in ((1, c), (-1, -c)):
        r = ref if sign == 1 else oracle_mod.Feti(oracle_mod.Problem(n), s, s, coeff)
        assert rel(gpu.apply_dual_operator(lam, sign), r.apply_dual_operator(lam)) <= 1e-12
        assert rel(gpu.apply_dirichlet_preconditioner(lam, sign), r.apply_dirichlet_preconditioner(lam)) <= 1e-12
    gpu.close()


def test_feti_complex_factors_match_direct(fetigpu, oracle_mod):
    """test_feti.cpp:309-332: n=16, 2x2, phi=2e-8, tol 1e-10, <=1e-8, with the reference test's
    augment=true on both sides (the GPU's and the oracle's edge-RBM coarse spaces), and the
    same case with augment=false."""
    n, phi = 16, 2e-8
    p = fetigpu.make_seeded_problem(n, phi)
    op = oracle_mod.Problem(n)
    K, V = op.dense(0), op.dense(1)
    rng = np.random.default_rng(29)
    rhs = rng.uniform(-1, 1, op.n).astype(complex)
    c = -1j / np.sqrt(phi)
    for augment in (True, False):
        for coeff in (c, -c):
            out = fetigpu.feti_solve(p, coeff, rhs, s_x=2, s_y=2, tol=1e-10, augment=augment)
            assert out["converged"]
            direct = np.linalg.solve(K + coeff * V, rhs)
            assert rel(out["x"], direct) <= 1e-8
            assert out["interface_jump"] <= 1e-8
            xo, so = oracle_mod.Feti(op, 2, 2, coeff, tol=1e-10, augment=augment).solve(rhs)
            assert abs(out["iterations"] - so["iterations"]) <= 2
            assert rel(out["x"], xo) <= 1e-8


def test_feti_criterion5_n32(fetigpu, oracle_mod):
    """verify.cpp:150-191: n=32, 4x4, phi=2e-8, tol 1e-10, FETI vs direct <= 1e-8, jump <= 1e-8."""
    n, phi = 32, 2e-8
    p = fetigpu.make_thermal_problem(n, phi)
    op = oracle_mod.Problem(n)
    K, V, Kc = op.dense(0), op.dense(1), op.dense(2)
    rhs = (K @ op.target_thermal() + Kc @ op.boundary_thermal()).astype(complex)
    c = -1j / np.sqrt(phi)
    for coeff in (c, -c):
        out = fetigpu.feti_solve(p, coeff, rhs, s_x=4, s_y=4, tol=1e-10)
        assert out["converged"]
        direct = np.linalg.solve(K + coeff * V, rhs)
        assert rel(out["x"], direct) <= 1e-8
        assert out["interface_jump"] <= 1e-8 * np.abs(out["x"]).max()


def test_conjugate_pair_iterations(fetigpu):
    """test_feti.cpp:334-351: the two conjugate factors need iteration counts within 2."""
    n, phi = 16, 2e-6
    p = fetigpu.make_seeded_problem(n, phi)
    rng = np.random.default_rng(31)
    rhs = rng.uniform(-1, 1, p.n).astype(complex)
    c = -1j / np.sqrt(phi)
    its = [fetigpu.feti_solve(p, coeff, rhs, tol=1e-10)["iterations"] for coeff in (c, -c)]
    assert abs(its[0] - its[1]) <= 2


def test_feti_zero_rhs(fetigpu):
    """test_feti.cpp:300-307: zero rhs -> zero solution in zero iterations."""
    p = fetigpu.make_seeded_problem(8, 1e-4)
    out = fetigpu.feti_solve(p, -1j * 100.0, np.zeros(p.n, dtype=complex))
    assert out["iterations"] == 0 and out["converged"]
    assert np.linalg.norm(out["x"]) == 0.0


def test_range_space_matches_dense_kkt_n8(fetigpu, oracle_mod):
    """test_control.cpp:152-163 / test_smoke.py:25-38: n=8, phi=2e-5, <= 1e-8."""
    n, phi = 8, 2e-5
    p = fetigpu.make_thermal_problem(n, phi)
    out = fetigpu.solve_range_space(p, tol=1e-12)
    assert out["converged"] and not out["imag_leak_warning"]
    y, u, lam = dense_kkt_solution(oracle_mod.Problem(n), phi, p.target_state, p.boundary_values)
    assert rel(out["y"], y) <= 1e-8
    assert rel(out["u"], u) <= 1e-8
    assert rel(out["lambda"], lam) <= 1e-8


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_config1_schur_matches_oracle(fetigpu, oracle_mod, seed):
    """BASELINE config 1: 64x64 Q1, 4x4 subdomains, phi=1e-4, seeded sine target, tol 1e-10."""
    n, s, phi = 64, 4, 1e-4
    p = fetigpu.make_seeded_problem(n, phi, seed=seed)
    op = oracle_mod.Problem(n)
    ybar = op.target_sine(seed)
    assert np.array_equal(ybar, p.target_state)
    ref = op.schur_solve(s, s, phi, ybar, None, tol=1e-10, max_iter=2000, threads=4)
    solver = fetigpu.SchurSolver(p, s, s, tol=1e-10, max_iter=2000)
    out = solver.solve()
    solver.close()
    assert out["converged"]
    for k in ("y", "u", "lambda"):
        assert rel(out[k], ref[k]) <= 1e-8, k
    assert abs(out["plus_stats"]["iterations"] - ref["plus_stats"]["iterations"]) <= 2
    assert abs(out["minus_stats"]["iterations"] - ref["minus_stats"]["iterations"]) <= 2


def test_schur_solver_reuse_is_deterministic(fetigpu):
    """Factor once, solve twice: bit-identical results (verify.cpp:354-369 determinism)."""
    p = fetigpu.make_seeded_problem(64, 1e-4)
    solver = fetigpu.SchurSolver(p, 4, 4, tol=1e-10)
    a = solver.solve()
    b = solver.solve()
    solver.close()
    for k in ("y", "u", "lambda"):
        assert np.array_equal(a[k], b[k])


def test_graph_and_eager_gmres_identical(fetigpu):
    """The CUDA-graph (conditional WHILE) Arnoldi loop and the eager step-by-step loop
    (profiling mode) launch the same kernels: results must be bit-identical."""
    p = fetigpu.make_seeded_problem(64, 1e-6, seed=5)
    solver = fetigpu.SchurSolver(p, 4, 4, tol=1e-10)
    a = solver.solve()
    solver.profile(True)
    b = solver.solve()
    prof = solver.profile_read()
    solver.profile(False)
    solver.close()
    assert prof["dual_gemv"]["launches"] > 0
    for k in ("y", "u", "lambda"):
        assert np.array_equal(a[k], b[k])
    assert a["plus_stats"]["iterations"] == b["plus_stats"]["iterations"]


@pytest.mark.parametrize("n,s", [(80, 2), (136, 34)])
def test_wide_bands_match_oracle(fetigpu, oracle_mod, n, s):
    """Half-bandwidths above one warp (NS = 2 register window): A_ii with W = 39 (80^2, 2x2)
    and the coarse matrix with W = 34 (136^2, 34x34 subdomains)."""
    phi = 1e-6
    p = fetigpu.make_seeded_problem(n, phi, seed=4)
    c = -1j / np.sqrt(phi)
    gpu = fetigpu.SchurSolver(p, s, s, tol=1e-10, max_iter=2000)
    ref = oracle_mod.Feti(oracle_mod.Problem(n), s, s, c, tol=1e-10, max_iter=2000)
    rng = np.random.default_rng(11)
    lam = rng.uniform(-1, 1, ref.n_lambda) + 1j * rng.uniform(-1, 1, ref.n_lambda)
    assert rel(gpu.apply_dual_operator(lam), ref.apply_dual_operator(lam)) <= 1e-12
    assert rel(gpu.apply_dirichlet_preconditioner(lam), ref.apply_dirichlet_preconditioner(lam)) <= 1e-12
    rhs = rng.uniform(-1, 1, p.n) + 0j
    x, st = gpu.feti_solve(rhs)
    xo, so = ref.solve(rhs)
    assert rel(x, xo) <= 1e-8
    assert abs(st["iterations"] - so["iterations"]) <= 2
    gpu.close()


def test_plane_strain_matches_oracle(fetigpu, oracle_mod):
    """Plane-strain elasticity (dpn = 2, clamped x = 0, fem.cpp:83-128):
    W = 64 interior bands (banded substitution path), 8 corner dofs per subdomain, free
    top/bottom/right boundaries (ragged interiors).  Operators to 1e-12, Schur solve to 1e-8."""
    n_x, n_y, s_x, s_y, phi = 48, 32, 6, 4, 1e-4
    p = fetigpu.make_problem(n_x, n_y, phi, physics=1, len_x=1.5, len_y=1.0, young=1.0, poisson=0.3)
    op = oracle_mod.Problem(n_x, n_y, len_x=1.5, len_y=1.0, physics=1, young=1.0, poisson=0.3)
    assert op.n == p.n
    rng = np.random.default_rng(3)
    ybar = rng.standard_normal(p.n)
    ref = op.schur_solve(s_x, s_y, phi, ybar, None, tol=1e-10, max_iter=2000, threads=4)
    solver = fetigpu.SchurSolver(p, s_x, s_y, tol=1e-10, max_iter=2000)
    out = solver.solve(ybar, np.zeros(p.m))  # y_c = 0 (None would take the problem's trace)
    feti = oracle_mod.Feti(op, s_x, s_y, -1j / np.sqrt(phi), tol=1e-10, max_iter=2000)
    lam = rng.uniform(-1, 1, feti.n_lambda) + 1j * rng.uniform(-1, 1, feti.n_lambda)
    assert rel(solver.apply_dual_operator(lam), feti.apply_dual_operator(lam)) <= 1e-12
    assert rel(solver.apply_dirichlet_preconditioner(lam), feti.apply_dirichlet_preconditioner(lam)) <= 1e-12
    solver.close()
    assert out["converged"]
    for k in ("y", "u", "lambda"):
        assert rel(out[k], ref[k]) <= 1e-8, k
    assert abs(out["plus_stats"]["iterations"] - ref["plus_stats"]["iterations"]) <= 2
    assert abs(out["minus_stats"]["iterations"] - ref["minus_stats"]["iterations"]) <= 2


@pytest.mark.parametrize("n,s,phi", [(16, 2, 2e-8), (64, 4, 1e-4), (128, 8, 1e-6)])
def test_augmented_feti_matches_oracle(fetigpu, oracle_mod, n, s, phi):
    """Edge-RBM augmentation: augmented coupling/coarse (dense, pivoted),
    projected dual space.  Operators, FETI solves and iteration counts vs the oracle."""
    p = fetigpu.make_seeded_problem(n, phi, seed=2)
    c = -1j / np.sqrt(phi)
    gpu = fetigpu.SchurSolver(p, s, s, tol=1e-10, max_iter=2000, augment=True)
    ref = oracle_mod.Feti(oracle_mod.Problem(n), s, s, c, tol=1e-10, max_iter=2000, augment=True)
    rng = np.random.default_rng(17)
    lam = rng.uniform(-1, 1, ref.n_lambda) + 1j * rng.uniform(-1, 1, ref.n_lambda)
    assert rel(gpu.apply_dual_operator(lam), ref.apply_dual_operator(lam)) <= 1e-11
    assert rel(gpu.apply_dirichlet_preconditioner(lam), ref.apply_dirichlet_preconditioner(lam)) <= 1e-12
    rhs = rng.uniform(-1, 1, p.n) + 0j
    x, st = gpu.feti_solve(rhs)
    xo, so = ref.solve(rhs)
    gpu.close()
    assert st["converged"] and so["converged"]
    assert rel(x, xo) <= 1e-8
    assert abs(st["iterations"] - so["iterations"]) <= 2


def test_augmented_spans_interface_zero_iterations(fetigpu, oracle_mod):
    """test_feti.cpp:407-425: H/h = 2, the edge modes span the whole interface."""
    p = fetigpu.make_seeded_problem(16, 1e-4, seed=0)
    gpu = fetigpu.SchurSolver(p, 8, 8, tol=1e-10, max_iter=100, augment=True)
    rhs = np.random.default_rng(53).standard_normal(p.n) + 0j
    x, st = gpu.feti_solve(rhs)
    gpu.close()
    ref = oracle_mod.Feti(oracle_mod.Problem(16), 8, 8, -1j / np.sqrt(1e-4), tol=1e-10, augment=True)
    xo, so = ref.solve(rhs)
    assert st["converged"] and st["iterations"] == 0 == so["iterations"]
    assert rel(x, xo) <= 1e-9


def test_augmented_schur_matches_oracle(fetigpu, oracle_mod):
    """Range-space Schur solve with augmentation, config-1 mesh, vs the oracle."""
    n, s, phi = 64, 4, 1e-4
    p = fetigpu.make_seeded_problem(n, phi, seed=1)
    ref = oracle_mod.Problem(n).schur_solve(s, s, phi, p.target_state, None, tol=1e-10, max_iter=2000, threads=4,
                                            augment=True)
    solver = fetigpu.SchurSolver(p, s, s, tol=1e-10, max_iter=2000, augment=True)
    out = solver.solve()
    solver.close()
    assert out["converged"]
    for k in ("y", "u", "lambda"):
        assert rel(out[k], ref[k]) <= 1e-8, k
    assert abs(out["plus_stats"]["iterations"] - ref["plus_stats"]["iterations"]) <= 2
    assert abs(out["minus_stats"]["iterations"] - ref["minus_stats"]["iterations"]) <= 2


@pytest.mark.gpu
def test_schur_zero_target_deferred_path(fetigpu):
    """A zero target through the Schur solve (the deferred-GMRES graph path): zero y, u,
    lambda, converged in 0 iterations for both factors (feti.cpp:640-644); then a regular
    solve on the same context is unaffected."""
    p = fetigpu.make_seeded_problem(64, 1e-4, seed=0)
    solver = fetigpu.SchurSolver(p, 4, 4, tol=1e-10, max_iter=500)
    try:
        z = solver.solve(np.zeros(p.n))
        assert z["converged"]
        assert z["plus_stats"]["iterations"] == 0 and z["minus_stats"]["iterations"] == 0
        for k in ("y", "u", "lambda"):
            assert not np.any(z[k]), k
        r1 = solver.solve()
        r2 = solver.solve()
        assert r1["converged"] and r1["plus_stats"]["iterations"] > 0
        for k in ("y", "u", "lambda"):
            assert np.array_equal(r1[k], r2[k]), k
    finally:
        solver.close()


@pytest.mark.gpu
def test_nonconvergence_is_not_an_error(fetigpu, oracle_mod):
    """krylov.hpp:97-100: hitting max_iter returns converged = false with the best iterate
    (rc 0), iterations = max_iter; the oracle agrees on the count and the relative residual."""
    n, s, phi = 64, 4, 1e-4
    p = fetigpu.make_seeded_problem(n, phi, seed=0)
    rhs = np.random.default_rng(5).standard_normal(p.n).astype(complex)
    solver = fetigpu.SchurSolver(p, s, s, tol=1e-10, max_iter=4, mass_coeff=-1j / np.sqrt(phi))
    try:
        x, st = solver.feti_solve(rhs)
    finally:
        solver.close()
    assert not st["converged"] and st["iterations"] == 4
    assert np.all(np.isfinite(x))
    ref_x, ref = oracle_mod.Feti(oracle_mod.Problem(n), s, s, -1j / np.sqrt(phi), tol=1e-10, max_iter=4).solve(rhs)
    assert not ref["converged"] and ref["iterations"] == 4
    assert abs(st["relative_residual"] - ref["relative_residual"]) <= 1e-6 * ref["relative_residual"]
    assert np.linalg.norm(x - ref_x) <= 1e-8 * np.linalg.norm(ref_x)


@pytest.mark.parametrize("switch", ["FETIGPU_NO_ZBASIS", "FETIGPU_NO_RI_COMPACT", "FETIGPU_NO_ELIM_REUSE",
                                    "FETIGPU_NO_DEFER", "FETIGPU_NO_SPLIT", "FETIGPU_NO_FDM",
                                    "FETIGPU_COOP_REJECT", "FETIGPU_NO_FUSED_TAIL", "FETIGPU_NO_PDL",
                                    "FETIGPU_EAGER", "FETIGPU_NO_AIC", "FETIGPU_NO_STENCIL", "FETIGPU_NO_BT",
                                    "FETIGPU_NO_ASIDE", "FETIGPU_ASIDE_GIVEUP", "FETIGPU_NO_TAIL_PF", "FETIGPU_TAIL_HCS", "FETIGPU_TAIL_MR", "FETIGPU_BASIS0",
                                    "FETIGPU_BASIS0+FETIGPU_EAGER", "FETIGPU_BASIS0+FETIGPU_NO_DEFER", "FETIGPU_NO_PREFIX",
                                    "FETIGPU_NO_PREFIX+FETIGPU_NO_SPLIT"])
def test_fast_paths_agree_with_plain_paths(fetigpu, monkeypatch, switch):
    """Each reuse/fusion of the solve path (preconditioned basis Z, compact interior rhs,
    GEMV-free final elimination, deferred GMRES completion, Givens folded into the next
    GEMV, the cooperative fused Arnoldi tail -- FETIGPU_COOP_REJECT makes the setup's
    cooperative-launch probe act as rejected, as under an MPS SM limit, so the step falls
    back to the multi-launch tail; the coarse solve beside the dual GEMV -- FETIGPU_NO_ASIDE
    keeps it in the tail, FETIGPU_ASIDE_GIVEUP makes the coarse CTAs miss their arrivals and
    give up, so the tail computes z itself; FETIGPU_TAIL_MR forces the multi-row tail that
    large interfaces use; FETIGPU_BASIS0 starts with a Krylov basis of 4 vectors, so every cycle
    is continued several times on a larger basis -- bitwise the same iteration) against the
    plain path it replaces: same iterations, results equal to rounding."""
    p = fetigpu.make_seeded_problem(128, 1e-4, seed=3)
    solver = fetigpu.SchurSolver(p, 8, 8, tol=1e-10)
    a = solver.solve()
    solver.close()
    for sw in switch.split("+"):  # HCS: dot vectors beyond 4 entries in global scratch; BASIS0: 4 basis vectors
        monkeypatch.setenv(sw, "4" if sw in ("FETIGPU_TAIL_HCS", "FETIGPU_BASIS0") else "1")
    solver = fetigpu.SchurSolver(p, 8, 8, tol=1e-10)
    b = solver.solve()
    solver.close()
    for side in ("plus_stats", "minus_stats"):
        assert a[side]["iterations"] == b[side]["iterations"]
    for k in ("y", "u", "lambda"):
        assert rel(a[k], b[k]) <= 1e-11, k
        if switch == "FETIGPU_BASIS0":  # the continued cycle is the same arithmetic
            assert np.array_equal(a[k], b[k]), k


def test_prefix_graphs_reproduce_the_while_loop(fetigpu, monkeypatch):
    """From its second solve on a context runs each GMRES cycle on a graph with (last iteration
    count) unconditional Arnoldi steps in front of the WHILE node.  Targets with different
    iteration counts (phi-scaled copies and other seeds), solved in sequence on one context,
    must equal the WHILE-only path (FETIGPU_NO_PREFIX) bit for bit."""
    n, s, phi = 96, 6, 1e-4
    p = fetigpu.make_seeded_problem(n, phi, seed=0)
    targets = [fetigpu.make_seeded_problem(n, phi, seed=k).target_state for k in range(5)]
    targets.append(np.zeros_like(targets[0]))  # zero target: 0 iterations, then a normal one again
    targets.append(targets[1])

    def run():
        solver = fetigpu.SchurSolver(p, s, s, tol=1e-10)
        outs = [solver.solve(t) for t in targets]
        solver.close()
        return outs

    a = run()
    monkeypatch.setenv("FETIGPU_NO_PREFIX", "1")
    b = run()
    for x, y in zip(a, b):
        assert x["plus_stats"]["iterations"] == y["plus_stats"]["iterations"]
        assert x["minus_stats"]["iterations"] == y["minus_stats"]["iterations"]
        for k in ("y", "u", "lambda"):
            assert np.array_equal(x[k], y[k]), k


@pytest.mark.parametrize("n,s", [(36, 4), (40, 4), (66, 3)])
def test_separable_solve_even_odd_grids(fetigpu, monkeypatch, n, s):
    """Separable interior solve on even and odd interior line lengths (m = n/s - 1 = 8, 9,
    21) against the block-Thomas path."""
    p = fetigpu.make_seeded_problem(n, 1e-4, seed=1)
    solver = fetigpu.SchurSolver(p, s, s, tol=1e-10)
    a = solver.solve()
    solver.close()
    monkeypatch.setenv("FETIGPU_NO_FDM", "1")
    solver = fetigpu.SchurSolver(p, s, s, tol=1e-10)
    b = solver.solve()
    solver.close()
    for side in ("plus_stats", "minus_stats"):
        assert a[side]["iterations"] == b[side]["iterations"]
    for k in ("y", "u", "lambda"):
        assert rel(a[k], b[k]) <= 1e-11, k


def test_packed_coarse_inverse_agrees_with_dense(fetigpu, monkeypatch):
    """Coarse spaces of >= 1536 corners keep C^-1 packed symmetric (half the bytes of the
    per-step coarse GEMV); FETIGPU_DENSE_COARSE keeps the dense inverse.  41 x 41 subdomains
    of 4 x 4 elements: 1600 corners."""
    p = fetigpu.make_seeded_problem(164, 1e-4, seed=5)
    out = []
    for dense in (False, True):
        if dense:
            monkeypatch.setenv("FETIGPU_DENSE_COARSE", "1")
        solver = fetigpu.SchurSolver(p, 41, 41, tol=1e-10)
        assert solver.coarse_dim == 1600
        out.append(solver.solve())
        solver.close()
    a, b = out
    for side in ("plus_stats", "minus_stats"):
        assert a[side]["iterations"] == b[side]["iterations"]
    for k in ("y", "u", "lambda"):
        assert rel(a[k], b[k]) <= 1e-11, k
