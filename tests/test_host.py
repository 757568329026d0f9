"""CPU tests of the product's host side: the C-ABI library loads and exports every
symbol of include/fetigpu.h, and the C++ host core (mesh, partition, targets) agrees
with the oracle.  No kernel is launched (no GPU in this container)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "fetigpu.h")).read()
    return sorted(set(re.findall(r"\b(fetigpu(?:3d)?_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol(fetigpu):
    import ctypes

    from paper_1312_5653_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTED_SYMBOLS)


def test_library_is_sm100a(fetigpu):
    import subprocess

    from paper_1312_5653_b200 import _native

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n,s", [(8, 2), (16, 2), (32, 4), (64, 4), (128, 8), (1024, 32), (2048, 64)])
def test_partition_matches_oracle(fetigpu, oracle_mod, n, s):
    p = fetigpu.make_problem(n, n, 1e-4, target="sine")
    info = fetigpu.partition_info(p, s, s)
    ref = oracle_mod.Problem(n).partition_info(s, s) if n <= 1024 else None
    if ref:
        for k in ("n_subdomains", "n_corner_dofs", "n_lambda", "n_edges", "ex", "ey"):
            assert info[k] == ref[k], k
    if n == 2048:
        assert (info["n_subdomains"], info["n_corner_dofs"], info["n_lambda"], info["n_edges"]) == (
            4096, 3969, 249984, 8064)
        assert info["band_halfwidth"] == 32


def test_partition_sizes_rectangles(fetigpu, oracle_mod):
    for nx, ny, sx, sy in ((16, 8, 4, 2), (24, 12, 3, 2), (8, 8, 1, 2), (12, 8, 2, 4)):
        p = fetigpu.make_problem(nx, ny, 1e-4, len_x=nx / 8.0, len_y=ny / 8.0)
        info = fetigpu.partition_info(p, sx, sy)
        ref = oracle_mod.Problem(nx, ny, nx / 8.0, ny / 8.0).partition_info(sx, sy)
        assert all(info[k] == ref[k] for k in ref), (nx, ny, sx, sy)


def test_targets_match_oracle_bitwise(fetigpu, oracle_mod):
    for n in (8, 64, 256):
        p = fetigpu.make_thermal_problem(n, 1e-4)
        o = oracle_mod.Problem(n)
        assert np.array_equal(p.target_state, o.target_thermal())
        assert np.array_equal(p.boundary_values, o.boundary_thermal())
        for seed in (0, 1, 2):
            q = fetigpu.make_seeded_problem(n, 1e-4, seed=seed)
            assert np.array_equal(q.target_state, o.target_sine(seed))


def test_sine_modes_recipe(oracle_mod):
    """mt19937_64(seed), Box-Muller amplitudes, modes in 1..8."""
    a, m, n = oracle_mod.sine_modes(0)
    assert a.shape == (8,) and np.all((m >= 1) & (m <= 8)) and np.all((n >= 1) & (n <= 8))
    a1, _, _ = oracle_mod.sine_modes(1)
    assert not np.array_equal(a, a1)


def test_contract_errors(fetigpu):
    F = fetigpu
    with pytest.raises(ValueError):
        F.make_thermal_problem(1, 1e-4)  # test_smoke.py:81-83
    with pytest.raises(ValueError):
        F.make_thermal_problem(8, 0.0)
    p = F.make_thermal_problem(6, 1e-4)
    for sx, sy in ((4, 2), (6, 6), (1, 1)):  # test_feti.cpp:70-77
        with pytest.raises(ValueError):
            F.partition_info(p, sx, sy)
    # augmentation: a one-node edge has no rotation mode (feti.cpp:219-222) -> NumericalError,
    # raised by the host partition before any device work
    q = F.make_problem(12, 4, 1e-4, physics=1, len_x=3.0, len_y=1.0, young=20.7e6, poisson=0.45)
    with pytest.raises(RuntimeError, match="rotation"):
        F.SchurSolver(q, 2, 2, augment=True)
    with pytest.raises(ValueError):
        F.solve_range_space(F.make_thermal_problem(8, 1e-4), method="direct")


def test_problem_sizes(fetigpu):
    p = fetigpu.make_thermal_problem(4, 1e-3)
    assert (p.n, p.m) == (9, 16)  # test_mesh_fem.cpp:128-133
    q = fetigpu.make_problem(12, 4, 1e-4, physics=1, len_x=3.0, len_y=1.0, young=20.7e6, poisson=0.45)
    assert (q.n, q.m) == (2 * 12 * 5, 2 * 5)  # clamped x = 0 edge (fem.cpp:124-128)


def _dst(m):
    i = np.arange(1, m + 1)
    return np.sqrt(2.0 / (m + 1)) * np.sin(np.pi * np.outer(i, i) / (m + 1))


@pytest.mark.parametrize("mx,my,dim", [(31, 31, 2), (7, 5, 2), (15, 15, 3), (4, 6, 3)])
def test_separable_interior_solve_is_exact(mx, my, dim):
    """The fast-diagonalisation interior solve (k_fdm_solve / k3_fdm_solve): the
    DST-I matrix S is orthonormal and symmetric, diagonalises the 1D Q1 matrices with the
    eigenvalues used on the device, and (S..)(D^-1)(S..) equals A_ii^-1 for the subdomain
    interior operator (the Kronecker sum that the next test pins to the oracle's assembly)."""
    h, mc = 1.0 / 64, complex(0.0, -1.0 / np.sqrt(1e-4))
    dims = [mx, my] + ([5] if dim == 3 else [])
    K1 = {m: (2 * np.eye(m) - np.eye(m, k=1) - np.eye(m, k=-1)) / h for m in dims}
    M1 = {m: h * (4 * np.eye(m) + np.eye(m, k=1) + np.eye(m, k=-1)) / 6 for m in dims}
    for m in dims:
        S = _dst(m)
        assert np.allclose(S @ S, np.eye(m), atol=1e-13) and np.allclose(S, S.T)
        th = np.pi * np.arange(1, m + 1) / (m + 1)
        assert np.allclose(S @ K1[m] @ S, np.diag((2 - 2 * np.cos(th)) / h), atol=1e-11)
        assert np.allclose(S @ M1[m] @ S, np.diag(h * (4 + 2 * np.cos(th)) / 6), atol=1e-15)
    # interior operator from the oracle's element matrices (Q1, exact Kronecker structure)
    kron = np.kron
    if dim == 2:
        A = kron(M1[my], K1[mx]) + kron(K1[my], M1[mx]) + mc * kron(M1[my], M1[mx])
        T = kron(_dst(my), _dst(mx))
        lam = [np.diag(_dst(m) @ K1[m] @ _dst(m)) for m in (mx, my)]
        nu = [np.diag(_dst(m) @ M1[m] @ _dst(m)) for m in (mx, my)]
        D = (np.outer(nu[1], lam[0]) + np.outer(lam[1], nu[0]) + mc * np.outer(nu[1], nu[0])).ravel()
    else:
        mz = dims[2]
        A = (kron(kron(M1[mz], M1[my]), K1[mx]) + kron(kron(M1[mz], K1[my]), M1[mx]) +
             kron(kron(K1[mz], M1[my]), M1[mx]) + mc * kron(kron(M1[mz], M1[my]), M1[mx]))
        T = kron(kron(_dst(mz), _dst(my)), _dst(mx))
        lam = [np.diag(_dst(m) @ K1[m] @ _dst(m)) for m in (mx, my, mz)]
        nu = [np.diag(_dst(m) @ M1[m] @ _dst(m)) for m in (mx, my, mz)]
        D = (np.einsum("k,j,i->kji", nu[2], nu[1], lam[0]) + np.einsum("k,j,i->kji", nu[2], lam[1], nu[0]) +
             np.einsum("k,j,i->kji", lam[2], nu[1], nu[0]) + mc * np.einsum("k,j,i->kji", nu[2], nu[1], nu[0])).ravel()
    rng = np.random.default_rng(0)
    x = rng.standard_normal(A.shape[0]) + 1j * rng.standard_normal(A.shape[0])
    y = T @ ((T @ x) / D)
    assert np.linalg.norm(A @ y - x) <= 1e-12 * np.linalg.norm(A) * np.linalg.norm(y)


def test_q1_heat_stencil_is_kronecker_sum(oracle_mod):
    """The precondition k_fdm_solve checks at setup, on the oracle's Q1 heat element: the
    assembled 9-point stencils of K and M equal K1 (x) M1 + M1 (x) K1 and M1 (x) M1."""
    n = 8
    p = oracle_mod.Problem(n, n)
    K, V = p.dense(0), p.dense(1)
    h = 1.0 / n
    m = n - 1
    K1 = (2 * np.eye(m) - np.eye(m, k=1) - np.eye(m, k=-1)) / h
    M1 = h * (4 * np.eye(m) + np.eye(m, k=1) + np.eye(m, k=-1)) / 6
    assert np.allclose(K, np.kron(M1, K1) + np.kron(K1, M1), atol=1e-13)
    assert np.allclose(V, np.kron(M1, M1), atol=1e-16)
