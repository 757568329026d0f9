"""ctypes wrapper of the CPU oracle (oracle/feti_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py — never by the product
package ``paper_1312_5653_b200``.  See feti_oracle.cpp for the reference
file:line map of every restated function.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


class OracleStats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("converged", C.c_int),
        ("relative_residual", C.c_double),
        ("primal_residual", C.c_double),
        ("interface_jump", C.c_double),
        ("setup_seconds", C.c_double),
        ("solve_seconds", C.c_double),
        ("n_lambda", C.c_int),
        ("coarse_dim", C.c_int),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ContractError(ValueError):
    pass


class NumericalError(RuntimeError):
    pass


def set_band_ldlt(on):
    """Subdomain blocks by symmetric band LDL^T (a third of the pivoted LU's memory; exact,
    agrees to rounding) -- for the full-size 3D digests (tests/golden/make_3d_digest.py)."""
    lib().orc_set_band_ldlt(int(bool(on)))


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.orc_last_error.restype = C.c_char_p
        L.orc_set_band_ldlt.argtypes = [C.c_int]
        L.orc_problem_create.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_double,
                                         C.c_double, C.POINTER(vp)]
        L.orc_problem_create3.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                          C.c_double, C.c_double, C.POINTER(vp)]
        L.orc_problem_destroy.argtypes = [vp]
        for f in ("orc_problem_n", "orc_problem_m"):
            getattr(L, f).argtypes = [vp]
        L.orc_problem_mass_sum.argtypes = [vp]
        L.orc_problem_mass_sum.restype = C.c_double
        L.orc_element_matrices.argtypes = [vp, dp, dp]
        L.orc_dense.argtypes = [vp, C.c_int, dp]
        L.orc_apply.argtypes = [vp, C.c_int, dp, dp]
        L.orc_target_thermal.argtypes = [vp, dp]
        L.orc_boundary_thermal.argtypes = [vp, dp]
        L.orc_target_sine.argtypes = [vp, C.c_ulonglong, C.c_int, C.c_int, dp]
        L.orc_sine_modes.argtypes = [C.c_ulonglong, C.c_int, C.c_int, dp, ip, ip]
        L.orc_partition_info.argtypes = [vp, C.c_int, C.c_int, ip]
        L.orc_partition_info3.argtypes = [vp, C.c_int, C.c_int, C.c_int, ip]
        L.orc_partition_sizes.argtypes = [vp, C.c_int, C.c_int, C.c_int, ip]
        L.orc_target_sine3.argtypes = [vp, C.c_ulonglong, C.c_int, C.c_int, dp]
        L.orc_feti_create3.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
        L.orc_schur_solve3.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, dp, dp, C.c_double, C.c_int,
                                       C.c_int, C.c_int, dp, dp, dp, C.POINTER(OracleStats),
                                       C.POINTER(OracleStats), dp, dp]
        L.orc_schur_create3.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                        C.c_int, C.POINTER(vp), dp]
        L.orc_schur_create4.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.POINTER(vp), dp]
        L.orc_feti_create.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
        L.orc_feti_destroy.argtypes = [vp]
        L.orc_feti_n_lambda.argtypes = [vp]
        L.orc_feti_coarse_dim.argtypes = [vp]
        L.orc_feti_setup_seconds.argtypes = [vp]
        L.orc_feti_setup_seconds.restype = C.c_double
        L.orc_feti_apply_dual.argtypes = [vp, dp, dp]
        L.orc_feti_apply_precond.argtypes = [vp, dp, dp]
        L.orc_feti_solve.argtypes = [vp, dp, dp, C.POINTER(OracleStats), dp, C.c_int]
        L.orc_schur_solve.argtypes = [vp, C.c_int, C.c_int, C.c_double, dp, dp, C.c_double, C.c_int, C.c_int,
                                      C.c_int, dp, dp, dp, C.POINTER(OracleStats), C.POINTER(OracleStats), dp, dp]
        L.orc_schur_create.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(vp), dp]
        L.orc_schur_destroy.argtypes = [vp]
        L.orc_schur_run.argtypes = [vp, dp, dp, dp, dp, dp, C.POINTER(OracleStats), C.POINTER(OracleStats), dp]
        L.orc_gmres_dense.argtypes = [C.c_int, dp, dp, C.c_double, C.c_int, dp, ip, dp, ip, dp, C.c_int]
        _lib = L
    return _lib


def _check(rc):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 1:
        raise ContractError(msg)
    raise NumericalError(msg)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


class Problem:
    """Mesh + Q1 assembly (mesh.cpp:7-36, fem.cpp:133-192). physics 0=heat, 1=plane strain
    (2D) / linear elasticity (3D).  n_z > 0: the 3D extension (trilinear hexahedra; BASELINE
    configs 4-5), whole-boundary Dirichlet for heat, clamped face x = 0 for elasticity."""

    def __init__(self, n_x, n_y=None, len_x=1.0, len_y=1.0, physics=0, young=0.0, poisson=0.0, n_z=0, len_z=1.0):
        n_y = n_x if n_y is None else n_y
        h = C.c_void_p()
        _check(lib().orc_problem_create3(n_x, n_y, n_z, len_x, len_y, len_z, physics, young, poisson, C.byref(h)))
        self._h = h
        self.n_x, self.n_y, self.n_z, self.physics = n_x, n_y, n_z, physics
        self.dim = 3 if n_z > 0 else 2
        self.n = lib().orc_problem_n(h)
        self.m = lib().orc_problem_m(h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_problem_destroy(self._h)
            self._h = None

    @property
    def mass_entry_sum(self):
        return lib().orc_problem_mass_sum(self._h)

    def element_matrices(self):
        npe = 8 if self.dim == 3 else 4
        ed = npe * (1 if self.physics == 0 else self.dim)
        ke = np.zeros((ed, ed))
        me = np.zeros((ed, ed))
        lib().orc_element_matrices(self._h, _dp(ke), _dp(me))
        return ke, me

    def dense(self, which):
        shape = (self.n, self.m) if which == 2 else (self.n, self.n)
        out = np.zeros(shape)
        lib().orc_dense(self._h, which, _dp(out))
        return out

    def apply(self, which, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.n)
        lib().orc_apply(self._h, which, _dp(x), _dp(y))
        return y

    def target_thermal(self):
        out = np.zeros(self.n)
        lib().orc_target_thermal(self._h, _dp(out))
        return out

    def boundary_thermal(self):
        out = np.zeros(self.m)
        lib().orc_boundary_thermal(self._h, _dp(out))
        return out

    def target_sine(self, seed, modes=8, mmax=8):
        out = np.zeros(self.n)
        if self.dim == 3:
            lib().orc_target_sine3(self._h, seed, modes, mmax, _dp(out))
        else:
            lib().orc_target_sine(self._h, seed, modes, mmax, _dp(out))
        return out

    def partition_info(self, s_x, s_y, s_z=1):
        info = np.zeros(7, dtype=np.int32)
        _check(lib().orc_partition_info3(self._h, s_x, s_y, s_z, _ip(info)))
        keys = ("n_subdomains", "n_corner_dofs", "n_lambda", "n_edges", "ex", "ey", "ez")
        d = dict(zip(keys, (int(v) for v in info)))
        if self.dim == 2:
            d.pop("ez")
        return d

    def partition_sizes(self, s_x, s_y, s_z=1):
        """Per subdomain (n_r, n_i, n_b, n_c, jump entries)."""
        ns = s_x * s_y * s_z
        out = np.zeros((ns, 5), dtype=np.int32)
        _check(lib().orc_partition_sizes(self._h, s_x, s_y, s_z, _ip(out)))
        return out

    def schur_solve(self, s_x, s_y, phi, ybar, yc=None, tol=1e-10, max_iter=2000, threads=1, augment=False, s_z=1):
        n = self.n
        ybar = np.ascontiguousarray(ybar, dtype=np.float64)
        ycp = None
        if yc is not None and self.m > 0:
            yc = np.ascontiguousarray(yc, dtype=np.float64)
            ycp = _dp(yc)
        y, u, lam = np.zeros(n), np.zeros(n), np.zeros(n)
        sp, sm = OracleStats(), OracleStats()
        leak = np.zeros(1)
        times = np.zeros(2)
        _check(lib().orc_schur_solve3(self._h, s_x, s_y, s_z, phi, _dp(ybar), ycp, tol, max_iter, threads, int(augment),
                                      _dp(y), _dp(u), _dp(lam), C.byref(sp), C.byref(sm), _dp(leak), _dp(times)))
        return {"y": y, "u": u, "lambda": lam, "imag_leak": float(leak[0]), "plus_stats": sp.as_dict(),
                "minus_stats": sm.as_dict(), "setup_seconds": float(times[0]), "solve_seconds": float(times[1]),
                "converged": bool(sp.converged and sm.converged)}


class Feti:
    """One FETI-DP(H) solver on A = k*K + c*V (feti.cpp:373-717); augment: edge-RBM
    augmentation of the coarse space (feti.cpp:171-242, 394-454, 572-578)."""

    def __init__(self, problem: Problem, s_x, s_y, mass_coeff, stiffness_coeff=1.0, tol=1e-10, max_iter=1000,
                 threads=1, augment=False, s_z=1):
        self.problem = problem
        mc, kc = complex(mass_coeff), complex(stiffness_coeff)
        h = C.c_void_p()
        _check(lib().orc_feti_create3(problem._h, s_x, s_y, s_z, kc.real, kc.imag, mc.real, mc.imag, tol, max_iter,
                                      threads, int(augment), C.byref(h)))
        self._h = h
        self.n_lambda = lib().orc_feti_n_lambda(h)
        self.coarse_dim = lib().orc_feti_coarse_dim(h)
        self.setup_seconds = lib().orc_feti_setup_seconds(h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_feti_destroy(self._h)
            self._h = None

    def _lam_op(self, fn, v):
        v = np.ascontiguousarray(v, dtype=np.complex128)
        out = np.zeros(self.n_lambda, dtype=np.complex128)
        _check(fn(self._h, _dp(v.view(np.float64)), _dp(out.view(np.float64))))
        return out

    def apply_dual_operator(self, lam):
        return self._lam_op(lib().orc_feti_apply_dual, lam)

    def apply_dirichlet_preconditioner(self, r):
        return self._lam_op(lib().orc_feti_apply_precond, r)

    def solve(self, rhs, history=False):
        rhs = np.ascontiguousarray(rhs, dtype=np.complex128)
        x = np.zeros(self.problem.n, dtype=np.complex128)
        st = OracleStats()
        cap = 4096
        hist = np.zeros(cap)
        _check(lib().orc_feti_solve(self._h, _dp(rhs.view(np.float64)), _dp(x.view(np.float64)), C.byref(st),
                                    _dp(hist), cap))
        d = st.as_dict()
        if history:
            d["history"] = hist[: d["iterations"]].copy()
        return x, d


class SchurPair:
    """Both reference factor solvers built once (control.cpp:303-304); run() = one Schur solve."""

    def __init__(self, problem: Problem, s_x, s_y, phi, tol=1e-10, max_iter=2000, threads=1, augment=False, s_z=1,
                 setup_threads=1):
        self.problem = problem
        h = C.c_void_p()
        t = np.zeros(1)
        _check(lib().orc_schur_create4(problem._h, s_x, s_y, s_z, phi, tol, max_iter, threads, int(augment),
                                       setup_threads, C.byref(h), _dp(t)))
        self._h = h
        self.setup_seconds = float(t[0])

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_schur_destroy(self._h)
            self._h = None

    def run(self, ybar, yc=None):
        n = self.problem.n
        ybar = np.ascontiguousarray(ybar, dtype=np.float64)
        ycp = None
        if yc is not None and self.problem.m > 0:
            yc = np.ascontiguousarray(yc, dtype=np.float64)
            ycp = _dp(yc)
        y, u, lam = np.zeros(n), np.zeros(n), np.zeros(n)
        sp, sm = OracleStats(), OracleStats()
        leak = np.zeros(1)
        _check(lib().orc_schur_run(self._h, _dp(ybar), ycp, _dp(y), _dp(u), _dp(lam), C.byref(sp), C.byref(sm),
                                   _dp(leak)))
        return {"y": y, "u": u, "lambda": lam, "imag_leak": float(leak[0]), "plus_stats": sp.as_dict(),
                "minus_stats": sm.as_dict(), "converged": bool(sp.converged and sm.converged)}


def sine_modes(seed, modes=8, mmax=8):
    a = np.zeros(modes)
    m = np.zeros(modes, dtype=np.int32)
    n = np.zeros(modes, dtype=np.int32)
    lib().orc_sine_modes(seed, modes, mmax, _dp(a), _ip(m), _ip(n))
    return a, m, n


def gmres_dense(a, b, tol=1e-10, max_iter=2000):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    b = np.ascontiguousarray(b, dtype=np.complex128)
    n = b.shape[0]
    x = np.zeros(n, dtype=np.complex128)
    it, conv = np.zeros(1, dtype=np.int32), np.zeros(1, dtype=np.int32)
    rr = np.zeros(1)
    hist = np.zeros(max(1, max_iter))
    _check(lib().orc_gmres_dense(n, _dp(a.view(np.float64)), _dp(b.view(np.float64)), tol, max_iter,
                                 _dp(x.view(np.float64)), _ip(it), _dp(rr), _ip(conv), _dp(hist), hist.size))
    return x, {"iterations": int(it[0]), "relative_residual": float(rr[0]), "converged": bool(conv[0]),
               "history": hist[: int(it[0])].copy()}
