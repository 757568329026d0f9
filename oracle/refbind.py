"""ctypes wrapper of oracle/_ref/libpdeopt_ref.so: the UNMODIFIED reference sources
(/root/reference/proj/src) compiled against the Eigen-API shim (oracle/ref_shim), behind the
thin extern "C" driver oracle/ref_driver.cpp.

TEST INFRASTRUCTURE ONLY: imported by tests/, tests/golden/ generators and bench.py's
reference arm — never by the product package.  The library is built here (where
/root/reference exists) by ``make -C oracle ref``; on the GPU box only the prebuilt
``oracle/_ref`` files exist (``available()`` tells which).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_ref", "libpdeopt_ref.so")
REF_SRC = "/root/reference/proj"
_lib = None

HEAT, CANTILEVER = 0, 1


class ContractError(ValueError):
    pass


class NumericalError(RuntimeError):
    pass


def build():
    """Compiles oracle/_ref from the reference sources (only where they exist)."""
    if not os.path.isdir(REF_SRC):
        raise FileNotFoundError("reference sources absent; oracle/_ref must be prebuilt")
    subprocess.check_call(["make", "-s", "-j8", "-C", _HERE, "ref"])


def available():
    return os.path.exists(_LIB_PATH) or os.path.isdir(REF_SRC)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.ref_last_error.restype = C.c_char_p
        L.ref_problem_size.argtypes = [C.c_int, C.c_int, ip, ip]
        L.ref_problem_data.argtypes = [C.c_int, C.c_int, dp, dp]
        L.ref_schur_solve.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, dp, dp, C.c_double, C.c_int,
                                      C.c_int, C.c_int, dp, dp, dp, dp]
        L.ref_pair_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                      C.c_int, C.POINTER(vp), dp]
        L.ref_pair_destroy.argtypes = [vp]
        L.ref_pair_solve.argtypes = [vp, dp, dp, dp]
        L.ref_feti_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
        L.ref_feti_destroy.argtypes = [vp]
        L.ref_feti_sizes.argtypes = [vp, ip]
        L.ref_feti_solve.argtypes = [vp, dp, dp, dp]
        L.ref_feti_apply.argtypes = [vp, C.c_int, dp, dp]
        _lib = L
    return _lib


def _check(rc):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    if rc == 1:
        raise ContractError(msg)
    if rc == 2:
        raise NumericalError(msg)
    raise RuntimeError(msg)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def problem_size(kind, n):
    nf, m = C.c_int(), C.c_int()
    _check(lib().ref_problem_size(kind, n, C.byref(nf), C.byref(m)))
    return nf.value, m.value


def problem_data(kind, n):
    """The reference's own target state and Dirichlet values (control.cpp:24-46)."""
    nf, m = problem_size(kind, n)
    ybar, yc = np.zeros(nf), np.zeros(m)
    _check(lib().ref_problem_data(kind, n, _dp(ybar), _dp(yc)))
    return ybar, yc


def schur_solve(n, s_x, s_y, phi, ybar=None, yc=None, tol=1e-10, max_iter=2000, augment=False, threads=1,
                kind=HEAT):
    """pdeopt::solve_range_space(make_*_problem(n, phi) [target := ybar, y_c := yc or 0],
    {FetiDp, tol, max_iter, feti={s_x, s_y, augment, threads}})."""
    nf, m = problem_size(kind, n)
    ybar_a = None if ybar is None else np.ascontiguousarray(ybar, dtype=np.float64)
    yc_a = None if yc is None else np.ascontiguousarray(yc, dtype=np.float64)
    if ybar_a is not None and ybar_a.size != nf:
        raise ContractError("ybar length != n")
    if yc_a is not None and yc_a.size != m:
        raise ContractError("yc length != m")
    y, u, lam, st = np.zeros(nf), np.zeros(nf), np.zeros(nf), np.zeros(10)
    _check(lib().ref_schur_solve(kind, n, s_x, s_y, phi, _dp(ybar_a), _dp(yc_a), tol, max_iter, int(augment),
                                 threads, _dp(y), _dp(u), _dp(lam), _dp(st)))
    return {
        "y": y, "u": u, "lambda": lam,
        "plus_stats": {"iterations": int(st[0]), "converged": bool(st[2]), "relative_residual": st[4]},
        "minus_stats": {"iterations": int(st[1]), "converged": bool(st[3]), "relative_residual": st[5]},
        "imag_leak": st[6], "factor_setup_seconds": st[7], "seconds": st[8], "imag_leak_warning": bool(st[9]),
    }


class FactorPair:
    """solve_range_space's two ComplexFactorSolver(FetiDp) (control.cpp:302-304), set up once;
    solve() runs the dual part (control.cpp:306-320) with the factors reused and returns
    lambda plus the reference's per_solve_seconds (experiments.cpp:265)."""

    def __init__(self, n, s_x, s_y, phi, tol=1e-10, max_iter=2000, augment=False, threads=1, kind=HEAT):
        h, setup = C.c_void_p(), C.c_double()
        _check(lib().ref_pair_create(kind, n, s_x, s_y, phi, tol, max_iter, int(augment), threads, C.byref(h),
                                     C.byref(setup)))
        self._h, self.setup_seconds = h, setup.value
        self.n = problem_size(kind, n)[0]

    def close(self):
        if getattr(self, "_h", None):
            lib().ref_pair_destroy(self._h)
            self._h = None

    __del__ = close

    def solve(self, ybar):
        yb = np.ascontiguousarray(ybar, dtype=np.float64)
        if yb.size != self.n:
            raise ContractError("ybar length != n")
        lam, st = np.zeros(self.n), np.zeros(5)
        _check(lib().ref_pair_solve(self._h, _dp(yb), _dp(lam), _dp(st)))
        return lam, {"iterations": (int(st[0]), int(st[1])), "converged": bool(st[2]), "per_solve_seconds": st[3],
                     "seconds": st[4]}


class Feti:
    """pdeopt::FetiSolver<Complex> on A = stiffness_coeff K + mass_coeff V of make_*_problem(n)."""

    def __init__(self, n, s_x, s_y, mass_coeff, stiffness_coeff=1.0, tol=1e-10, max_iter=1000, augment=False,
                 threads=1, kind=HEAT):
        h = C.c_void_p()
        mc = complex(mass_coeff)
        _check(lib().ref_feti_create(kind, n, s_x, s_y, stiffness_coeff, mc.real, mc.imag, tol, max_iter,
                                     int(augment), threads, C.byref(h)))
        self._h = h
        sz = (C.c_int * 4)()
        _check(lib().ref_feti_sizes(h, sz))
        self.n_free, self.n_lambda, self.coarse_dim, self.n_subdomains = list(sz)

    def close(self):
        if getattr(self, "_h", None):
            lib().ref_feti_destroy(self._h)
            self._h = None

    __del__ = close

    def solve(self, rhs):
        b = np.ascontiguousarray(rhs, dtype=np.complex128)
        if b.size != self.n_free:
            raise ContractError("rhs length != n_free")
        x, st = np.zeros(self.n_free, np.complex128), np.zeros(6)
        _check(lib().ref_feti_solve(self._h, _dp(b.view(np.float64)), _dp(x.view(np.float64)), _dp(st)))
        return x, {"iterations": int(st[0]), "relative_residual": st[1], "converged": bool(st[2]),
                   "primal_residual": st[3], "interface_jump": st[4], "solve_seconds": st[5]}

    def _apply(self, which, v):
        a = np.ascontiguousarray(v, dtype=np.complex128)
        if a.size != self.n_lambda:
            raise ContractError("vector length != n_lambda")
        out = np.zeros(self.n_lambda, np.complex128)
        _check(lib().ref_feti_apply(self._h, which, _dp(a.view(np.float64)), _dp(out.view(np.float64))))
        return out

    def apply_dual_operator(self, lam):
        return self._apply(0, lam)

    def apply_dirichlet_preconditioner(self, r):
        return self._apply(1, r)

    def project_out_augmentation(self, v):
        return self._apply(2, v)
