"""3D extension of the B200 range-space Schur solve (BASELINE.json configs 4-5).

The reference is 2D only.  This module exposes the same surface as the
2D package for trilinear Q1 hexahedra on a box, over the ``fetigpu3d_*`` C-ABI:

    make_box_problem(n, phi, physics, seed)    heat (whole-boundary Dirichlet) or linear
                                               elasticity (E, nu; clamped on x = 0)
    box_partition_info(problem, s)             sizes of the 3D partition (host C++)
    BoxSchurSolver(problem, s_x, s_y, s_z)     persistent context: factor once, solve many
    solve_range_space_3d(problem, s, ...)      one range-space Schur solve
    feti_solve_3d(problem, mass_coeff, rhs, s) one FETI-DP solve on K + mass_coeff V

Everything numeric runs in ``_lib/libfetigpu.so``; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import ContractError, _check, _dp, _out_arrays, _schur_result, _stats_dict
from . import _native
from ._native import Desc3, FetiStats, SchurStats

__all__ = ["BoxProblem", "make_box_problem", "box_partition_info", "BoxSchurSolver", "solve_range_space_3d",
           "feti_solve_3d", "emulated_schur_solve_3d", "rank_info_3d"]

INFO_KEYS = ("n", "m", "n_subdomains", "n_corner_dofs", "n_lambda", "NI", "NB", "NC", "MR", "block_halfwidth",
             "dofs_per_node", "ex", "ey", "ez", "maxe_bi", "maxe_ib")


@dataclass
class BoxProblem:
    n_x: int
    n_y: int
    n_z: int
    phi: float
    physics: int = 0
    young: float = 0.0
    poisson: float = 0.0
    len_x: float = 1.0
    len_y: float = 1.0
    len_z: float = 1.0
    target_state: np.ndarray = field(default=None, repr=False)
    boundary_values: np.ndarray = field(default=None, repr=False)

    def desc(self, s_x=1, s_y=1, s_z=1, tol=1e-10, max_iter=1000, mass_coeff=None, device=0):
        d = Desc3()
        d.n_x, d.n_y, d.n_z = self.n_x, self.n_y, self.n_z
        d.len_x, d.len_y, d.len_z = self.len_x, self.len_y, self.len_z
        d.physics, d.young, d.poisson = self.physics, self.young, self.poisson
        d.s_x, d.s_y, d.s_z = s_x, s_y, s_z
        if mass_coeff is None:
            d.phi = self.phi
        else:
            d.phi = 0.0
            d.mass_coeff_re, d.mass_coeff_im = complex(mass_coeff).real, complex(mass_coeff).imag
        d.tol, d.max_iter, d.device = tol, max_iter, device
        return d

    def info(self, s_x=0, s_y=0, s_z=0):
        out = np.zeros(16, dtype=np.int64)
        _check(_native.lib().fetigpu3d_problem_info(C.byref(self.desc(s_x, s_y, s_z)),
                                                    out.ctypes.data_as(C.POINTER(C.c_longlong))))
        return dict(zip(INFO_KEYS, (int(v) for v in out)))

    @property
    def n(self):
        return self.info()["n"]

    @property
    def m(self):
        return self.info()["m"]


def make_box_problem(n_x, n_y=None, n_z=None, phi=1e-6, physics=0, young=1.0, poisson=0.3, seed=0, modes=8, mmax=6):
    """Unit-cube control problem with the seeded sine-mode target (BASELINE configs 4-5:
    l, m, n ~ U{1..mmax}, a_k ~ N(0, 1); the same field for every displacement component)."""
    n_y = n_x if n_y is None else n_y
    n_z = n_x if n_z is None else n_z
    if physics == 0:
        young, poisson = 0.0, 0.0
    p = BoxProblem(n_x, n_y, n_z, phi, physics, young, poisson)
    n = p.n
    ybar = np.zeros(n)
    _check(_native.lib().fetigpu3d_target_sine(C.byref(p.desc()), seed, modes, mmax, _dp(ybar)))
    p.target_state = ybar
    return p


def box_partition_info(problem: BoxProblem, s_x, s_y=None, s_z=None):
    s_y = s_x if s_y is None else s_y
    s_z = s_x if s_z is None else s_z
    return problem.info(s_x, s_y, s_z)


class BoxSchurSolver:
    """Persistent 3D context (the two ComplexFactorSolver(FetiDp) of control.cpp:303-304,
    factored once through conjugate reuse)."""

    def __init__(self, problem: BoxProblem, s_x=2, s_y=None, s_z=None, tol=1e-10, max_iter=1000, mass_coeff=None,
                 device=0, rank=None, world=None, nccl_id=None):
        s_y = s_x if s_y is None else s_y
        s_z = s_x if s_z is None else s_z
        self.problem = problem
        self._desc = problem.desc(s_x, s_y, s_z, tol, max_iter, mass_coeff, device)
        h = C.c_void_p()
        if world is not None and world > 1:  # contiguous subdomain ranges sharded over NCCL
            if nccl_id is None or rank is None:
                raise ContractError("sharded BoxSchurSolver needs rank, world and the nccl_id of rank 0")
            _check(_native.lib().fetigpu3d_create_sharded(C.byref(self._desc), rank, world, bytes(nccl_id),
                                                          C.byref(h)))
        else:
            _check(_native.lib().fetigpu3d_create(C.byref(self._desc), C.byref(h)))
        self._h = h
        info = problem.info(s_x, s_y, s_z)
        self.info = info
        self.n, self.m, self.n_lambda, self.coarse_dim = info["n"], info["m"], info["n_lambda"], info["n_corner_dofs"]

    def close(self):
        if getattr(self, "_h", None):
            _native.lib().fetigpu3d_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve(self, ybar=None, yc=None, out=None):
        p = self.problem
        ybar = np.ascontiguousarray(p.target_state if ybar is None else ybar, dtype=np.float64)
        if ybar.shape != (self.n,):
            raise ContractError("ControlProblem: target length != n")
        ycp = None
        if yc is not None and self.m > 0:
            yc = np.ascontiguousarray(yc, dtype=np.float64)
            if yc.shape != (self.m,):
                raise ContractError("ControlProblem: boundary length != m")
            ycp = _dp(yc)
        y, u, lam = _out_arrays(out, self.n)
        st = SchurStats()
        _check(_native.lib().fetigpu3d_schur_solve(self._h, _dp(ybar), ycp, _dp(y), _dp(u), _dp(lam), C.byref(st)))
        return _schur_result(y, u, lam, st)

    def solve_device(self, d_ybar, d_yc, d_y, d_u, d_lambda):
        st = SchurStats()
        _check(_native.lib().fetigpu3d_schur_solve_device(self._h, d_ybar, d_yc, d_y, d_u, d_lambda, C.byref(st)))
        return _stats_dict(st)

    def feti_solve(self, rhs, sign=1):
        rhs = np.ascontiguousarray(rhs, dtype=np.complex128)
        if rhs.shape != (self.n,):
            raise ContractError("feti: rhs dimension mismatch")
        x = np.zeros(self.n, dtype=np.complex128)
        st = FetiStats()
        _check(_native.lib().fetigpu3d_feti_solve(self._h, sign, _dp(rhs.view(np.float64)), _dp(x.view(np.float64)),
                                                  C.byref(st)))
        return x, st.as_dict()

    def _lam_op(self, fn, v, sign):
        v = np.ascontiguousarray(v, dtype=np.complex128)
        if v.shape != (self.n_lambda,):
            raise ContractError("multiplier vector length != n_lambda")
        out = np.zeros(self.n_lambda, dtype=np.complex128)
        _check(fn(self._h, sign, _dp(v.view(np.float64)), _dp(out.view(np.float64))))
        return out

    def apply_dual_operator(self, lam, sign=1):
        return self._lam_op(_native.lib().fetigpu3d_apply_dual, lam, sign)

    def apply_dirichlet_preconditioner(self, r, sign=1):
        return self._lam_op(_native.lib().fetigpu3d_apply_precond, r, sign)

    @property
    def stream(self):
        return _native.lib().fetigpu3d_stream(self._h)

    def launch_count(self, reset=False):
        return int(_native.lib().fetigpu3d_launch_count(self._h, int(reset)))

    def profile(self, enable=True):
        _check(_native.lib().fetigpu3d_profile(self._h, int(enable)))

    def profile_read(self, reset=True):
        ms = np.zeros(len(_native.K_CLASSES))
        n = (C.c_longlong * len(_native.K_CLASSES))()
        _check(_native.lib().fetigpu3d_profile_read(self._h, _dp(ms), n, int(reset)))
        return {k: {"ms": float(ms[i]), "launches": int(n[i])} for i, k in enumerate(_native.K_CLASSES)}

    def class_bytes(self, klass):
        return float(_native.lib().fetigpu3d_class_bytes(self._h, _native.K_CLASSES.index(klass)))

    def setup_times(self):
        out = np.zeros(8)
        _native.lib().fetigpu3d_setup_times(self._h, _dp(out))
        keys = ("assembly", "aii_factor", "multi_rhs", "sbb_build", "sbb_inverse", "coupling_coarse", "pack", "total")
        return dict(zip(keys, (float(v) for v in out)))


def solve_range_space_3d(problem: BoxProblem, s_x=2, s_y=None, s_z=None, tol=1e-10, max_iter=1000):
    solver = BoxSchurSolver(problem, s_x, s_y, s_z, tol, max_iter)
    try:
        return solver.solve()
    finally:
        solver.close()


def feti_solve_3d(problem: BoxProblem, mass_coeff, rhs, s_x=2, s_y=None, s_z=None, tol=1e-10, max_iter=1000):
    solver = BoxSchurSolver(problem, s_x, s_y, s_z, tol, max_iter, mass_coeff=mass_coeff)
    try:
        return solver.feti_solve(rhs)
    finally:
        solver.close()


def emulated_schur_solve_3d(problem: BoxProblem, s_x, world, s_y=None, s_z=None, tol=1e-10, max_iter=1000):
    """`world` ranks of the sharded path emulated by host threads on one GPU (rank 0's result)."""
    s_y = s_x if s_y is None else s_y
    s_z = s_x if s_z is None else s_z
    d = problem.desc(s_x, s_y, s_z, tol, max_iter)
    n = problem.n
    ybar = np.ascontiguousarray(problem.target_state, dtype=np.float64)
    y, u, lam = np.zeros(n), np.zeros(n), np.zeros(n)
    st = SchurStats()
    _check(_native.lib().fetigpu3d_emulated_schur_solve(C.byref(d), world, _dp(ybar), None, _dp(y), _dp(u), _dp(lam),
                                                        C.byref(st)))
    return _schur_result(y, u, lam, st)


def rank_info_3d(problem: BoxProblem, s_x, rank, world, s_y=None, s_z=None):
    s_y = s_x if s_y is None else s_y
    s_z = s_x if s_z is None else s_z
    out = np.zeros(6, dtype=np.int64)
    _check(_native.lib().fetigpu3d_rank_info(C.byref(problem.desc(s_x, s_y, s_z)), rank, world,
                                             out.ctypes.data_as(C.POINTER(C.c_longlong))))
    keys = ("sub_first", "n_sub_local", "row_owners", "rows_both_local", "corner_slots", "n_lambda")
    return dict(zip(keys, (int(v) for v in out)))
