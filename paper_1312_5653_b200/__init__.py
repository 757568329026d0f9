"""B200-native range-space Schur solve (arXiv 1312.5653): two complex-symmetric
FETI-DP(H) solves on K -/+ i phi^-1/2 M behind the reference's python surface.

Mirrors the ``pdeopt`` python package of the reference (python/bindings.cpp):

    make_thermal_problem(n, phi)                          bindings.cpp:87-88
    solve_range_space(problem, method, tol, s_x, s_y, augment)   bindings.cpp:93-111
    feti_solve(problem, mass_coeff, rhs, s_x, s_y, augment, tol) bindings.cpp:158-185
    solve_full_space(problem, precond, outer, tol, inner_method, inner_tol, s_x, s_y)
                                                          bindings.cpp:113-145
    diagnostics(problem, y, u, lambda)                    bindings.cpp:147-156
    ContractError -> ValueError, NumericalError -> RuntimeError (bindings.cpp:60-61)

plus ``make_seeded_problem`` (the BASELINE.json sine-mode target) and ``SchurSolver``,
a persistent context that factors once and solves many right-hand sides (the
reference's per_solve_seconds regime, experiments.cpp:265).

Everything numeric runs in ``_lib/libfetigpu.so`` (C++ host core + sm_100a CUDA);
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import Desc, FetiStats, SchurStats

__all__ = [
    "ContractError", "NumericalError", "ControlProblem", "make_thermal_problem", "make_seeded_problem",
    "make_problem", "make_cantilever_problem", "partition_info", "SchurSolver", "solve_range_space", "feti_solve",
    "solve_full_space",
    "diagnostics", "nccl_unique_id", "rank_info", "emulated_schur_solve",
]


class ContractError(ValueError):
    """Contract violation (reference ContractError, csr.hpp:26-29)."""


class NumericalError(RuntimeError):
    """Numerical failure (reference NumericalError, csr.hpp:33-36)."""


def _check(rc):
    if rc == 0:
        return
    msg = _native.lib().fetigpu_last_error().decode()
    if rc == 1:
        raise ContractError(msg)
    if rc == 2:
        raise NumericalError(msg)
    raise RuntimeError(msg)


def _out_arrays(out, n):
    """Caller-supplied (y, u, lambda) output arrays, checked before their raw pointers reach the
    C-ABI (which writes n float64 into each)."""
    if out is None:
        return np.zeros(n), np.zeros(n), np.zeros(n)
    if len(out) != 3:
        raise ContractError("solve: out must be (y, u, lambda)")
    for a in out:
        if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.shape != (n,) or not a.flags.c_contiguous \
                or not a.flags.writeable:
            raise ContractError("solve: out arrays must be writeable contiguous float64 of length n")
    return tuple(out)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass
class ControlProblem:
    """Discrete distributed control problem (control.hpp:15-31) on a structured mesh.

    Stores the mesh/physics description and the data vectors; K, V and Kc are never
    materialised on the host — the device applies them element by element.
    """

    n_x: int
    n_y: int
    phi: float
    physics: int = 0
    len_x: float = 1.0
    len_y: float = 1.0
    young: float = 0.0
    poisson: float = 0.0
    target_state: np.ndarray = field(default=None, repr=False)
    boundary_values: np.ndarray = field(default=None, repr=False)

    def desc(self, s_x=2, s_y=2, tol=1e-10, max_iter=1000, mass_coeff=None, device=0, augment=False):
        d = Desc()
        d.n_x, d.n_y, d.len_x, d.len_y = self.n_x, self.n_y, self.len_x, self.len_y
        d.physics, d.young, d.poisson = self.physics, self.young, self.poisson
        d.s_x, d.s_y = s_x, s_y
        if mass_coeff is None:
            d.phi = self.phi
        else:
            d.phi = 0.0
            d.mass_coeff_re, d.mass_coeff_im = complex(mass_coeff).real, complex(mass_coeff).imag
        d.tol, d.max_iter, d.augment, d.device = tol, max_iter, int(bool(augment)), device
        return d

    def _info(self, s_x=2, s_y=2):
        info = np.zeros(10, dtype=np.int32)
        _check(_native.lib().fetigpu_problem_info(C.byref(self.desc(s_x, s_y)),
                                                  info.ctypes.data_as(C.POINTER(C.c_int))))
        return info

    @property
    def n(self):
        return int(self._info(0, 0)[0])

    @property
    def m(self):
        return int(self._info(0, 0)[1])

    def validate(self):  # control.cpp:7-13
        if not (self.phi > 0.0):
            raise ContractError("ControlProblem: phi must be positive")
        if self.target_state is None or len(self.target_state) != self.n:
            raise ContractError("ControlProblem: target length != n")
        if self.boundary_values is not None and len(self.boundary_values) != self.m:
            raise ContractError("ControlProblem: boundary length != m")


def _base_desc(n_x, n_y, physics=0, len_x=1.0, len_y=1.0, young=0.0, poisson=0.0):
    d = Desc()
    d.n_x, d.n_y, d.len_x, d.len_y = n_x, n_y, len_x, len_y
    d.physics, d.young, d.poisson = physics, young, poisson
    d.s_x = d.s_y = 1
    d.tol, d.max_iter = 1e-10, 1
    return d


def make_problem(n_x, n_y=None, phi=1e-4, physics=0, len_x=1.0, len_y=1.0, young=0.0, poisson=0.0,
                 target="thermal", seed=0, modes=8, mmax=8):
    """Build a ControlProblem.  target: "thermal" (fem.cpp:194-220, y_c = target trace)
    or "sine" (BASELINE.json seeded sine modes, y_c = 0)."""
    n_y = n_x if n_y is None else n_y
    if n_x < 2 or n_y < 2:
        raise ContractError("build_rectangle_mesh: need at least 2 elements per axis")
    p = ControlProblem(n_x=n_x, n_y=n_y, phi=phi, physics=physics, len_x=len_x, len_y=len_y, young=young,
                       poisson=poisson)
    info = p._info(0, 0)
    n, m = int(info[0]), int(info[1])
    d = _base_desc(n_x, n_y, physics, len_x, len_y, young, poisson)
    ybar = np.zeros(n)
    if target == "thermal":
        yc = np.zeros(m)
        _check(_native.lib().fetigpu_target_thermal(C.byref(d), _dp(ybar), _dp(yc) if m else None))
    elif target == "sine":
        yc = None  # homogeneous Dirichlet data, y_c = 0 (BASELINE.json configs)
        _check(_native.lib().fetigpu_target_sine(C.byref(d), seed, modes, mmax, _dp(ybar)))
    else:
        raise ContractError("target must be 'thermal' or 'sine'")
    p.target_state, p.boundary_values = ybar, yc
    return p


def make_thermal_problem(n, phi):
    """Unit-square heat control problem with the piecewise target (control.cpp:24-34)."""
    if not (phi > 0.0):
        raise ContractError("ControlProblem: phi must be positive")
    return make_problem(n, n, phi, target="thermal")


def make_seeded_problem(n, phi, seed=0, modes=8, mmax=8):
    """BASELINE.json configs 1-3: unit square, seeded sine-mode target, y_c = 0."""
    if not (phi > 0.0):
        raise ContractError("ControlProblem: phi must be positive")
    return make_problem(n, n, phi, target="sine", seed=seed, modes=modes, mmax=mmax)


def partition_info(problem: ControlProblem, s_x, s_y):
    """Sizes of partition_structured (feti.cpp:34-169) computed by the C++ host core."""
    info = problem._info(s_x, s_y)
    keys = ("n", "m", "n_subdomains", "n_corner_dofs", "n_lambda", "n_edges", "ex", "ey", "dofs_per_node",
            "band_halfwidth")
    return dict(zip(keys, (int(v) for v in info)))


class SchurSolver:
    """Persistent GPU context: partition + factor once (K + cV only), solve many.

    Replaces the pair of ComplexFactorSolver(FetiDp) of solve_range_space
    (control.cpp:303-304).  ``mass_coeff`` (instead of phi) binds the context to a
    single factor K + mass_coeff*V for feti_solve parity runs.
    """

    def __init__(self, problem: ControlProblem, s_x=2, s_y=2, tol=1e-10, max_iter=1000, mass_coeff=None,
                 device=0, augment=False, rank=None, world=None, nccl_id=None):
        self.problem = problem
        self._desc = problem.desc(s_x, s_y, tol, max_iter, mass_coeff, device, augment)
        h = C.c_void_p()
        if world is not None and world > 1:
            # sharded over NCCL: this process is `rank` (subdomain rows rank*s_y/world ...)
            if nccl_id is None or rank is None:
                raise ContractError("sharded SchurSolver needs rank, world and the nccl_id of rank 0")
            _check(_native.lib().fetigpu_create_sharded(C.byref(self._desc), rank, world, bytes(nccl_id),
                                                        C.byref(h)))
        else:
            _check(_native.lib().fetigpu_create(C.byref(self._desc), C.byref(h)))
        self._h = h
        if world is not None and world > 1:
            info = problem._info(s_x, s_y)
        else:  # the context's own partition (no second host partition build)
            info = (C.c_int * 10)()
            _check(_native.lib().fetigpu_context_info(h, info))
        self.n, self.m, self.n_lambda, self.coarse_dim = int(info[0]), int(info[1]), int(info[4]), int(info[3])
        self.augment = bool(augment)
        if augment:  # coarse = corners + edge-RBM columns (1 per edge, 3 for plane strain)
            self.coarse_dim += int(info[5]) * (1 if int(info[8]) == 1 else 3)

    def close(self):
        if getattr(self, "_h", None):
            _native.lib().fetigpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- range space ---------------------------------------------------------------
    def solve(self, ybar=None, yc=None, out=None):
        """Range-space Schur solve with host buffers (control.cpp:297-334).  ``out`` may
        supply preallocated (e.g. pinned) float64 arrays (y, u, lambda)."""
        p = self.problem
        ybar = np.ascontiguousarray(p.target_state if ybar is None else ybar, dtype=np.float64)
        if yc is None:
            yc = p.boundary_values
        ycp = None
        if yc is not None and self.m > 0:
            yc = np.ascontiguousarray(yc, dtype=np.float64)
            if yc.shape != (self.m,):
                raise ContractError("ControlProblem: boundary length != m")
            ycp = _dp(yc)
        if ybar.shape != (self.n,):
            raise ContractError("ControlProblem: target length != n")
        y, u, lam = _out_arrays(out, self.n)
        st = SchurStats()
        _check(_native.lib().fetigpu_schur_solve(self._h, _dp(ybar), ycp, _dp(y), _dp(u), _dp(lam), C.byref(st)))
        return _schur_result(y, u, lam, st)

    def solve_device(self, d_ybar, d_yc, d_y, d_u, d_lambda):
        """Range-space Schur solve on device pointers (ints); returns the stats dict."""
        st = SchurStats()
        _check(_native.lib().fetigpu_schur_solve_device(self._h, d_ybar, d_yc, d_y, d_u, d_lambda, C.byref(st)))
        return _stats_dict(st)

    # -- single factor -------------------------------------------------------------
    def feti_solve(self, rhs, sign=1):
        rhs = np.ascontiguousarray(rhs, dtype=np.complex128)
        if rhs.shape != (self.n,):
            raise ContractError("feti: rhs dimension mismatch")  # feti.cpp:639
        x = np.zeros(self.n, dtype=np.complex128)
        st = FetiStats()
        _check(_native.lib().fetigpu_feti_solve(self._h, sign, _dp(rhs.view(np.float64)), _dp(x.view(np.float64)),
                                                C.byref(st)))
        return x, st.as_dict()

    def apply_dual_operator(self, lam, sign=1):
        return self._lam_op(_native.lib().fetigpu_apply_dual, lam, sign)

    def apply_dirichlet_preconditioner(self, r, sign=1):
        return self._lam_op(_native.lib().fetigpu_apply_precond, r, sign)

    def _lam_op(self, fn, v, sign):
        v = np.ascontiguousarray(v, dtype=np.complex128)
        if v.shape != (self.n_lambda,):
            raise ContractError("multiplier vector length != n_lambda")
        out = np.zeros(self.n_lambda, dtype=np.complex128)
        _check(fn(self._h, sign, _dp(v.view(np.float64)), _dp(out.view(np.float64))))
        return out

    # -- instrumentation -----------------------------------------------------------
    @property
    def stream(self):
        return _native.lib().fetigpu_stream(self._h)

    def launch_count(self, reset=False):
        return int(_native.lib().fetigpu_launch_count(self._h, int(reset)))

    def profile(self, enable=True):
        _check(_native.lib().fetigpu_profile(self._h, int(enable)))

    def profile_read(self, reset=True):
        ms = np.zeros(len(_native.K_CLASSES))
        n = (C.c_longlong * len(_native.K_CLASSES))()
        _check(_native.lib().fetigpu_profile_read(self._h, _dp(ms), n, int(reset)))
        return {k: {"ms": float(ms[i]), "launches": int(n[i])} for i, k in enumerate(_native.K_CLASSES)}

    def gemv_timing(self, reps=20):
        """Per-launch ms of the Arnoldi GEMVs, CUDA events inside a captured graph of
        back-to-back (precond, dual) pairs: {precond_gemv: ms, dual_gemv: ms}."""
        out = np.zeros(4)
        _check(_native.lib().fetigpu_gemv_timing(self._h, reps, _dp(out)))
        return {"precond_gemv": float(out[0]), "dual_gemv": float(out[1])}

    def step_spans(self):
        """Mean in-graph kernel spans (us) of the last FETI solve's Arnoldi steps:
        dict(precond, gap_pd, dual, gap_dt, tail, gap_tp, steps) or None."""
        out = np.zeros(6)
        k = _native.lib().fetigpu_step_spans(self._h, _dp(out))
        if k <= 0:
            return None
        keys = ("precond", "gap_pd", "dual", "gap_dt", "tail", "gap_tp")
        d = dict(zip(keys, (float(v) for v in out)))
        d["steps"] = int(k)
        return d

    def class_bytes(self, klass):
        return float(_native.lib().fetigpu_class_bytes(self._h, _native.K_CLASSES.index(klass)))


def nccl_unique_id():
    """128-byte NCCL unique id for SchurSolver(..., rank, world, nccl_id) (create on rank 0)."""
    buf = C.create_string_buffer(128)
    _check(_native.lib().fetigpu_nccl_unique_id(buf))
    return buf.raw


def rank_info(problem: ControlProblem, s_x, s_y, rank, world):
    """Host-side layout of one rank of the sharded path (no GPU needed)."""
    info = np.zeros(12, dtype=np.int32)
    _check(_native.lib().fetigpu_rank_info(C.byref(problem.desc(s_x, s_y)), rank, world,
                                           info.ctypes.data_as(C.POINTER(C.c_int))))
    keys = ("sub_first", "n_sub_local", "n_phantom", "lam_base", "n_ghost", "n_owned", "n_top_cut", "free_first",
            "free_count", "halo_up", "halo_down", "n_lambda_local")
    return dict(zip(keys, (int(v) for v in info)))


def emulated_schur_solve(problem: ControlProblem, world, s_x=2, s_y=2, tol=1e-10, max_iter=1000, device=0):
    """The sharded solve with `world` ranks emulated by host threads on ONE GPU (test path)."""
    problem.validate()
    d = problem.desc(s_x, s_y, tol, max_iter, None, device)
    n = problem.n
    ybar = np.ascontiguousarray(problem.target_state, dtype=np.float64)
    yc = problem.boundary_values
    ycp = _dp(np.ascontiguousarray(yc, dtype=np.float64)) if yc is not None and problem.m > 0 else None
    y, u, lam = np.zeros(n), np.zeros(n), np.zeros(n)
    st = SchurStats()
    _check(_native.lib().fetigpu_emulated_schur_solve(C.byref(d), world, _dp(ybar), ycp, _dp(y), _dp(u), _dp(lam),
                                                      C.byref(st)))
    return _schur_result(y, u, lam, st)


def _stats_dict(st: SchurStats):
    return {"plus_stats": _solve_stats(st.plus), "minus_stats": _solve_stats(st.minus),
            "imag_leak": st.imag_leak, "imag_leak_warning": bool(st.imag_leak_warning),
            "converged": bool(st.converged), "factor_setup_seconds": st.factor_setup_seconds,
            "solve_seconds": st.solve_seconds}


def _solve_stats(s: FetiStats):  # SolveStats dict of bindings.cpp:35-42 (+ FETI extras)
    return {"iterations": s.iterations, "relative_residual": s.relative_residual, "converged": bool(s.converged),
            "wall_time": s.solve_seconds, "primal_residual": s.primal_residual, "interface_jump": s.interface_jump}


def _schur_result(y, u, lam, st):
    d = {"y": y, "u": u, "lambda": lam}
    d.update(_stats_dict(st))
    return d


def solve_range_space(problem: ControlProblem, method="feti", tol=1e-12, s_x=2, s_y=2, augment=True,
                      max_iter=1000):
    """Dual solve through the two complex-conjugate factors, then primal recovery
    (bindings.cpp:93-111).  Only the FETI-DP method runs on the B200 path."""
    if method != "feti":
        raise ContractError("factor method must be feti on the B200 path (direct/gmres are CPU reference methods)")
    problem.validate()
    solver = SchurSolver(problem, s_x, s_y, tol, max_iter, augment=augment)
    try:
        return solver.solve()
    finally:
        solver.close()


def feti_solve(problem: ControlProblem, mass_coeff, rhs, s_x=2, s_y=2, augment=True, tol=1e-10, max_iter=1000):
    """FETI-DP solve of (K + mass_coeff V) x = rhs (bindings.cpp:158-185)."""
    solver = SchurSolver(problem, s_x, s_y, tol, max_iter, mass_coeff=mass_coeff, augment=augment)
    try:
        x, st = solver.feti_solve(rhs)
    finally:
        solver.close()
    return {"x": x, "iterations": st["iterations"], "converged": st["converged"],
            "interface_jump": st["interface_jump"], "primal_residual": st["primal_residual"],
            "n_lambda": st["n_lambda"], "coarse_dim": st["coarse_dim"]}


def solve_full_space(problem: ControlProblem, precond="none", outer="minres", tol=1e-10, inner_method="feti",
                     inner_tol=1e-12, s_x=2, s_y=2, augment=True, max_iter=5000):
    """Simultaneous KKT solve, optionally with the block-diagonal Murphy-Golub-Wathen
    preconditioner (bindings.cpp:113-145, control.cpp:418-476).  precond: "none", "sp"
    (Pearson-Wathen approximate Schur complement) or "sc" (exact Schur through the complex
    FETI factors, GMRES only); outer: "minres" or "gmres".  The inner factor solves run on
    the B200 FETI-DP path (inner_method "feti"; the reference's "direct"/"gmres" inner
    backends are CPU-only and not provided)."""
    pc = {"none": 0, "sp": 1, "sc": 2}.get(precond)
    if pc is None:
        raise ContractError("precond must be none, sp or sc")
    oc = {"minres": 0, "gmres": 1}.get(outer)
    if oc is None:
        raise ContractError("outer must be minres or gmres")
    if inner_method != "feti":
        raise ContractError("solve_full_space: the B200 path's inner factor solves are FETI-DP (inner_method='feti')")
    problem.validate()
    solver = SchurSolver(problem, s_x, s_y, inner_tol, 2000, augment=augment)
    n = problem.n
    ybar = np.ascontiguousarray(problem.target_state, dtype=np.float64)
    yc = problem.boundary_values
    ycp = _dp(np.ascontiguousarray(yc, dtype=np.float64)) if yc is not None and problem.m > 0 else None
    y, u, lam = np.zeros(n), np.zeros(n), np.zeros(n)
    st = FetiStats()
    leak = np.zeros(1)
    try:
        _check(_native.lib().fetigpu_full_space(solver._h, pc, oc, tol, max_iter, _dp(ybar), ycp, _dp(y), _dp(u),
                                                _dp(lam), C.byref(st), _dp(leak)))
    finally:
        solver.close()
    stats = {"iterations": st.iterations, "relative_residual": st.relative_residual, "converged": bool(st.converged),
             "wall_time": st.solve_seconds}
    return {"y": y, "u": u, "lambda": lam, "stats": stats, "imag_leak": float(leak[0]),
            "inner_iterations": st.coarse_dim, "precond_setup_seconds": st.setup_seconds}


def make_cantilever_problem(n, phi, pressure=100e3, tol=1e-13):
    """Plane-strain 3:1 rubber cantilever clamped at x = 0 (control.cpp:36-46): 3n x n Q1
    mesh on [0,3]x[0,1], E = 20.7e6, nu = 0.45; the target is the displacement under a
    bottom-edge pressure, K ybar = f (fem.cpp:222-260), solved here by the GPU FETI-DP path
    with mass coefficient 0 (the reference uses a refined sparse Cholesky)."""
    if not (phi > 0.0):
        raise ContractError("ControlProblem: phi must be positive")
    p = make_problem(3 * n, n, phi, physics=1, len_x=3.0, len_y=1.0, young=20.7e6, poisson=0.45)
    f = np.zeros(p.n)
    _check(_native.lib().fetigpu_pressure_load(C.byref(_base_desc(3 * n, n, 1, 3.0, 1.0, 20.7e6, 0.45)),
                                               float(pressure), _dp(f)))
    p.boundary_values = np.zeros(p.m)  # clamped edge
    if np.linalg.norm(f) == 0.0:
        p.target_state = np.zeros(p.n)
        return p
    q = next(d for d in range(1, n + 1) if n % d == 0 and n // d <= 24)  # square subdomains <= 24 h
    out = feti_solve(p, 0.0, f.astype(complex), s_x=3 * q, s_y=q, augment=False, tol=tol, max_iter=2000)
    p.target_state = np.ascontiguousarray(out["x"].real)
    return p


def diagnostics(problem: ControlProblem, y, u, lam, K=None, V=None, Kc=None):
    """Optimality diagnostics (control.cpp:122-141; bindings.cpp:147-156).  Without operator
    arguments K, V, Kc are applied on the device (fetigpu_diagnostics); scipy/numpy
    operators may be passed instead (host evaluation, for tests)."""
    if K is None or V is None:
        yv = np.ascontiguousarray(y, dtype=np.float64)
        uv = np.ascontiguousarray(u, dtype=np.float64)
        yb = np.ascontiguousarray(problem.target_state, dtype=np.float64)
        yc = problem.boundary_values
        ycp = _dp(np.ascontiguousarray(yc, dtype=np.float64)) if yc is not None and problem.m > 0 else None
        out = np.zeros(5)
        _check(_native.lib().fetigpu_diagnostics(C.byref(problem.desc()), _dp(yv), _dp(uv), _dp(yb), ycp,
                                                 _dp(out)))
        return {"violation_defined": bool(out[4]), "constraint_violation": float(out[0]),
                "target_mismatch": float(out[1]), "control_norm": float(out[2]), "objective": float(out[3])}
    yc = problem.boundary_values
    ky = K @ y
    res = ky - V @ u
    if Kc is not None and yc is not None and len(yc):
        res = res + Kc @ yc
    kyn = np.linalg.norm(ky)
    rep = {"violation_defined": kyn != 0.0, "constraint_violation": (np.linalg.norm(res) / kyn) if kyn else 0.0}
    dy = y - problem.target_state
    dyv = math.sqrt(dy @ (V @ dy))
    ybv = math.sqrt(problem.target_state @ (V @ problem.target_state))
    rep["target_mismatch"] = dyv / ybv if ybv > 0 else dyv
    rep["control_norm"] = math.sqrt(u @ (V @ u))
    rep["objective"] = 0.5 * dyv * dyv + 0.5 * problem.phi * rep["control_norm"] ** 2
    return rep
