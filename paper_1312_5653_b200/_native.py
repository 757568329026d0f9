"""ctypes binding of the in-tree C-ABI library ``_lib/libfetigpu.so`` (include/fetigpu.h).

There is no fallback: if the library is missing or fails to load, importing the
solver API raises.  The library is built by ``paper_1312_5653_b200.build`` (or
``__graft_entry__.build()``) with nvcc for sm_100a.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FETIGPU_LIB") or os.path.join(_HERE, "_lib", "libfetigpu.so")  # (experiment builds)

K_CLASSES = ("precond_gemv", "dual_gemv", "coarse", "lambda", "ortho", "band", "global", "other")


class Desc(C.Structure):
    _fields_ = [
        ("n_x", C.c_int), ("n_y", C.c_int), ("len_x", C.c_double), ("len_y", C.c_double),
        ("physics", C.c_int), ("young", C.c_double), ("poisson", C.c_double),
        ("s_x", C.c_int), ("s_y", C.c_int), ("phi", C.c_double),
        ("mass_coeff_re", C.c_double), ("mass_coeff_im", C.c_double),
        ("tol", C.c_double), ("max_iter", C.c_int), ("augment", C.c_int), ("device", C.c_int),
    ]


class FetiStats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int), ("converged", C.c_int), ("relative_residual", C.c_double),
        ("primal_residual", C.c_double), ("interface_jump", C.c_double), ("n_lambda", C.c_int),
        ("coarse_dim", C.c_int), ("setup_seconds", C.c_double), ("solve_seconds", C.c_double),
    ]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["converged"] = bool(d["converged"])
        return d


class SchurStats(C.Structure):
    _fields_ = [
        ("plus", FetiStats), ("minus", FetiStats), ("imag_leak", C.c_double), ("imag_leak_warning", C.c_int),
        ("converged", C.c_int), ("factor_setup_seconds", C.c_double), ("solve_seconds", C.c_double),
    ]


class Desc3(C.Structure):
    """fetigpu3d_desc (include/fetigpu.h, 3D extension)."""
    _fields_ = [
        ("n_x", C.c_int), ("n_y", C.c_int), ("n_z", C.c_int),
        ("len_x", C.c_double), ("len_y", C.c_double), ("len_z", C.c_double),
        ("physics", C.c_int), ("young", C.c_double), ("poisson", C.c_double),
        ("s_x", C.c_int), ("s_y", C.c_int), ("s_z", C.c_int), ("phi", C.c_double),
        ("mass_coeff_re", C.c_double), ("mass_coeff_im", C.c_double),
        ("tol", C.c_double), ("max_iter", C.c_int), ("device", C.c_int),
    ]


_lib = None


def lib():
    """Load libfetigpu.so (raises OSError / ImportError when absent: no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"paper_1312_5653_b200: native library missing at {LIB_PATH}; "
                          "run `python -m paper_1312_5653_b200.build` (nvcc, sm_100a)")
    L = C.CDLL(LIB_PATH)
    dp, vp, ip = C.POINTER(C.c_double), C.c_void_p, C.POINTER(C.c_int)
    pdesc = C.POINTER(Desc)
    L.fetigpu_last_error.restype = C.c_char_p
    L.fetigpu_problem_info.argtypes = [pdesc, ip]
    L.fetigpu_context_info.argtypes = [C.c_void_p, ip]
    L.fetigpu_target_thermal.argtypes = [pdesc, dp, dp]
    L.fetigpu_target_sine.argtypes = [pdesc, C.c_ulonglong, C.c_int, C.c_int, dp]
    L.fetigpu_create.argtypes = [pdesc, C.POINTER(vp)]
    L.fetigpu_destroy.argtypes = [vp]
    L.fetigpu_schur_solve.argtypes = [vp, dp, dp, dp, dp, dp, C.POINTER(SchurStats)]
    L.fetigpu_schur_solve_device.argtypes = [vp, vp, vp, vp, vp, vp, C.POINTER(SchurStats)]
    L.fetigpu_feti_solve.argtypes = [vp, C.c_int, dp, dp, C.POINTER(FetiStats)]
    L.fetigpu_apply_dual.argtypes = [vp, C.c_int, dp, dp]
    L.fetigpu_apply_precond.argtypes = [vp, C.c_int, dp, dp]
    L.fetigpu_stream.argtypes = [vp]
    L.fetigpu_stream.restype = vp
    L.fetigpu_launch_count.argtypes = [vp, C.c_int]
    L.fetigpu_launch_count.restype = C.c_longlong
    L.fetigpu_profile.argtypes = [vp, C.c_int]
    L.fetigpu_profile_read.argtypes = [vp, dp, C.POINTER(C.c_longlong), C.c_int]
    L.fetigpu_nccl_unique_id.argtypes = [C.c_char_p]
    L.fetigpu_create_sharded.argtypes = [pdesc, C.c_int, C.c_int, C.c_char_p, C.POINTER(vp)]
    L.fetigpu_rank_info.argtypes = [pdesc, C.c_int, C.c_int, ip]
    L.fetigpu_nccl_selftest.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, dp]
    L.fetigpu_emulated_schur_solve.argtypes = [pdesc, C.c_int, dp, dp, dp, dp, dp, C.POINTER(SchurStats)]
    L.fetigpu_step_spans.argtypes = [vp, dp]
    L.fetigpu_pressure_load.argtypes = [pdesc, C.c_double, dp]
    L.fetigpu_diagnostics.argtypes = [pdesc, dp, dp, dp, dp, dp]
    L.fetigpu_full_space.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_int, dp, dp, dp, dp, dp,
                                     C.POINTER(FetiStats), dp]
    L.fetigpu_gemv_timing.argtypes = [vp, C.c_int, dp]
    L.fetigpu_class_bytes.argtypes = [vp, C.c_int]
    L.fetigpu_class_bytes.restype = C.c_double
    pd3, lp = C.POINTER(Desc3), C.POINTER(C.c_longlong)
    L.fetigpu3d_problem_info.argtypes = [pd3, lp]
    L.fetigpu3d_target_sine.argtypes = [pd3, C.c_ulonglong, C.c_int, C.c_int, dp]
    L.fetigpu3d_create.argtypes = [pd3, C.POINTER(vp)]
    L.fetigpu3d_destroy.argtypes = [vp]
    L.fetigpu3d_schur_solve.argtypes = [vp, dp, dp, dp, dp, dp, C.POINTER(SchurStats)]
    L.fetigpu3d_schur_solve_device.argtypes = [vp, vp, vp, vp, vp, vp, C.POINTER(SchurStats)]
    L.fetigpu3d_feti_solve.argtypes = [vp, C.c_int, dp, dp, C.POINTER(FetiStats)]
    L.fetigpu3d_apply_dual.argtypes = [vp, C.c_int, dp, dp]
    L.fetigpu3d_apply_precond.argtypes = [vp, C.c_int, dp, dp]
    L.fetigpu3d_stream.argtypes = [vp]
    L.fetigpu3d_stream.restype = vp
    L.fetigpu3d_launch_count.argtypes = [vp, C.c_int]
    L.fetigpu3d_launch_count.restype = C.c_longlong
    L.fetigpu3d_profile.argtypes = [vp, C.c_int]
    L.fetigpu3d_profile_read.argtypes = [vp, dp, C.POINTER(C.c_longlong), C.c_int]
    L.fetigpu3d_class_bytes.argtypes = [vp, C.c_int]
    L.fetigpu3d_class_bytes.restype = C.c_double
    L.fetigpu3d_setup_times.argtypes = [vp, dp]
    L.fetigpu3d_create_sharded.argtypes = [pd3, C.c_int, C.c_int, C.c_char_p, C.POINTER(vp)]
    L.fetigpu3d_emulated_schur_solve.argtypes = [pd3, C.c_int, dp, dp, dp, dp, dp, C.POINTER(SchurStats)]
    L.fetigpu3d_rank_info.argtypes = [pd3, C.c_int, C.c_int, lp]
    _lib = L
    return L


EXPORTED_SYMBOLS = (
    "fetigpu_problem_info", "fetigpu_context_info", "fetigpu_target_thermal", "fetigpu_target_sine", "fetigpu_create",
    "fetigpu_destroy", "fetigpu_schur_solve", "fetigpu_schur_solve_device", "fetigpu_feti_solve",
    "fetigpu_apply_dual", "fetigpu_apply_precond", "fetigpu_stream", "fetigpu_launch_count",
    "fetigpu_profile", "fetigpu_profile_read", "fetigpu_class_bytes", "fetigpu_last_error",
    "fetigpu_nccl_unique_id", "fetigpu_create_sharded", "fetigpu_rank_info", "fetigpu_emulated_schur_solve",
    "fetigpu_step_spans", "fetigpu_full_space", "fetigpu_pressure_load", "fetigpu_diagnostics",
    "fetigpu_nccl_selftest", "fetigpu_gemv_timing",
    "fetigpu3d_problem_info", "fetigpu3d_target_sine", "fetigpu3d_create", "fetigpu3d_destroy",
    "fetigpu3d_schur_solve", "fetigpu3d_schur_solve_device", "fetigpu3d_feti_solve", "fetigpu3d_apply_dual",
    "fetigpu3d_apply_precond", "fetigpu3d_stream", "fetigpu3d_launch_count", "fetigpu3d_profile",
    "fetigpu3d_profile_read", "fetigpu3d_class_bytes", "fetigpu3d_setup_times", "fetigpu3d_create_sharded",
    "fetigpu3d_emulated_schur_solve", "fetigpu3d_rank_info",
)
