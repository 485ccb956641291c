"""ctypes binding of libelastodyn_b200.so (include/elastodyn_b200.h).

The library is the product: CUDA kernels for sm_100a behind a C-ABI.  It is
built in-tree by ``__graft_entry__.build()`` (``paper_1809_06350_b200/csrc/
Makefile``).  There is no CPU fallback: if the library is missing, or there is
no CUDA device, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libelastodyn_b200.so")

_i32, _i64, _f64 = C.c_int32, C.c_int64, C.c_double

ED_OK, ED_ELEMENT_INVERSION, ED_ZERO_DIAGONAL, ED_INVALID_ARGUMENT = 0, 1, 2, 3
ED_CUDA_ERROR, ED_NOT_READY, ED_UNSUPPORTED = 4, 5, 6

EXPORTED = [
    "ed_ctx_create", "ed_ctx_destroy", "ed_last_error", "ed_ctx_set_threads", "ed_kernel_launches",
    "ed_mesh_upload", "ed_dofs_build", "ed_set_material", "ed_set_loads", "ed_state_upload",
    "ed_state_download", "ed_assemble_residuals", "ed_assemble_tangent", "ed_tangent_export",
    "ed_foldin_download", "ed_block_system_upload", "ed_solve_block_system",
    "ed_solve_block_system_device", "ed_newton_first_pass", "ed_step_generalized_alpha", "ed_block_matvec", "ed_gmres_a",
    "ed_amg_vcycle", "ed_shat_export", "ed_block_matvec_device", "ed_spmv_bytes", "ed_state_save",
    "ed_state_restore", "ed_timer", "ed_bench_kernels", "ed_bench_assembly", "ed_kernel_accounting", "ed_kernel_account_count",
    "ed_kernel_account_get", "ed_set_fiber_field", "ed_set_prescribed_displacement", "ed_coupled_matvec",
]


class KrylovConfig(C.Structure):
    """KrylovConfig (krylov.hpp:64-69)."""
    _fields_ = [("restart", _i32), ("max_iters", _i32), ("rel_tol", _f64), ("abs_tol", _f64)]


class AmgOptions(C.Structure):
    """AmgOptions (amg.hpp:16-37); use_dof_row_maps reproduces set_amg_maps."""
    _fields_ = [("block_size", _i32), ("max_levels", _i32), ("coarse_max_rows", _i32),
                ("smoother", _i32), ("pre_sweeps", _i32), ("post_sweeps", _i32),
                ("smooth_prolongator", _i32), ("use_dof_row_maps", _i32),
                ("strength_theta", _f64), ("jacobi_weight", _f64)]


class BlockSolverOptions(C.Structure):
    """BlockSolverOptions (precond.hpp:167-175)."""
    _fields_ = [("precond", _i32), ("scale", _i32), ("outer", KrylovConfig), ("a", KrylovConfig),
                ("s", KrylovConfig), ("inner", KrylovConfig), ("amg_a", AmgOptions),
                ("amg_s", AmgOptions), ("eps_diag", _f64)]


class LinearStats(C.Structure):
    """LinearStats (precond.hpp:19-49)."""
    _fields_ = [("outer_iters", _i64), ("a_solves", _i64), ("a_iters", _i64), ("s_solves", _i64),
                ("s_iters", _i64), ("schur_applies", _i64), ("inner_iters", _i64),
                ("converged", _i32), ("pad", _i32), ("t_solve", _f64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


class SolveResult(C.Structure):
    """SolveResult (krylov.hpp:71-77) without the history vector."""
    _fields_ = [("converged", _i32), ("iterations", _i32), ("initial_norm", _f64), ("final_norm", _f64)]


class Material(C.Structure):
    """Material (materials.hpp:137-157) as POD."""
    _fields_ = [("kind", _i32), ("incompressible", _i32), ("rho0", _f64), ("mu", _f64),
                ("kappa", _f64), ("k1", _f64), ("k2", _f64), ("h1", _f64 * 9), ("h2", _f64 * 9)]


class TimeScalars(C.Structure):
    """TimeScalars (assembly.hpp:62-71)."""
    _fields_ = [("dt", _f64), ("alpha_m", _f64), ("alpha_f", _f64), ("gamma", _f64)]

    def chi(self):
        return self.alpha_f * self.gamma * self.dt


class NonlinearConfig(C.Structure):
    """NonlinearConfig (timeint.hpp:26-30)."""
    _fields_ = [("tol_R", _f64), ("tol_A", _f64), ("l_max", _i32), ("pad", _i32)]


class StepStats(C.Structure):
    """StepStats (timeint.hpp:35-45) without the vectors."""
    _fields_ = [("converged", _i32), ("newton_iters", _i32), ("n_res", _i32), ("pad", _i32), ("res0", _f64),
                ("res_final", _f64), ("t_assembly", _f64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


class PhaseTimes(C.Structure):
    _fields_ = [("residual_ms", _f64), ("tangent_ms", _f64), ("planes_ms", _f64), ("shat_ms", _f64),
                ("amg_setup_ms", _f64), ("fgmres_ms", _f64), ("update_ms", _f64), ("total_ms", _f64),
                ("amg_host_ms", _f64), ("kernel_launches", _i64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load the native library (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"native library missing: {LIB_PATH}; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    dp, ip = C.POINTER(_f64), C.POINTER(_i32)
    u8p = C.POINTER(C.c_uint8)
    sig = {
        "ed_ctx_create": (C.c_int, [C.c_int, C.POINTER(P)]),
        "ed_ctx_destroy": (None, [P]),
        "ed_last_error": (C.c_char_p, [P]),
        "ed_ctx_set_threads": (C.c_int, [P, C.c_int]),
        "ed_kernel_launches": (_i64, [P]),
        "ed_mesh_upload": (C.c_int, [P, C.c_int, C.c_int, ip, dp, dp, dp]),
        "ed_dofs_build": (C.c_int, [P, u8p, ip, ip]),
        "ed_set_material": (C.c_int, [P, C.POINTER(Material)]),
        "ed_set_loads": (C.c_int, [P, dp, C.c_int, ip, dp, dp]),
        "ed_set_fiber_field": (C.c_int, [P, C.c_int, dp]),
        "ed_coupled_matvec": (C.c_int, [P, C.POINTER(BlockSolverOptions), dp, dp, dp]),
        "ed_set_prescribed_displacement": (C.c_int, [P, C.c_int, ip, dp]),
        "ed_state_upload": (C.c_int, [P] + [dp] * 6),
        "ed_state_download": (C.c_int, [P] + [dp] * 6),
        "ed_assemble_residuals": (C.c_int, [P, dp, dp, ip]),
        "ed_assemble_tangent": (C.c_int, [P, C.POINTER(TimeScalars), dp, ip]),
        "ed_tangent_export": (C.c_int, [P, C.c_int, ip, ip, ip, dp]),
        "ed_foldin_download": (C.c_int, [P, dp, dp]),
        "ed_block_system_upload": (C.c_int, [P, C.c_int, C.c_int] + [ip, ip, dp] * 4),
        "ed_solve_block_system": (C.c_int, [P, dp, dp, C.POINTER(BlockSolverOptions),
                                            C.POINTER(LinearStats), dp, _i32, ip]),
        "ed_solve_block_system_device": (C.c_int, [P, C.c_void_p, C.c_void_p, C.POINTER(BlockSolverOptions),
                                                   C.POINTER(LinearStats), dp, _i32, ip]),
        "ed_newton_first_pass": (C.c_int, [P, C.POINTER(TimeScalars), C.POINTER(BlockSolverOptions), dp, dp,
                                           C.POINTER(LinearStats), dp, _i32, ip, C.POINTER(PhaseTimes)]),
        "ed_step_generalized_alpha": (C.c_int, [P, C.POINTER(TimeScalars), C.POINTER(NonlinearConfig),
                                                C.POINTER(BlockSolverOptions), C.POINTER(StepStats),
                                                C.POINTER(LinearStats), dp, _i32]),
        "ed_block_matvec": (C.c_int, [P, dp, dp]),
        "ed_gmres_a": (C.c_int, [P, dp, dp, C.POINTER(KrylovConfig), C.c_int, C.c_int,
                                 C.POINTER(AmgOptions), C.POINTER(SolveResult), dp, _i32, ip]),
        "ed_amg_vcycle": (C.c_int, [P, C.c_int, C.POINTER(BlockSolverOptions), dp, dp, ip]),
        "ed_shat_export": (C.c_int, [P, C.POINTER(BlockSolverOptions), ip, ip, ip, dp]),
        "ed_block_matvec_device": (C.c_int, [P, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_float)]),
        "ed_spmv_bytes": (C.c_int, [P, dp, dp]),
        "ed_state_save": (C.c_int, [P]),
        "ed_state_restore": (C.c_int, [P]),
        "ed_timer": (C.c_int, [P, C.c_int, C.POINTER(C.c_float)]),
        "ed_bench_kernels": (C.c_int, [P, C.POINTER(BlockSolverOptions), C.c_int, dp]),
        "ed_bench_assembly": (C.c_int, [P, C.POINTER(TimeScalars), C.c_int, dp]),
        "ed_kernel_accounting": (C.c_int, [P, C.c_int]),
        "ed_kernel_account_count": (C.c_int, [P, C.POINTER(C.c_int)]),
        "ed_kernel_account_get": (C.c_int, [P, C.c_int, C.c_char_p, C.c_int, C.POINTER(_i64), dp, dp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(_f64))


def ip(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(_i32))


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)
