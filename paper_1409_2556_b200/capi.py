"""ctypes binding of the C ABI declared in include/laptomo_gpu.h.

This is the only way Python reaches the device code: there is no CPU fallback.
If the library is missing the import of `lib()` raises; if no sm_100 device is
present `lt_ctx_create` fails with LT_ERR_CUDA.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("LT_LIB") or Path(__file__).resolve().parent / "_lib" / "liblaptomo_gpu.so")

LT_OK = 0
LT_ERR_INVALID_ARGUMENT = 1
LT_ERR_PRECONDITIONER = 2
LT_ERR_NOT_CONVERGED = 3
LT_ERR_CUDA = 4
LT_ERR_OOM = 5
LT_ERR_INTERNAL = 6
LT_MEM_HOST = 0
LT_MEM_DEVICE = 1
LT_VARIANT_FOM = 0
LT_VARIANT_GMRES = 1
LT_SOLVER_SINGLE = 0
LT_SOLVER_FLEXIBLE = 1
LT_SOLVER_DIRECT = 2
LT_GRID_FD_CELL = 0
LT_GRID_P1_TRI = 1


class LtComplex(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class LtTalbotParams(C.Structure):
    _fields_ = [("sigma0", C.c_double), ("mu0", C.c_double), ("nu", C.c_double), ("alpha", C.c_double)]


class LtGrid(C.Structure):
    _fields_ = [("kind", C.c_int), ("dim", C.c_int), ("shape", C.c_int * 3), ("h", C.c_double)]


class LtSolveOptions(C.Structure):
    _fields_ = [("variant", C.c_int), ("tol", C.c_double), ("maxit", C.c_int), ("keep_basis", C.c_int),
                ("record_history", C.c_int)]


class LtShiftStatus(C.Structure):
    _fields_ = [("converged", C.c_int), ("iteration", C.c_int), ("estimate", C.c_double),
                ("true_residual", C.c_double)]


class LtSolverConfig(C.Structure):
    _fields_ = [("kind", C.c_int), ("variant", C.c_int), ("tol", C.c_double), ("maxit", C.c_int)]


class LtSparse(C.Structure):
    _fields_ = [("outer", C.c_void_p), ("inner", C.c_void_p), ("values", C.POINTER(C.c_double)),
                ("index_bytes", C.c_int)]


PREDICT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double))
JACOBIAN_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_void_p, C.POINTER(C.c_double))


class LtGnProblem(C.Structure):
    _fields_ = [("n_y", C.c_int), ("n_s", C.c_int), ("p", C.c_int), ("y", C.POINTER(C.c_double)),
                ("r_diag", C.POINTER(C.c_double)), ("drift", C.POINTER(C.c_double)), ("prior", C.POINTER(C.c_double)),
                ("grid", LtGrid), ("n_blocks", C.c_int), ("variance", C.c_double * 2), ("corr", (C.c_double * 3) * 2),
                ("predict", PREDICT_FN), ("jacobian_and_predict", JACOBIAN_FN), ("user", C.c_void_p)]


class LtGnOptions(C.Structure):
    _fields_ = [("max_gn", C.c_int), ("rtol", C.c_double), ("damping", C.c_int), ("max_halvings", C.c_int)]


class LtGnStats(C.Structure):
    _fields_ = [("objective", C.c_double), ("misfit", C.c_double), ("prior", C.c_double), ("step_norm", C.c_double),
                ("alpha", C.c_double), ("saddle_residual", C.c_double), ("drift_violation", C.c_double)]


class LtTimeDiag(C.Structure):
    _fields_ = [("iterations", C.c_int), ("all_converged", C.c_int)]


class LtExperiment(C.Structure):
    _fields_ = [("sources", C.POINTER(C.c_double)), ("rates", C.POINTER(C.c_double)), ("n_src", C.c_int),
                ("receivers", C.POINTER(C.c_double)), ("n_rec", C.c_int),
                ("times", C.POINTER(C.c_double)), ("n_times", C.c_int), ("n_quad", C.c_int),
                ("contour", LtTalbotParams), ("solver", LtSolverConfig),
                ("include_storativity", C.c_int), ("storativity_z_factor", C.c_int)]


P = C.c_void_p
D = C.c_double
I = C.c_int
I64 = C.c_int64
PD = C.POINTER(C.c_double)
PI = C.POINTER(C.c_int)
PI64 = C.POINTER(C.c_int64)
PC = C.POINTER(LtComplex)

# name -> (restype, argtypes); every symbol of include/laptomo_gpu.h
SIGNATURES = {
    "lt_version": (C.c_char_p, []),
    "lt_last_error": (C.c_char_p, []),
    "lt_last_unconverged": (I, [PI, I]),
    "lt_ctx_create": (I, [I, C.POINTER(P)]),
    "lt_ctx_destroy": (I, [P]),
    "lt_ctx_synchronize": (I, [P]),
    "lt_ctx_stream": (P, [P]),
    "lt_ctx_set_profiling": (I, [P, I]),
    "lt_ctx_reset_profile": (I, [P]),
    "lt_ctx_set_profile_sampling": (I, [P, I]),
    "lt_ctx_profile": (I, [P, I, C.c_char_p, PD, PI64, PD]),
    "lt_ctx_launch_count": (I64, [P]),
    "lt_talbot_default_params": (None, [C.POINTER(LtTalbotParams)]),
    "lt_talbot_build": (I, [I, D, C.POINTER(LtTalbotParams), PD, PC, PC, PC]),
    "lt_qhat_step": (I, [D, LtComplex, PC]),
    "lt_sample_field_grid": (I, [P, I, PI, D, D, PD, D, C.c_uint64, PC, I, PD]),
    "lt_select_preconditioner_shifts": (I, [PC, I, PC, PI, PI, PI]),
    "lt_pencil_create_grid": (I, [P, C.POINTER(LtGrid), PD, PD, I, C.POINTER(P)]),
    "lt_pencil_create_csr": (I, [P, C.POINTER(LtGrid), I64, C.POINTER(LtSparse), C.POINTER(LtSparse), C.POINTER(P)]),
    "lt_pencil_destroy": (I, [P]),
    "lt_pencil_rows": (I64, [P]),
    "lt_pencil_parameters": (I64, [P]),
    "lt_pencil_levels": (I, [P]),
    "lt_pencil_apply": (I, [P, LtComplex, PC, PC, I, I]),
    "lt_pencil_apply_adjoint": (I, [P, LtComplex, PC, PC, I, I]),
    "lt_pencil_apply_mass": (I, [P, PC, PC, I, I]),
    "lt_pencil_prepare": (I, [P, PC, I]),
    "lt_pencil_factorization_count": (I, [P]),
    "lt_pencil_set_inner_tolerance": (I, [P, D, I]),
    "lt_pencil_solve": (I, [P, LtComplex, PC, PC, I, I]),
    "lt_pencil_solve_adjoint": (I, [P, LtComplex, PC, PC, I, I]),
    "lt_pencil_point_weights": (I, [P, PD, PI64, PD, PI]),
    "lt_solve_default_options": (None, [C.POINTER(LtSolveOptions)]),
    "lt_solve_shifted": (I, [P, PC, I, PC, I, PC, I, PI, I, C.POINTER(LtSolveOptions), I, PC,
                             C.POINTER(LtShiftStatus), PI, PD]),
    "lt_last_basis": (I, [P, I, PI, PD, PC, PC, PC, PC]),
    "lt_solve_shifted_direct": (I, [P, PC, I, PC, I, I, PC]),
    "lt_residual_estimate": (I, [PC, PC, I, LtComplex, PC, I, PD]),
    "lt_solver_default_config": (None, [C.POINTER(LtSolverConfig)]),
    "lt_forward": (I, [P, PD, PD, I, PD, PD, I, I, C.POINTER(LtTalbotParams), C.POINTER(LtSolverConfig), I, I,
                       PD, PD, I, PD, C.POINTER(LtTimeDiag), PD]),
    "lt_experiment_defaults": (None, [C.POINTER(LtExperiment)]),
    "lt_jacobian_slice": (I, [P, C.POINTER(LtExperiment), I, I, PD, PD]),
    "lt_jacobian": (I, [P, C.POINTER(LtExperiment), PD, PD]),
    "lt_predict": (I, [P, C.POINTER(LtExperiment), PD]),
    "lt_crank_nicolson": (I, [P, PD, PD, I, PD, D, PD, I, I, PD, PI]),
    "lt_pencil_condest": (I, [P, LtComplex, PD, PD, PD]),
    "lt_gn_default_options": (None, [C.POINTER(LtGnOptions)]),
    "lt_gn_step": (I, [P, C.POINTER(LtGnProblem), PD, PD, C.POINTER(LtGnOptions), PD, PD, PD, C.POINTER(LtGnStats)]),
    "lt_gn_invert": (I, [P, C.POINTER(LtGnProblem), PD, PD, C.POINTER(LtGnOptions), PD, PD, C.POINTER(LtGnStats), PI, PI,
                         C.c_char_p, I]),
    "lt_gn_objective": (I, [P, C.POINTER(LtGnProblem), PD, PD, PD, PD, PD]),
    "lt_split_solve": (I, [P, C.POINTER(LtExperiment), I, I, I, C.POINTER(P)]),
    "lt_split_columns": (I, [P]),
    "lt_split_coefficients": (I, [P, I, PC, PI]),
    "lt_split_export": (I, [P, I, I, I, P, I]),
    "lt_split_predictions": (I, [P, PD]),
    "lt_split_destroy": (I, [P]),
    "lt_jacobian_assemble_slab": (I, [P, C.POINTER(LtExperiment), I, I, I, P, I, PC, PI, I, P]),
}

_lib = None


def lib():
    """Load the in-tree library (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} not built; run paper_1409_2556_b200/build.py "
                               "(there is no CPU fallback)")
        lib_ = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib_, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib_
    return _lib


class LaptomoError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class FactorizationError(LaptomoError):
    """errors.hpp:14-17."""


class ConvergenceError(LaptomoError):
    """errors.hpp:20-25: unconverged_shifts carries the indices."""

    def __init__(self, status, message, unconverged):
        super().__init__(status, message)
        self.unconverged_shifts = list(unconverged)


class CudaError(LaptomoError):
    pass


def check(status: int) -> None:
    if status == LT_OK:
        return
    msg = lib().lt_last_error().decode(errors="replace")
    if status == LT_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == LT_ERR_PRECONDITIONER:
        raise FactorizationError(status, msg)
    if status == LT_ERR_NOT_CONVERGED:
        buf = (C.c_int * 4096)()
        cnt = lib().lt_last_unconverged(buf, 4096)
        raise ConvergenceError(status, msg, list(buf[: min(cnt, 4096)]))
    if status in (LT_ERR_CUDA, LT_ERR_OOM):
        raise CudaError(status, msg)
    raise LaptomoError(status, msg)


def cptr(a: np.ndarray):
    assert a.dtype == np.complex128 and a.flags.c_contiguous
    return a.ctypes.data_as(PC)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(PD)


def lc(z) -> LtComplex:
    z = complex(z)
    return LtComplex(z.real, z.imag)
