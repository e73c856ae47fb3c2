"""POD layouts, constants and error classes of the C ABI (include/veloreg_gpu.h).

Pure ctypes declarations: importing this module never loads libveloreg_gpu.so,
so the test-only oracle harness (oracle/ref.py) can share the layouts without
mapping the product library into the reference arm's process.
"""
from __future__ import annotations

import ctypes as C

# ---- error hierarchy mirroring veloreg::Error (proj/include/veloreg/errors.hpp:9-67)


class VelouregError(RuntimeError):
    category = 0


class IoError(VelouregError):
    category = 2


class FormatError(VelouregError):
    category = 3


class ArgumentError(VelouregError):
    category = 4


class DimensionError(ArgumentError):
    pass


class NumericError(VelouregError):
    category = 5


class ConvergenceError(VelouregError):
    category = 6


class ResourceError(VelouregError):
    category = 7


class LogicError(VelouregError):
    category = 8


_EXC_BY_CLASS = {
    1: IoError,
    2: FormatError,
    3: ArgumentError,
    4: DimensionError,
    5: NumericError,
    6: ConvergenceError,
    7: ResourceError,
    8: LogicError,
}
_EXC_BY_STATUS = {2: IoError, 3: FormatError, 4: ArgumentError, 5: NumericError,
                  6: ConvergenceError, 7: ResourceError, 8: LogicError}

# ---- POD mirrors ------------------------------------------------------------


class RegNorm(C.Structure):
    _fields_ = [("kind", C.c_int), ("gamma", C.c_double), ("helmholtz_squared", C.c_int),
                ("div_penalty", C.c_int), ("beta_w", C.c_double)]


class Model(C.Structure):
    _fields_ = [("norm", RegNorm), ("projection", C.c_int), ("beta_v", C.c_double),
                ("nt", C.c_int), ("gauss_newton", C.c_int)]


class SolverParams(C.Structure):
    _fields_ = [("eps_opt", C.c_double), ("abs_grad_tol", C.c_double), ("max_newton", C.c_int),
                ("max_krylov", C.c_int), ("armijo_c1", C.c_double),
                ("armijo_backtrack", C.c_double), ("armijo_max_trials", C.c_int),
                ("squared_norm_stop", C.c_int)]


class Counters(C.Structure):
    _fields_ = [("objective_evals", C.c_long), ("gradient_evals", C.c_long),
                ("hessian_matvecs", C.c_long), ("pde_solves", C.c_long)]


class IterationRecord(C.Structure):
    _fields_ = [("k", C.c_int), ("objective", C.c_double), ("mismatch_rel", C.c_double),
                ("grad_norm", C.c_double), ("grad_rel", C.c_double),
                ("step_length", C.c_double), ("forcing", C.c_double),
                ("inner_iterations", C.c_int), ("fine_matvecs", C.c_long),
                ("coarse_matvecs", C.c_long), ("pde_solves", C.c_long),
                ("wall_time_s", C.c_double)]


class SolveReport(C.Structure):
    _fields_ = [("stop", C.c_int), ("success", C.c_int), ("outer_iterations", C.c_int),
                ("grad0", C.c_double), ("final_grad_rel", C.c_double),
                ("final_mismatch_rel", C.c_double), ("final_objective", C.c_double),
                ("wall_time_s", C.c_double), ("fine", Counters), ("coarse", Counters),
                ("n_records", C.c_int)]


class TwoLevelOptions(C.Structure):
    _fields_ = [("inner", C.c_int), ("kappa", C.c_double), ("cheb_iterations", C.c_int),
                ("max_inner_iterations", C.c_int), ("lanczos_iterations", C.c_int),
                ("lanczos_seed", C.c_ulonglong)]


class PcgStats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("rel_residual", C.c_double), ("converged", C.c_int),
                ("negative_curvature", C.c_int), ("hit_max_iterations", C.c_int)]


class BetaSearchParams(C.Structure):
    _fields_ = [("eps_J", C.c_double), ("beta_lo", C.c_double), ("beta_hi", C.c_double),
                ("max_bisections", C.c_int), ("min_width_decades", C.c_double)]


class DetSummary(C.Structure):
    _fields_ = [("min", C.c_double), ("mean", C.c_double), ("max", C.c_double)]


class BetaTrial(C.Structure):
    _fields_ = [("beta", C.c_double), ("feasible", C.c_int), ("det", DetSummary),
                ("report", SolveReport)]


class Overlap(C.Structure):
    _fields_ = [("dice", C.c_double), ("false_positive_rate", C.c_double),
                ("false_negative_rate", C.c_double)]


# constants (veloreg_gpu.h)
REG_H1, REG_H2, REG_H3, REG_HELMHOLTZ = 0, 1, 2, 3
REGOP_APPLY, REGOP_INVERSE, REGOP_INVERSE_SQRT = 0, 1, 2
PROJ_IDENTITY, PROJ_INCOMPRESSIBLE, PROJ_NEAR_INCOMPRESSIBLE = 0, 1, 2
TRACE_BACKWARD, TRACE_FORWARD = 0, 1
PRECOND_NONE, PRECOND_SPECTRAL, PRECOND_TWO_LEVEL = 0, 1, 2
INNER_PCG, INNER_CHEB = 0, 1
STOP_NAMES = ["zero_gradient", "converged_rel", "converged_abs", "max_iterations",
              "line_search_failure"]
(STATE_V, STATE_X_BWD, STATE_X_FWD, STATE_FACTOR, STATE_M_HISTORY, STATE_GRADIENT, STATE_GRAD_M,
 STATE_LAMBDA_HISTORY) = range(8)


_KIND = {"h1": REG_H1, "h2": REG_H2, "h3": REG_H3, "helmholtz": REG_HELMHOLTZ}
_PROJ = {"identity": PROJ_IDENTITY, "incompressible": PROJ_INCOMPRESSIBLE,
         "near_incompressible": PROJ_NEAR_INCOMPRESSIBLE}


def _enum(table, v):
    return table[v] if isinstance(v, str) else int(v)


def make_norm(kind="h2", gamma=1.0, helmholtz_squared=True, div_penalty=False, beta_w=1e-4):
    """RegNorm (spectral.hpp:75-102)."""
    return RegNorm(_enum(_KIND, kind), gamma, int(helmholtz_squared), int(div_penalty), beta_w)


def make_model(kind="h2", beta_v=1e-2, nt=4, projection="identity", gamma=1.0,
               helmholtz_squared=True, div_penalty=False, beta_w=1e-4, gauss_newton=True):
    """RegModel (objective.hpp:11-23); defaults are the reference's."""
    m = Model()
    m.norm = make_norm(kind, gamma, helmholtz_squared, div_penalty, beta_w)
    m.projection = _enum(_PROJ, projection)
    m.beta_v = beta_v
    m.nt = nt
    m.gauss_newton = int(gauss_newton)
    return m
