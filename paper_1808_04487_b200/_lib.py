"""ctypes binding of the C ABI in include/veloreg_gpu.h (libveloreg_gpu.so).

The shared library is built in-tree (``make -C paper_1808_04487_b200``). There is
no CPU fallback: importing the package without the library, or calling it
without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VR_LIB", os.path.join(_HERE, "libveloreg_gpu.so"))

from ._abi_types import *  # noqa: F401,F403  (POD layouts, constants, errors)
from ._abi_types import _EXC_BY_CLASS, _EXC_BY_STATUS  # noqa: F401

P = C.c_void_p
D = C.c_double
I = C.c_int
DP = C.c_void_p  # device pointer
HP = C.c_void_p  # host pointer

# name -> (restype, argtypes); all status-returning functions have restype int
SIGNATURES = {
    "vr_last_error": (C.c_char_p, []),
    "vr_last_error_class": (I, []),
    "vr_abi_version": (I, []),
    "vr_model_default": (None, [C.POINTER(Model)]),
    "vr_solver_params_default": (None, [C.POINTER(SolverParams)]),
    "vr_model_validate": (I, [C.POINTER(Model)]),
    "vr_solver_params_validate": (I, [C.POINTER(SolverParams)]),
    "vr_ctx_create": (I, [I, I, I, I, C.POINTER(P)]),
    "vr_ctx_destroy": (I, [P]),
    "vr_ctx_synchronize": (I, [P]),
    "vr_ctx_stream": (P, [P]),
    "vr_ctx_grid": (I, [P, C.POINTER(C.c_int)]),
    "vr_ctx_kernel_launches": (C.c_longlong, [P]),
    "vr_ctx_reset_kernel_launches": (None, [P]),
    "vr_ctx_memory": (I, [P, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "vr_ctx_reset_memory_peak": (I, [P]),
    "vr_ctx_set_profiling": (I, [P, I]),
    "vr_ctx_profile_read": (I, [P, C.c_char_p, C.c_size_t]),
    "vr_device_alloc": (I, [P, C.c_size_t, C.POINTER(P)]),
    "vr_device_free": (I, [P, P]),
    "vr_host_alloc_pinned": (I, [C.c_size_t, C.POINTER(P)]),
    "vr_host_free_pinned": (I, [P]),
    "vr_memcpy_h2d": (I, [P, DP, HP, C.c_size_t]),
    "vr_memcpy_d2h": (I, [P, HP, DP, C.c_size_t]),
    "vr_memcpy_d2d": (I, [P, DP, DP, C.c_size_t]),
    "vr_memset_zero": (I, [P, DP, C.c_size_t]),
    "vr_scale": (I, [P, DP, I, D]),
    "vr_add_scaled": (I, [P, DP, D, DP, I]),
    "vr_lin_comb": (I, [P, DP, D, DP, D, DP, I]),
    "vr_dot_l2": (I, [P, DP, DP, I, C.POINTER(D)]),
    "vr_norm_l2": (I, [P, DP, I, C.POINTER(D)]),
    "vr_max_abs": (I, [P, DP, I, C.POINTER(D)]),
    "vr_max_magnitude": (I, [P, DP, C.POINTER(D)]),
    "vr_all_finite": (I, [P, DP, I, C.POINTER(C.c_int)]),
    "vr_inner_product": (I, [P, DP, DP, I, C.POINTER(D)]),
    "vr_fft_r2c": (I, [P, DP, DP]),
    "vr_fft_c2r": (I, [P, DP, DP]),
    "vr_gradient": (I, [P, DP, DP]),
    "vr_divergence": (I, [P, DP, DP]),
    "vr_laplacian": (I, [P, DP, DP, I]),
    "vr_helmholtz1_apply": (I, [P, DP, DP]),
    "vr_gaussian_smooth": (I, [P, DP, DP, I, C.POINTER(D)]),
    "vr_apply_reg_operator": (I, [P, DP, DP, C.POINTER(RegNorm), I, D]),
    "vr_apply_projection": (I, [P, DP, DP, I, D, D]),
    "vr_rescale_intensity": (I, [P, DP, DP, C.POINTER(C.c_int)]),
    "vr_tricubic_interpolate": (I, [P, DP, DP, DP, I]),
    "vr_trace_characteristics": (I, [P, DP, I, I, DP]),
    "vr_continuity_factor": (I, [P, DP, DP, D, DP]),
    "vr_solve_state": (I, [P, DP, DP, I, DP]),
    "vr_solve_adjoint": (I, [P, DP, DP, I, DP, DP]),
    "vr_gradient_dot": (I, [P, DP, DP, DP]),
    "vr_solve_inc_state": (I, [P, DP, DP, DP, I, DP]),
    "vr_solve_inc_adjoint": (I, [P, DP, DP, I, DP, DP]),
    "vr_objective_create": (I, [P, DP, DP, C.POINTER(Model), C.POINTER(P)]),
    "vr_objective_destroy": (I, [P]),
    "vr_objective_initial_mismatch": (I, [P, C.POINTER(D)]),
    "vr_objective_counters": (I, [P, C.POINTER(Counters)]),
    "vr_objective_reset_counters": (I, [P]),
    "vr_objective_set_beta": (I, [P, D]),
    "vr_evaluate": (I, [P, DP, C.POINTER(P)]),
    "vr_state_destroy": (I, [P]),
    "vr_state_scalars": (I, [P, C.POINTER(D), C.POINTER(D), C.POINTER(D), C.POINTER(C.c_int),
                             C.POINTER(C.c_int)]),
    "vr_state_get": (I, [P, I, DP]),
    "vr_compute_gradient": (I, [P, P, DP]),
    "vr_hessian_matvec": (I, [P, P, DP, DP]),
    "vr_hessian_matvec_host": (I, [P, P, HP, HP]),
    "vr_hessian_data_matvec": (I, [P, P, DP, DP]),
    "vr_hessian_matvec_host_async": (I, [P, P, HP, HP]),
    "vr_tricubic_interpolate_f32": (I, [P, DP, DP, DP, I]),
    "vr_trace_characteristics_f32": (I, [P, DP, I, I, DP]),
    "vr_solve_state_f32": (I, [P, DP, DP, I, DP]),
    "vr_objective_f32_create": (I, [P, DP, DP, C.POINTER(Model), C.POINTER(P)]),
    "vr_objective_f32_destroy": (I, [P]),
    "vr_objective_f32_counters": (I, [P, C.POINTER(Counters)]),
    "vr_evaluate_f32": (I, [P, DP, C.POINTER(P)]),
    "vr_state_f32_destroy": (I, [P]),
    "vr_state_f32_scalars": (I, [P, C.POINTER(D), C.POINTER(D), C.POINTER(D)]),
    "vr_compute_gradient_f32": (I, [P, P, DP]),
    "vr_hessian_matvec_f32": (I, [P, P, DP, DP]),
    "vr_gauss_newton_solve_f32": (I, [P, DP, DP, DP, C.POINTER(Model), C.POINTER(SolverParams), I,
                                      DP, C.POINTER(SolveReport), C.POINTER(IterationRecord), I]),
    "vr_gauss_newton_solve_two_level_f32": (I, [P, DP, DP, DP, C.POINTER(Model), C.POINTER(SolverParams),
                                                C.POINTER(TwoLevelOptions), DP, C.POINTER(SolveReport),
                                                C.POINTER(IterationRecord), I]),
    "vr_parameter_continuation_f32": (I, [P, DP, DP, DP, C.POINTER(Model), C.POINTER(SolverParams), I,
                                          DP, C.POINTER(SolveReport), I, C.POINTER(C.c_int),
                                          C.POINTER(IterationRecord), I]),
    "vr_fft_r2c_f32": (I, [P, DP, DP]),
    "vr_fft_c2r_f32": (I, [P, DP, DP]),
    "vr_gradient_f32": (I, [P, DP, DP]),
    "vr_divergence_f32": (I, [P, DP, DP]),
    "vr_gaussian_smooth_f32": (I, [P, DP, DP, I, C.POINTER(D)]),
    "vr_apply_reg_operator_f32": (I, [P, DP, DP, C.POINTER(RegNorm), I, D]),
    "vr_apply_projection_f32": (I, [P, DP, DP, I, D, D]),
    "vr_objective_wait": (I, [P]),
    "vr_objective_apply_reg": (I, [P, DP, I, DP]),
    "vr_objective_apply_K": (I, [P, DP, DP]),
    "vr_compute_forcing": (I, [D, D, C.POINTER(D)]),
    "vr_solve_report_csv": (I, [C.POINTER(SolveReport), C.POINTER(IterationRecord), C.c_char_p,
                                C.POINTER(C.c_char), C.c_size_t, C.POINTER(C.c_size_t)]),
    "vr_pcg_solve": (I, [P, P, DP, D, I, I, DP, C.POINTER(PcgStats)]),
    "vr_gauss_newton_solve": (I, [P, DP, DP, DP, C.POINTER(Model), C.POINTER(SolverParams), I,
                                  DP, C.POINTER(SolveReport), C.POINTER(IterationRecord), I]),
    "vr_parameter_continuation": (I, [P, DP, DP, DP, C.POINTER(Model),
                                      C.POINTER(SolverParams), I, DP, C.POINTER(SolveReport), I,
                                      C.POINTER(C.c_int), C.POINTER(IterationRecord), I]),
    "vr_generate_synthetic": (I, [P, I, D, DP, DP, DP]),
    "vr_grid_continuation": (I, [P, DP, DP, DP, C.POINTER(Model), C.POINTER(SolverParams), I, I,
                                 DP, C.POINTER(SolveReport), I, C.POINTER(C.c_int),
                                 C.POINTER(IterationRecord), I]),
    "vr_scale_continuation": (I, [P, DP, DP, DP, C.POINTER(Model), C.POINTER(SolverParams), I,
                                  C.POINTER(D), I, DP, C.POINTER(SolveReport), I,
                                  C.POINTER(C.c_int), C.POINTER(IterationRecord), I]),
    "vr_beta_search_params_default": (None, [C.POINTER(BetaSearchParams)]),
    "vr_beta_search": (I, [P, DP, DP, DP, C.POINTER(Model), C.POINTER(SolverParams), I,
                           C.POINTER(BetaSearchParams), C.POINTER(D), DP, C.POINTER(BetaTrial), I,
                           C.POINTER(C.c_int)]),
    "vr_det_deformation_gradient": (I, [P, DP, I, DP]),
    "vr_deformation_map": (I, [P, DP, I, I, DP]),
    "vr_det_stats": (I, [P, DP, DP, D, C.POINTER(DetSummary)]),
    "vr_transport_labels": (I, [P, DP, DP, I, DP]),
    "vr_overlap_scores": (I, [P, DP, DP, DP, I, C.POINTER(C.c_int), C.POINTER(C.c_int),
                              C.POINTER(Overlap), C.POINTER(Overlap)]),
    "vr_twolevel_options_default": (None, [C.POINTER(TwoLevelOptions)]),
    "vr_spectral_resample": (I, [P, DP, I, P, DP]),
    "vr_frequency_filter": (I, [P, DP, I, I, C.POINTER(C.c_int), DP]),
    "vr_split_matvec": (I, [P, P, DP, DP]),
    "vr_twolevel_create": (I, [C.POINTER(TwoLevelOptions), C.POINTER(P)]),
    "vr_twolevel_destroy": (I, [P]),
    "vr_twolevel_rebuild": (I, [P, P, P, D]),
    "vr_twolevel_apply": (I, [P, P, DP, DP]),
    "vr_twolevel_coarse_matvec": (I, [P, DP, DP]),
    "vr_twolevel_info": (I, [P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                             C.POINTER(D), C.POINTER(Counters)]),
    "vr_gauss_newton_solve_two_level": (I, [P, DP, DP, DP, C.POINTER(Model),
                                            C.POINTER(SolverParams), C.POINTER(TwoLevelOptions),
                                            DP, C.POINTER(SolveReport),
                                            C.POINTER(IterationRecord), I]),
    "vr_nccl_unique_id": (I, [C.c_char_p]),
    "vr_slab_layout": (I, [I, I, I, I, I, I, C.POINTER(C.c_longlong)]),
    "vr_slab_halo_required": (I, [C.c_double, I, I, C.POINTER(C.c_int)]),
    "vr_ctx_create_dist": (I, [I, I, I, I, I, I, C.c_char_p, I, C.POINTER(P)]),
    "vr_ctx_slab": (I, [P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                        C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "vr_dist_selftest_objective": (I, [I, I, I, I, I, I, C.POINTER(Model), HP, HP, HP, HP, HP, HP,
                                       HP, HP]),
    "vr_dist_selftest_solve": (I, [I, I, I, I, I, I, C.POINTER(Model), C.POINTER(SolverParams),
                                   HP, HP, HP, HP, C.POINTER(SolveReport)]),
    "vr_dist_selftest_postprocess": (I, [I, I, I, I, I, I, HP, I, HP, HP, HP]),
    "vr_dist_selftest_labels": (I, [I, I, I, I, I, I, HP, HP, I, HP, I, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(Overlap), C.POINTER(Overlap)]),
    "vr_dist_selftest_solve_precond": (I, [I, I, I, I, I, I, C.POINTER(Model), C.POINTER(SolverParams), I,
                                           C.POINTER(TwoLevelOptions), HP, HP, HP, HP,
                                           C.POINTER(SolveReport)]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libveloreg_gpu.so and declare every exported symbol. Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `make -C {_HERE}` (no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status == 0:
        return
    lib = load()
    msg = lib.vr_last_error().decode(errors="replace")
    cls = _EXC_BY_CLASS.get(lib.vr_last_error_class(), _EXC_BY_STATUS.get(status, VelouregError))
    raise cls(msg)


def call(name: str, *args):
    fn = getattr(load(), name)
    check(fn(*args))
