"""CPU-only checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/veloreg_gpu.h declares, and maps errors/defaults like the reference."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "veloreg_gpu.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vr_[A-Za-z0-9_]+)\s*\(", text)))


def test_header_declares_api():
    names = declared_functions()
    for must in ["vr_ctx_create", "vr_evaluate", "vr_compute_gradient", "vr_hessian_matvec",
                 "vr_hessian_matvec_host", "vr_gauss_newton_solve", "vr_fft_r2c", "vr_tricubic_interpolate"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1808_04487_b200 import _lib
    lib = _lib.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # every declared function has a Python signature and vice versa
    assert set(declared_functions()) == set(_lib.SIGNATURES)


def test_defaults_match_reference():
    # RegModel defaults objective.hpp:11-16, RegNorm spectral.hpp:76-80, SolverParams solver.hpp:13-23
    import paper_1808_04487_b200 as vr
    from paper_1808_04487_b200 import _lib
    m = _lib.Model()
    _lib.load().vr_model_default(C.byref(m))
    assert (m.norm.kind, m.norm.gamma, m.norm.helmholtz_squared, m.norm.div_penalty, m.norm.beta_w) == (1, 1.0, 1, 0, 1e-4)
    assert (m.projection, m.beta_v, m.nt, m.gauss_newton) == (0, 1e-2, 4, 1)
    p = vr.make_params()
    assert (p.eps_opt, p.abs_grad_tol, p.max_newton, p.max_krylov) == (5e-2, 1e-6, 50, 100)
    assert (p.armijo_c1, p.armijo_backtrack, p.armijo_max_trials, p.squared_norm_stop) == (1e-4, 0.5, 20, 1)


def test_validation_and_error_mapping():
    import paper_1808_04487_b200 as vr
    from paper_1808_04487_b200 import _lib
    lib = _lib.load()
    bad = vr.make_model(beta_v=0.0)
    assert lib.vr_model_validate(C.byref(bad)) == 4  # ErrorCategory::argument
    with pytest.raises(vr.ArgumentError):
        _lib.check(lib.vr_model_validate(C.byref(bad)))
    bad = vr.make_model(kind="helmholtz", gamma=-1.0)
    with pytest.raises(vr.ArgumentError):
        _lib.check(lib.vr_model_validate(C.byref(bad)))
    p = vr.make_params(armijo_backtrack=1.5)
    with pytest.raises(vr.ArgumentError):
        _lib.check(lib.vr_solver_params_validate(C.byref(p)))
    # Grid3 rejects dims < 4 with DimensionError (grid.hpp:24-31) before touching a device
    with pytest.raises(vr.DimensionError):
        vr.Context((3, 8, 8))
    with pytest.raises(vr.DimensionError):
        vr.Context((12, 8, 10))
    # compute_forcing (solver.cpp:23-27)
    assert vr.compute_forcing(1.0, 1.0) == 0.5
    assert abs(vr.compute_forcing(0.04, 1.0) - 0.2) < 1e-15
    with pytest.raises(vr.LogicError):
        vr.compute_forcing(1.0, 0.0)


def test_dimension_error_is_argument_error():
    import paper_1808_04487_b200 as vr
    assert issubclass(vr.DimensionError, vr.ArgumentError)
    assert vr.NumericError.category == 5 and vr.LogicError.category == 8


def test_no_cpu_fallback_without_device():
    import paper_1808_04487_b200 as vr
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("device present")
    except ImportError:
        pass
    with pytest.raises(vr.ResourceError):
        vr.Context(16)
