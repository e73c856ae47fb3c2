"""oracle/ref.py -- TEST INFRASTRUCTURE ONLY: ctypes access to the compiled reference.

Loads oracle/_ref/libveloreg_ref.so (the UNMODIFIED reference sources from
/root/reference/proj/src compiled with the FFTW/doctest shims plus the
ref_capi.cpp harness, see oracle/Makefile) and exposes the reference's
operators on host numpy arrays with the same names as the product's Python
mirror (paper_1808_04487_b200.veloreg). Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libveloreg_ref.so")
sys.path.insert(0, os.path.dirname(_HERE))
# POD layouts only: _abi_types is pure ctypes declarations and the package __init__ is lazy,
# so this import never maps libveloreg_gpu.so into a reference-arm process
from paper_1808_04487_b200 import _abi_types as _gpu_lib_types  # noqa: E402

make_model = _gpu_lib_types.make_model
make_norm = _gpu_lib_types.make_norm

RegNorm = _gpu_lib_types.RegNorm
Model = _gpu_lib_types.Model
SolverParams = _gpu_lib_types.SolverParams
Counters = _gpu_lib_types.Counters
SolveReport = _gpu_lib_types.SolveReport
IterationRecord = _gpu_lib_types.IterationRecord
PcgStats = _gpu_lib_types.PcgStats
TwoLevelOptions = _gpu_lib_types.TwoLevelOptions
BetaSearchParams = _gpu_lib_types.BetaSearchParams

_lib = None
P, D, I = C.c_void_p, C.c_double, C.c_int
DIMS = C.POINTER(C.c_int)
_SIG = {
    "vref_last_error": (C.c_char_p, []),
    "vref_last_error_class": (I, []),
    "vref_set_workers": (None, [I]),
    "vref_workers": (I, []),
    "vref_fft_r2c": (I, [DIMS, P, P]),
    "vref_fft_c2r": (I, [DIMS, P, P]),
    "vref_gradient": (I, [DIMS, P, P]),
    "vref_divergence": (I, [DIMS, P, P]),
    "vref_laplacian": (I, [DIMS, P, P]),
    "vref_helmholtz1_apply": (I, [DIMS, P, P]),
    "vref_gaussian_smooth": (I, [DIMS, P, P, C.POINTER(D)]),
    "vref_apply_reg_operator": (I, [DIMS, P, P, C.POINTER(RegNorm), I, D]),
    "vref_apply_projection": (I, [DIMS, P, P, I, D, D]),
    "vref_rescale_intensity": (I, [DIMS, P, P, C.POINTER(C.c_int)]),
    "vref_inner_product": (I, [DIMS, P, P, I, C.POINTER(D)]),
    "vref_dot_l2": (I, [DIMS, P, P, I, C.POINTER(D)]),
    "vref_max_magnitude": (I, [DIMS, P, C.POINTER(D)]),
    "vref_tricubic_interpolate": (I, [DIMS, P, P, P, I]),
    "vref_trace_characteristics": (I, [DIMS, P, I, I, P]),
    "vref_continuity_factor": (I, [DIMS, P, P, D, P]),
    "vref_solve_state": (I, [DIMS, P, P, I, P]),
    "vref_solve_adjoint": (I, [DIMS, P, P, I, P, P]),
    "vref_gradient_dot": (I, [DIMS, P, P, P]),
    "vref_solve_inc_state": (I, [DIMS, P, P, P, I, I, P]),
    "vref_solve_inc_adjoint": (I, [DIMS, P, P, I, P, P]),
    "vref_objective_create": (I, [DIMS, P, P, C.POINTER(Model), C.POINTER(P)]),
    "vref_objective_destroy": (None, [P]),
    "vref_objective_initial_mismatch": (I, [P, C.POINTER(D)]),
    "vref_objective_counters": (I, [P, C.POINTER(Counters)]),
    "vref_evaluate": (I, [P, P, C.POINTER(P)]),
    "vref_state_destroy": (None, [P]),
    "vref_state_scalars": (I, [P, C.POINTER(D), C.POINTER(D), C.POINTER(D), C.POINTER(C.c_int),
                               C.POINTER(C.c_int)]),
    "vref_state_get": (I, [P, I, P]),
    "vref_compute_gradient": (I, [P, P, P]),
    "vref_hessian_matvec": (I, [P, P, P, P]),
    "vref_hessian_data_matvec": (I, [P, P, P, P]),
    "vref_objective_apply_reg": (I, [P, P, I, P]),
    "vref_objective_apply_K": (I, [P, P, P]),
    "vref_pcg_solve": (I, [P, P, P, D, I, I, P, C.POINTER(PcgStats)]),
    "vref_gauss_newton_solve_csv": (I, [DIMS, P, P, P, C.POINTER(Model), C.POINTER(SolverParams),
                                        C.POINTER(C.c_char), I]),
    "vref_gauss_newton_solve": (I, [DIMS, P, P, P, C.POINTER(Model), C.POINTER(SolverParams), I, P,
                                    C.POINTER(SolveReport), C.POINTER(IterationRecord), I]),
    "vref_parameter_continuation": (I, [DIMS, P, P, P, C.POINTER(Model), C.POINTER(SolverParams), I,
                                        P, C.POINTER(SolveReport), I, C.POINTER(C.c_int),
                                        C.POINTER(IterationRecord), I]),
    "vref_generate_synthetic": (I, [DIMS, I, D, P, P, P]),
    "vref_make_ball_labels": (I, [DIMS, I, P]),
    "vref_det_deformation_gradient": (I, [DIMS, P, I, P]),
    "vref_tricubic_interpolate_f32": (I, [DIMS, P, P, P, I]),
    "vref_objective_f32_create": (I, [DIMS, P, P, C.POINTER(Model), C.POINTER(P)]),
    "vref_objective_f32_destroy": (None, [P]),
    "vref_evaluate_f32": (I, [P, P, C.POINTER(P)]),
    "vref_state_f32_destroy": (None, [P]),
    "vref_state_f32_scalars": (I, [P, C.POINTER(D), C.POINTER(D), C.POINTER(D)]),
    "vref_compute_gradient_f32": (I, [P, P, P]),
    "vref_hessian_matvec_f32": (I, [P, P, P, P]),
    "vref_objective_f32_counters": (I, [P, C.POINTER(Counters)]),
    "vref_gauss_newton_solve_f32": (I, [DIMS, P, P, P, C.POINTER(Model), C.POINTER(SolverParams), I, P,
                                        C.POINTER(SolveReport), C.POINTER(IterationRecord), I]),
    "vref_parameter_continuation_f32": (I, [DIMS, P, P, P, C.POINTER(Model), C.POINTER(SolverParams), I,
                                            P, C.POINTER(SolveReport), I, C.POINTER(C.c_int),
                                            C.POINTER(IterationRecord), I]),
    "vref_fft_r2c_f32": (I, [DIMS, P, P]),
    "vref_fft_c2r_f32": (I, [DIMS, P, P]),
    "vref_gradient_f32": (I, [DIMS, P, P]),
    "vref_divergence_f32": (I, [DIMS, P, P]),
    "vref_gaussian_smooth_f32": (I, [DIMS, P, P, C.POINTER(D)]),
    "vref_apply_reg_operator_f32": (I, [DIMS, P, P, C.POINTER(RegNorm), I, D]),
    "vref_apply_projection_f32": (I, [DIMS, P, P, I, D, D]),
    "vref_trace_characteristics_f32": (I, [DIMS, P, I, I, P]),
    "vref_solve_state_f32": (I, [DIMS, P, P, I, P]),
    "vref_deformation_map": (I, [DIMS, P, I, I, P]),
    "vref_det_stats": (I, [DIMS, P, P, D, C.POINTER(D)]),
    "vref_transport_labels": (I, [DIMS, P, P, I, P]),
    "vref_overlap_scores": (I, [DIMS, P, P, P, I, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                C.POINTER(D), C.POINTER(D)]),
    "vref_grid_continuation": (I, [DIMS, P, P, P, C.POINTER(Model), C.POINTER(SolverParams), I, I,
                                   P, C.POINTER(SolveReport), I, C.POINTER(C.c_int),
                                   C.POINTER(IterationRecord), I]),
    "vref_scale_continuation": (I, [DIMS, P, P, P, C.POINTER(Model), C.POINTER(SolverParams), I,
                                    C.POINTER(D), I, P, C.POINTER(SolveReport), I,
                                    C.POINTER(C.c_int), C.POINTER(IterationRecord), I]),
    "vref_beta_search": (I, [DIMS, P, P, P, C.POINTER(Model), C.POINTER(SolverParams), I,
                             C.POINTER(BetaSearchParams), C.POINTER(D), P, C.POINTER(D),
                             C.POINTER(SolveReport), I, C.POINTER(C.c_int)]),
    "vref_spectral_resample": (I, [DIMS, P, I, DIMS, P]),
    "vref_frequency_filter": (I, [DIMS, P, I, I, DIMS, P]),
    "vref_split_matvec": (I, [P, P, P, P]),
    "vref_twolevel_create": (I, [C.POINTER(TwoLevelOptions), C.POINTER(P)]),
    "vref_twolevel_destroy": (None, [P]),
    "vref_twolevel_rebuild": (I, [P, P, P, D]),
    "vref_twolevel_apply": (I, [P, P, P]),
    "vref_twolevel_coarse_matvec": (I, [P, P, P]),
    "vref_twolevel_info": (I, [P, DIMS, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(D),
                               C.POINTER(Counters)]),
    "vref_gauss_newton_solve_two_level": (I, [DIMS, P, P, P, C.POINTER(Model),
                                              C.POINTER(SolverParams), C.POINTER(TwoLevelOptions),
                                              P, C.POINTER(SolveReport), C.POINTER(IterationRecord),
                                              I]),
    "vref_gauss_newton_solve_two_level_f32": (I, [DIMS, P, P, P, C.POINTER(Model),
                                                  C.POINTER(SolverParams), C.POINTER(TwoLevelOptions),
                                                  P, C.POINTER(SolveReport), C.POINTER(IterationRecord),
                                                  I]),
    "vref_random_smooth_scalar": (I, [DIMS, I, C.c_ulonglong, D, P]),
    "vref_random_smooth_vector": (I, [DIMS, I, C.c_ulonglong, D, P]),
    "vref_random_rough_scalar": (I, [DIMS, C.c_ulonglong, P]),
}


class RefError(RuntimeError):
    def __init__(self, status, cls, msg):
        super().__init__(msg)
        self.status, self.cls = status, cls


def available() -> bool:
    return os.path.exists(LIB_PATH)


def load():
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"{LIB_PATH} not built (make -C oracle lib)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIG.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _lib = lib
    return _lib


def _call(name, *args):
    lib = load()
    st = getattr(lib, name)(*args)
    if st:
        raise RefError(st, lib.vref_last_error_class(), lib.vref_last_error().decode())


def _lib_call_status(name, *args):
    return getattr(load(), name)(*args)


def _error(st):
    lib = load()
    return RefError(st, lib.vref_last_error_class(), lib.vref_last_error().decode())


def _dims(shape):
    return (C.c_int * 3)(*shape[-3:])


def _a(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def set_workers(n: int):
    load().vref_set_workers(int(n))


# ---- operators (host numpy in / out) --------------------------------------------
def fft_forward(f):
    f = _a(f)
    n1, n2, n3 = f.shape
    out = np.empty((n1, n2, n3 // 2 + 1), dtype=np.complex128)
    _call("vref_fft_r2c", _dims(f.shape), f.ctypes.data, out.ctypes.data)
    return out


def fft_inverse(spec, shape):
    s = np.ascontiguousarray(spec, dtype=np.complex128)
    out = np.empty(shape)
    _call("vref_fft_c2r", _dims(shape), s.ctypes.data, out.ctypes.data)
    return out


def _unary(name, f, out_fields):
    f = _a(f)
    shape = f.shape[-3:]
    out = np.empty((out_fields,) + shape if out_fields > 1 else shape)
    _call(name, _dims(shape), f.ctypes.data, out.ctypes.data)
    return out


def gradient(f):
    return _unary("vref_gradient", f, 3)


def divergence(v):
    return _unary("vref_divergence", v, 1)


def laplacian(f):
    return _unary("vref_laplacian", f, 1)


def helmholtz1_apply(f):
    return _unary("vref_helmholtz1_apply", f, 1)


def gaussian_smooth(f, sigma):
    f = _a(f)
    out = np.empty_like(f)
    _call("vref_gaussian_smooth", _dims(f.shape), f.ctypes.data, out.ctypes.data,
          (C.c_double * 3)(*sigma))
    return out


def apply_reg_operator(v, norm, mode, beta=1.0):
    v = _a(v)
    out = np.empty_like(v)
    _call("vref_apply_reg_operator", _dims(v.shape), v.ctypes.data, out.ctypes.data, C.byref(norm),
          mode, beta)
    return out


def apply_projection(v, kind, beta_v=0.0, beta_w=0.0):
    v = _a(v)
    out = np.empty_like(v)
    _call("vref_apply_projection", _dims(v.shape), v.ctypes.data, out.ctypes.data, kind, beta_v, beta_w)
    return out


def rescale_intensity(f):
    f = _a(f)
    out = np.empty_like(f)
    deg = C.c_int()
    _call("vref_rescale_intensity", _dims(f.shape), f.ctypes.data, out.ctypes.data, C.byref(deg))
    return out, bool(deg.value)


def inner_product(a, b):
    a, b = _a(a), _a(b)
    r = C.c_double()
    _call("vref_inner_product", _dims(a.shape), a.ctypes.data, b.ctypes.data, 3 if a.ndim == 4 else 1,
          C.byref(r))
    return r.value


def dot_l2(a, b):
    a, b = _a(a), _a(b)
    r = C.c_double()
    _call("vref_dot_l2", _dims(a.shape), a.ctypes.data, b.ctypes.data, 3 if a.ndim == 4 else 1, C.byref(r))
    return r.value


def max_magnitude(v):
    v = _a(v)
    r = C.c_double()
    _call("vref_max_magnitude", _dims(v.shape), v.ctypes.data, C.byref(r))
    return r.value


def tricubic_interpolate(f, points):
    f, p = _a(f), _a(points)
    nf = 1 if f.ndim == 3 else f.shape[0]
    out = np.empty_like(f)
    _call("vref_tricubic_interpolate", _dims(p.shape), f.ctypes.data, p.ctypes.data, out.ctypes.data, nf)
    return out


def trace_characteristics(v, nt, direction="backward"):
    v = _a(v)
    out = np.empty_like(v)
    _call("vref_trace_characteristics", _dims(v.shape), v.ctypes.data, nt,
          0 if direction == "backward" else 1, out.ctypes.data)
    return out


def continuity_factor(div_v, departure, dt):
    d, p = _a(div_v), _a(departure)
    out = np.empty_like(d)
    _call("vref_continuity_factor", _dims(d.shape), d.ctypes.data, p.ctypes.data, dt, out.ctypes.data)
    return out


def solve_state(m_T, v, nt):
    m, v = _a(m_T), _a(v)
    out = np.empty((nt + 1,) + m.shape)
    _call("vref_solve_state", _dims(m.shape), m.ctypes.data, v.ctypes.data, nt, out.ctypes.data)
    return out


def solve_adjoint(terminal, v, nt, needs_history=False):
    t, v = _a(terminal), _a(v)
    init = np.empty_like(t)
    hist = np.empty((nt + 1,) + t.shape) if needs_history else None
    _call("vref_solve_adjoint", _dims(t.shape), t.ctypes.data, v.ctypes.data, nt,
          hist.ctypes.data if hist is not None else None, init.ctypes.data)
    return init, hist


def solve_inc_adjoint(terminal, v, nt, needs_history=False):
    t, v = _a(terminal), _a(v)
    init = np.empty_like(t)
    hist = np.empty((nt + 1,) + t.shape) if needs_history else None
    _call("vref_solve_inc_adjoint", _dims(t.shape), t.ctypes.data, v.ctypes.data, nt,
          hist.ctypes.data if hist is not None else None, init.ctypes.data)
    return init, hist


def gradient_dot(f, w):
    f, w = _a(f), _a(w)
    out = np.empty_like(f)
    _call("vref_gradient_dot", _dims(f.shape), f.ctypes.data, w.ctypes.data, out.ctypes.data)
    return out


def solve_inc_state(m_history, v, v_tilde, nt):
    m, v, vt = _a(m_history), _a(v), _a(v_tilde)
    out = np.empty((nt + 1,) + m.shape[-3:])
    _call("vref_solve_inc_state", _dims(m.shape), m.ctypes.data, v.ctypes.data, vt.ctypes.data, nt,
          m.shape[0], out.ctypes.data)
    return out


def generate_synthetic(shape, nt, amplitude=1.0):
    mR, mT = np.empty(shape), np.empty(shape)
    vs = np.empty((3,) + tuple(shape))
    _call("vref_generate_synthetic", _dims(shape), nt, amplitude, mR.ctypes.data, mT.ctypes.data,
          vs.ctypes.data)
    return mR, mT, vs


def random_smooth_scalar(shape, max_mode, seed, amplitude):
    out = np.empty(shape)
    _call("vref_random_smooth_scalar", _dims(shape), max_mode, seed, amplitude, out.ctypes.data)
    return out


def random_smooth_vector(shape, max_mode, seed, amplitude):
    out = np.empty((3,) + tuple(shape))
    _call("vref_random_smooth_vector", _dims(shape), max_mode, seed, amplitude, out.ctypes.data)
    return out


def random_rough_scalar(shape, seed):
    out = np.empty(shape)
    _call("vref_random_rough_scalar", _dims(shape), seed, out.ctypes.data)
    return out


# ---- objective ------------------------------------------------------------------
class State:
    def __init__(self, obj, h):
        self.obj, self._h = obj, h

    def scalars(self):
        J, mis, rel = C.c_double(), C.c_double(), C.c_double()
        hg, hc = C.c_int(), C.c_int()
        _call("vref_state_scalars", self._h, C.byref(J), C.byref(mis), C.byref(rel), C.byref(hg), C.byref(hc))
        return {"objective": J.value, "mismatch": mis.value, "mismatch_rel": rel.value,
                "has_gradient": bool(hg.value), "has_adjoint_ctx": bool(hc.value)}

    def get(self, which):
        nt = self.obj.model.nt
        nf = {0: 3, 1: 3, 2: 3, 3: 1, 4: nt + 1, 5: 3}[which]
        out = np.empty((nf,) + self.obj.shape if nf > 1 else self.obj.shape)
        _call("vref_state_get", self._h, which, out.ctypes.data)
        return out

    def __del__(self):
        if _lib is not None and getattr(self, "_h", None):
            _lib.vref_state_destroy(self._h)
            self._h = None


class Objective:
    def __init__(self, m_R, m_T, model):
        self.shape = tuple(np.shape(m_R))
        self.model = model
        r, t = _a(m_R), _a(m_T)
        h = C.c_void_p()
        _call("vref_objective_create", _dims(self.shape), r.ctypes.data, t.ctypes.data, C.byref(model), C.byref(h))
        self._h = h

    def initial_mismatch(self):
        r = C.c_double()
        _call("vref_objective_initial_mismatch", self._h, C.byref(r))
        return r.value

    def counters(self):
        c = Counters()
        _call("vref_objective_counters", self._h, C.byref(c))
        return {k: getattr(c, k) for k, _ in Counters._fields_}

    def evaluate(self, v):
        v = _a(v)
        h = C.c_void_p()
        _call("vref_evaluate", self._h, v.ctypes.data, C.byref(h))
        return State(self, h)

    def compute_gradient(self, s):
        g = np.empty((3,) + self.shape)
        _call("vref_compute_gradient", self._h, s._h, g.ctypes.data)
        return g

    def hessian_matvec(self, s, vt):
        vt = _a(vt)
        out = np.empty_like(vt)
        _call("vref_hessian_matvec", self._h, s._h, vt.ctypes.data, out.ctypes.data)
        return out

    def hessian_data_matvec(self, s, vt):
        vt = _a(vt)
        out = np.empty_like(vt)
        _call("vref_hessian_data_matvec", self._h, s._h, vt.ctypes.data, out.ctypes.data)
        return out

    def apply_reg(self, u, mode):
        u = _a(u)
        out = np.empty_like(u)
        _call("vref_objective_apply_reg", self._h, u.ctypes.data, mode, out.ctypes.data)
        return out

    def apply_K(self, u):
        u = _a(u)
        out = np.empty_like(u)
        _call("vref_objective_apply_K", self._h, u.ctypes.data, out.ctypes.data)
        return out

    def split_matvec(self, s, w):
        w = _a(w)
        out = np.empty_like(w)
        _call("vref_split_matvec", self._h, s._h, w.ctypes.data, out.ctypes.data)
        return out

    def pcg_solve(self, s, rhs, rel_tol, max_iter, precond=1):
        rhs = _a(rhs)
        x = np.empty_like(rhs)
        st = PcgStats()
        _call("vref_pcg_solve", self._h, s._h, rhs.ctypes.data, rel_tol, max_iter, precond, x.ctypes.data, C.byref(st))
        return x, {k: getattr(st, k) for k, _ in PcgStats._fields_}

    def __del__(self):
        if _lib is not None and getattr(self, "_h", None):
            _lib.vref_objective_destroy(self._h)
            self._h = None


def _report(r):
    d = {k: getattr(r, k) for k, _ in SolveReport._fields_ if k not in ("fine", "coarse")}
    for nm in ("fine", "coarse"):
        c = getattr(r, nm)
        d[nm] = {k: getattr(c, k) for k, _ in Counters._fields_}
    return d


def gauss_newton_solve(m_R, m_T, v0, model, params, precond=1, max_records=512):
    r, t, v0 = _a(m_R), _a(m_T), _a(v0)
    vout = np.empty_like(v0)
    rep = SolveReport()
    recs = (IterationRecord * max_records)()
    _call("vref_gauss_newton_solve", _dims(r.shape), r.ctypes.data, t.ctypes.data, v0.ctypes.data,
          C.byref(model), C.byref(params), precond, vout.ctypes.data, C.byref(rep), recs, max_records)
    n = min(rep.n_records, max_records)
    return vout, _report(rep), [{k: getattr(recs[i], k) for k, _ in IterationRecord._fields_} for i in range(n)]


def gauss_newton_solve_csv(m_R, m_T, v0, model, params):
    """The reference's SolveReport::write_csv (solver.cpp:29-47) of a spectral-precond solve."""
    r, t, v0 = _a(m_R), _a(m_T), _a(v0)
    buf = C.create_string_buffer(1 << 16)
    _call("vref_gauss_newton_solve_csv", _dims(r.shape), r.ctypes.data, t.ctypes.data, v0.ctypes.data,
          C.byref(model), C.byref(params), buf, len(buf))
    return buf.value.decode()


def parameter_continuation(m_R, m_T, v0, model, params, precond=1, max_levels=16, max_records=1024):
    r, t, v0 = _a(m_R), _a(m_T), _a(v0)
    vout = np.empty_like(v0)
    reps = (SolveReport * max_levels)()
    recs = (IterationRecord * max_records)()
    nl = C.c_int()
    _call("vref_parameter_continuation", _dims(r.shape), r.ctypes.data, t.ctypes.data, v0.ctypes.data,
          C.byref(model), C.byref(params), precond, vout.ctypes.data, reps, max_levels, C.byref(nl),
          recs, max_records)
    reports = [_report(reps[i]) for i in range(min(nl.value, max_levels))]
    n = min(sum(x["n_records"] for x in reports), max_records)
    return vout, reports, [{k: getattr(recs[i], k) for k, _ in IterationRecord._fields_} for i in range(n)]


def _level_call(fn, args, vshape, max_levels, max_records):
    vout = np.empty(vshape)
    reps = (SolveReport * max_levels)()
    recs = (IterationRecord * max_records)()
    nl = C.c_int()
    _call(fn, *args, vout.ctypes.data, reps, max_levels, C.byref(nl), recs, max_records)
    reports = [_report(reps[i]) for i in range(min(nl.value, max_levels))]
    n = min(sum(x["n_records"] for x in reports), max_records)
    return vout, reports, [{k: getattr(recs[i], k) for k, _ in IterationRecord._fields_} for i in range(n)]


def grid_continuation(m_R, m_T, v0, levels, model, params, precond=1, max_levels=16, max_records=1024):
    """Restated grid continuation over the reference's solver (ref_capi.cpp)."""
    r, t, v0 = _a(m_R), _a(m_T), _a(v0)
    return _level_call("vref_grid_continuation",
                       (_dims(r.shape), r.ctypes.data, t.ctypes.data, v0.ctypes.data, C.byref(model),
                        C.byref(params), precond, int(levels)), v0.shape, max_levels, max_records)


def scale_continuation(m_R, m_T, v0, sigmas, model, params, precond=1, max_levels=16, max_records=1024):
    r, t, v0 = _a(m_R), _a(m_T), _a(v0)
    sg = (C.c_double * len(sigmas))(*[float(x) for x in sigmas])
    return _level_call("vref_scale_continuation",
                       (_dims(r.shape), r.ctypes.data, t.ctypes.data, v0.ctypes.data, C.byref(model),
                        C.byref(params), precond, sg, len(sigmas)), v0.shape, max_levels, max_records)


def beta_search(m_R, m_T, v0, model, params, search, precond=1, max_trials=64):
    """Restated beta search (ref_capi.cpp); returns (beta, v, trials)."""
    r, t, v0 = _a(m_R), _a(m_T), _a(v0)
    vout = np.empty_like(v0)
    tr = np.zeros((max_trials, 5))
    reps = (SolveReport * max_trials)()
    n = C.c_int()
    beta = C.c_double()
    st = _lib_call_status("vref_beta_search", _dims(r.shape), r.ctypes.data, t.ctypes.data,
                          v0.ctypes.data, C.byref(model), C.byref(params), precond, C.byref(search),
                          C.byref(beta), vout.ctypes.data, tr.ctypes.data_as(C.POINTER(C.c_double)),
                          reps, max_trials, C.byref(n))
    trials = [{"beta": tr[i, 0], "feasible": bool(tr[i, 1]), "det_min": tr[i, 2], "det_mean": tr[i, 3],
               "det_max": tr[i, 4], "report": _report(reps[i])} for i in range(min(n.value, max_trials))]
    if st != 0:
        e = _error(st)
        e.trials = trials
        raise e
    return beta.value, vout, trials


# ---- fp32 lane: the reference's float instantiations ----------------------------------
def _f(x):
    return np.ascontiguousarray(x, dtype=np.float32)


def tricubic_interpolate_f32(f, points):
    f, p = _f(f), _f(points)
    nf = 1 if f.ndim == 3 else f.shape[0]
    out = np.empty_like(f)
    _call("vref_tricubic_interpolate_f32", _dims(p.shape), f.ctypes.data, p.ctypes.data, out.ctypes.data, nf)
    return out


def trace_characteristics_f32(v, nt, direction="backward"):
    v = _f(v)
    out = np.empty_like(v)
    _call("vref_trace_characteristics_f32", _dims(v.shape), v.ctypes.data, nt,
          0 if direction == "backward" else 1, out.ctypes.data)
    return out


def _f32_unary(name, a, nout, *extra):
    a = _f(a)
    shape = a.shape if a.ndim == 3 else a.shape[1:]
    out = np.empty(((nout,) if nout > 1 else ()) + tuple(shape), dtype=np.float32)
    _call(name, _dims(shape), a.ctypes.data, out.ctypes.data, *extra)
    return out


def gradient_f32(f):
    return _f32_unary("vref_gradient_f32", f, 3)


def divergence_f32(v):
    return _f32_unary("vref_divergence_f32", v, 1)


def apply_reg_operator_f32(v, norm, mode, beta=1.0):
    return _f32_unary("vref_apply_reg_operator_f32", v, 3, C.byref(norm), mode, beta)


def apply_projection_f32(v, kind, beta_v=0.0, beta_w=0.0):
    return _f32_unary("vref_apply_projection_f32", v, 3, kind, beta_v, beta_w)


def gaussian_smooth_f32(f, sigma):
    return _f32_unary("vref_gaussian_smooth_f32", f, 1, (C.c_double * 3)(*sigma))


def fft_forward_f32(f):
    f = _f(f)
    out = np.empty((f.shape[0], f.shape[1], f.shape[2] // 2 + 1), dtype=np.complex128)
    _call("vref_fft_r2c_f32", _dims(f.shape), f.ctypes.data, out.ctypes.data)
    return out


def fft_inverse_f32(spec, shape):
    s = np.ascontiguousarray(spec, dtype=np.complex128)
    out = np.empty(shape, dtype=np.float32)
    _call("vref_fft_c2r_f32", _dims(shape), s.ctypes.data, out.ctypes.data)
    return out


class ObjectiveF32:
    """The reference's Objective<float> on host float32 arrays."""

    def __init__(self, m_R, m_T, model):
        self.shape = tuple(np.shape(m_R))
        self.model = model
        self._r, self._t = _f(m_R), _f(m_T)
        h = C.c_void_p()
        _call("vref_objective_f32_create", _dims(self.shape), self._r.ctypes.data, self._t.ctypes.data,
              C.byref(model), C.byref(h))
        self._h = h

    def evaluate(self, v):
        v = _f(v)
        h = C.c_void_p()
        _call("vref_evaluate_f32", self._h, v.ctypes.data, C.byref(h))
        return StateF32(h)

    def compute_gradient(self, s):
        g = np.empty((3,) + self.shape, dtype=np.float32)
        _call("vref_compute_gradient_f32", self._h, s._h, g.ctypes.data)
        return g

    def hessian_matvec(self, s, vt):
        vt = _f(vt)
        out = np.empty_like(vt)
        _call("vref_hessian_matvec_f32", self._h, s._h, vt.ctypes.data, out.ctypes.data)
        return out

    def counters(self):
        c = Counters()
        _call("vref_objective_f32_counters", self._h, C.byref(c))
        return {k: getattr(c, k) for k, _ in Counters._fields_}

    def __del__(self):
        try:
            load().vref_objective_f32_destroy(self._h)
        except Exception:
            pass


class StateF32:
    def __init__(self, h):
        self._h = h

    def scalars(self):
        J, mis, rel = C.c_double(), C.c_double(), C.c_double()
        _call("vref_state_f32_scalars", self._h, C.byref(J), C.byref(mis), C.byref(rel))
        return {"objective": J.value, "mismatch": mis.value, "mismatch_rel": rel.value}

    def __del__(self):
        try:
            load().vref_state_f32_destroy(self._h)
        except Exception:
            pass


def gauss_newton_solve_f32(m_R, m_T, v0, model, params, precond=1, max_records=512):
    r, t, v0 = _f(m_R), _f(m_T), _f(v0)
    vout = np.empty_like(v0)
    rep = SolveReport()
    recs = (IterationRecord * max_records)()
    _call("vref_gauss_newton_solve_f32", _dims(r.shape), r.ctypes.data, t.ctypes.data, v0.ctypes.data,
          C.byref(model), C.byref(params), precond, vout.ctypes.data, C.byref(rep), recs, max_records)
    n = min(rep.n_records, max_records)
    return vout, _report(rep), [{k: getattr(recs[i], k) for k, _ in IterationRecord._fields_} for i in range(n)]


def gauss_newton_solve_two_level_f32(m_R, m_T, v0, model, params, options, max_records=512):
    """gauss_newton_solve<float> with TwoLevelPreconditioner<float> (precond.cpp:153-249)."""
    r, t, v0 = _f(m_R), _f(m_T), _f(v0)
    vout = np.empty_like(v0)
    rep = SolveReport()
    recs = (IterationRecord * max_records)()
    _call("vref_gauss_newton_solve_two_level_f32", _dims(r.shape), r.ctypes.data, t.ctypes.data,
          v0.ctypes.data, C.byref(model), C.byref(params), C.byref(options), vout.ctypes.data,
          C.byref(rep), recs, max_records)
    n = min(rep.n_records, max_records)
    return vout, _report(rep), [{k: getattr(recs[i], k) for k, _ in IterationRecord._fields_} for i in range(n)]


def parameter_continuation_f32(m_R, m_T, v0, model, params, precond=1, max_levels=16, max_records=1024):
    r, t, v0 = _f(m_R), _f(m_T), _f(v0)
    vout = np.empty_like(v0)
    reps = (SolveReport * max_levels)()
    recs = (IterationRecord * max_records)()
    nl = C.c_int()
    _call("vref_parameter_continuation_f32", _dims(r.shape), r.ctypes.data, t.ctypes.data, v0.ctypes.data,
          C.byref(model), C.byref(params), precond, vout.ctypes.data, reps, max_levels, C.byref(nl),
          recs, max_records)
    reports = [_report(reps[i]) for i in range(min(nl.value, max_levels))]
    return vout, reports


def solve_state_f32(m_T, v, nt):
    m, v = _f(m_T), _f(v)
    out = np.empty((nt + 1,) + m.shape, dtype=np.float32)
    _call("vref_solve_state_f32", _dims(m.shape), m.ctypes.data, v.ctypes.data, nt, out.ctypes.data)
    return out


# ---- postprocess (postprocess.hpp:9-56) ----------------------------------------------
def det_deformation_gradient(v, nt):
    v = _a(v)
    out = np.empty(v.shape[1:])
    _call("vref_det_deformation_gradient", _dims(v.shape[1:]), v.ctypes.data, nt, out.ctypes.data)
    return out


def deformation_map(v, nt, absolute=False):
    v = _a(v)
    out = np.empty_like(v)
    _call("vref_deformation_map", _dims(v.shape[1:]), v.ctypes.data, nt, 1 if absolute else 0,
          out.ctypes.data)
    return out


def det_stats(det, foreground=None, threshold=0.05):
    d = _a(det)
    fg = _a(foreground) if foreground is not None else None
    out = (C.c_double * 3)()
    _call("vref_det_stats", _dims(d.shape), d.ctypes.data, fg.ctypes.data if fg is not None else None,
          float(threshold), out)
    return {"min": out[0], "mean": out[1], "max": out[2]}


def make_ball_labels(shape, count):
    out = np.empty(shape)
    _call("vref_make_ball_labels", _dims(shape), count, out.ctypes.data)
    return out


def transport_labels(labels, v, nt):
    lab, v = _a(labels), _a(v)
    out = np.empty_like(lab)
    _call("vref_transport_labels", _dims(lab.shape), lab.ctypes.data, v.ctypes.data, nt, out.ctypes.data)
    return out


def overlap_scores(reference, test, mask=None, max_labels=4096):
    a, b = _a(reference), _a(test)
    m = _a(mask) if mask is not None else None
    n = C.c_int()
    codes = (C.c_int * max_labels)()
    per = np.zeros((max_labels, 3))
    uni = (C.c_double * 3)()
    _call("vref_overlap_scores", _dims(a.shape), a.ctypes.data, b.ctypes.data,
          m.ctypes.data if m is not None else None, max_labels, C.byref(n), codes,
          per.ctypes.data_as(C.POINTER(C.c_double)), uni)
    k = min(n.value, max_labels)
    ov = lambda x: {"dice": x[0], "false_positive_rate": x[1], "false_negative_rate": x[2]}  # noqa: E731
    return {"per_label": {codes[i]: ov(per[i]) for i in range(k)}, "union": ov(uni), "n_labels": n.value}


# ---- two-level preconditioner / grid transfer (precond.hpp, spectral.hpp:131-153) ------
def spectral_resample(f, shape):
    f = _a(f)
    nc = 3 if f.ndim == 4 else 1
    out = np.empty(((3,) if nc == 3 else ()) + tuple(shape))
    _call("vref_spectral_resample", _dims(f.shape), f.ctypes.data, nc, _dims(shape), out.ctypes.data)
    return out


def frequency_filter(f, band, cutoff):
    f = _a(f)
    nc = 3 if f.ndim == 4 else 1
    out = np.empty_like(f)
    b = {"low": 0, "high": 1}.get(band, band)
    cut = (cutoff,) * 3 if isinstance(cutoff, int) else tuple(cutoff)
    _call("vref_frequency_filter", _dims(f.shape), f.ctypes.data, nc, b, _dims(cut), out.ctypes.data)
    return out


class TwoLevelPreconditioner:
    """TwoLevelPreconditioner<double> of the compiled reference (precond.hpp:93-110)."""

    def __init__(self, options):
        h = C.c_void_p()
        _call("vref_twolevel_create", C.byref(options), C.byref(h))
        self._h = h
        self.shape = None

    def rebuild(self, obj, state, eps_H):
        self.shape = obj.shape
        _call("vref_twolevel_rebuild", self._h, obj._h, state._h, eps_H)

    def apply(self, r):
        r = _a(r)
        z = np.empty_like(r)
        _call("vref_twolevel_apply", self._h, r.ctypes.data, z.ctypes.data)
        return z

    def coarse_matvec(self, u):
        u = _a(u)
        out = np.empty_like(u)
        _call("vref_twolevel_coarse_matvec", self._h, u.ctypes.data, out.ctypes.data)
        return out

    def info(self):
        dims = (C.c_int * 3)()
        runs, div = C.c_int(), C.c_int()
        b = (C.c_double * 2)()
        c = Counters()
        _call("vref_twolevel_info", self._h, dims, C.byref(runs), C.byref(div), b, C.byref(c))
        return {"coarse_dims": tuple(dims), "lanczos_runs": runs.value,
                "inner_diverged": bool(div.value), "bounds": (b[0], b[1]),
                "coarse": {k: getattr(c, k) for k, _ in Counters._fields_}}

    def __del__(self):
        if _lib is not None and getattr(self, "_h", None):
            _lib.vref_twolevel_destroy(self._h)
            self._h = None


def gauss_newton_solve_two_level(m_R, m_T, v0, model, params, options, max_records=512):
    r, t, v0 = _a(m_R), _a(m_T), _a(v0)
    vout = np.empty_like(v0)
    rep = SolveReport()
    recs = (IterationRecord * max_records)()
    _call("vref_gauss_newton_solve_two_level", _dims(r.shape), r.ctypes.data, t.ctypes.data,
          v0.ctypes.data, C.byref(model), C.byref(params), C.byref(options), vout.ctypes.data,
          C.byref(rep), recs, max_records)
    n = min(rep.n_records, max_records)
    return vout, _report(rep), [{k: getattr(recs[i], k) for k, _ in IterationRecord._fields_} for i in range(n)]
