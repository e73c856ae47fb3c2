"""Python mirror of the reference's operator API, running on the sm_100a C ABI.

Names, argument meaning and error behaviour follow the reference veloreg C++
API (/root/reference/proj/include/veloreg/*.hpp) so parity tests read like the
reference's own tests:

* spectral.hpp  -> gradient, divergence, laplacian, helmholtz1_apply,
  gaussian_smooth, apply_reg_operator, apply_projection, inner_product,
  rescale_intensity
* interp.hpp / transport.hpp -> tricubic_interpolate, trace_characteristics,
  continuity_factor, solve_state, solve_adjoint, gradient_dot, solve_inc_state,
  solve_inc_adjoint
* objective.hpp -> Objective (evaluate / compute_gradient / hessian_matvec /
  hessian_data_matvec / apply_reg / apply_K / counters / initial_mismatch)
* solver.hpp -> compute_forcing, pcg_solve, gauss_newton_solve, plus
  parameter_continuation

Every call goes through libveloreg_gpu.so; host numpy arrays are copied to the
device and back. Shapes: scalar (n1,n2,n3), vector (3,n1,n2,n3), time series
(nt+1,n1,n2,n3); all float64, C-contiguous (the reference's layout).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi_types, _lib
from ._lib import (ArgumentError, DimensionError, LogicError, NumericError,  # noqa: F401
                   ResourceError, VelouregError)

_lib.load()  # no CPU fallback: importing the mirror without the built library raises

_KIND = {"h1": _lib.REG_H1, "h2": _lib.REG_H2, "h3": _lib.REG_H3, "helmholtz": _lib.REG_HELMHOLTZ}
_PROJ = {"identity": _lib.PROJ_IDENTITY, "incompressible": _lib.PROJ_INCOMPRESSIBLE,
         "near_incompressible": _lib.PROJ_NEAR_INCOMPRESSIBLE}
_MODE = {"apply": _lib.REGOP_APPLY, "inverse": _lib.REGOP_INVERSE,
         "inverse_sqrt": _lib.REGOP_INVERSE_SQRT}


def _enum(table, v):
    return table[v] if isinstance(v, str) else int(v)


make_norm = _abi_types.make_norm
make_model = _abi_types.make_model


def make_params(**kw):
    """SolverParams (solver.hpp:13-33) with keyword overrides."""
    p = _lib.SolverParams()
    _lib.load().vr_solver_params_default(C.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise ArgumentError(f"SolverParams has no field {k}")
        setattr(p, k, int(v) if isinstance(getattr(p, k), int) else v)
    return p


# ---------------------------------------------------------------------------
class Context:
    """One grid on one device with its own CUDA stream (vr_ctx)."""

    def __init__(self, dims, device: int = 0):
        if isinstance(dims, int):
            dims = (dims, dims, dims)
        self.dims = tuple(int(d) for d in dims)
        self.local_dims = self.dims  # shape of this context's fields (a slab on x1 slabs)
        self.N = self.dims[0] * self.dims[1] * self.dims[2]
        self.nh = self.dims[2] // 2 + 1
        h = C.c_void_p()
        _lib.call("vr_ctx_create", self.dims[0], self.dims[1], self.dims[2], device, C.byref(h))
        self._h = h

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return _lib.load().vr_ctx_stream(self._h) or 0

    def synchronize(self):
        _lib.call("vr_ctx_synchronize", self._h)

    def kernel_launches(self) -> int:
        return int(_lib.load().vr_ctx_kernel_launches(self._h))

    def reset_kernel_launches(self):
        _lib.load().vr_ctx_reset_kernel_launches(self._h)

    def set_profiling(self, on: bool):
        _lib.call("vr_ctx_set_profiling", self._h, int(bool(on)))

    def profile_read(self) -> dict:
        """{category: (launches, total_ms)} since profiling was enabled / last read."""
        buf = C.create_string_buffer(1 << 16)
        _lib.call("vr_ctx_profile_read", self._h, buf, len(buf))
        out = {}
        for line in buf.value.decode().splitlines():
            cat, n, ms = line.split(",")
            out[cat] = (int(n), float(ms))
        return out

    def close(self):
        if getattr(self, "_h", None):
            _lib.call("vr_ctx_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def memory(self) -> dict:
        """Library device allocations of this context (vr_ctx_memory): live and peak bytes
        (the reference's FieldAllocStats), plus the device pool's reserved high-water mark."""
        a, b, c = C.c_longlong(), C.c_longlong(), C.c_longlong()
        _lib.call("vr_ctx_memory", self._h, C.byref(a), C.byref(b), C.byref(c))
        return {"live_bytes": a.value, "peak_bytes": b.value, "pool_reserved_high_bytes": c.value}

    def reset_memory_peak(self):
        _lib.call("vr_ctx_reset_memory_peak", self._h)

    # ---- device arrays
    def empty(self, nfields: int, complex_spectrum: bool = False) -> "DeviceArray":
        return DeviceArray(self, nfields, complex_spectrum)

    def to_device(self, arr) -> "DeviceArray":
        if isinstance(arr, DeviceArray):
            return arr
        a = np.ascontiguousarray(arr, dtype=np.float64)
        nf = a.size // self.N
        if nf * self.N != a.size:
            raise DimensionError(f"array of size {a.size} is not a whole number of {self.dims} fields")
        d = DeviceArray(self, nf)
        _lib.call("vr_memcpy_h2d", self._h, d.ptr, a.ctypes.data, a.nbytes)
        return d


class DeviceArray:
    """`nfields` consecutive fp64 fields (or spectra) in HBM."""

    def __init__(self, ctx: Context, nfields: int, complex_spectrum: bool = False):
        self.ctx = ctx
        self.nfields = nfields
        self.spectrum = complex_spectrum
        ld = ctx.local_dims
        per = ld[0] * ld[1] * ctx.nh * 2 if complex_spectrum else ctx.N
        self.count = per * nfields
        self.nbytes = 8 * self.count
        p = C.c_void_p()
        _lib.call("vr_device_alloc", ctx.handle, max(self.nbytes, 8), C.byref(p))
        self.ptr = p
        _lib.call("vr_memset_zero", ctx.handle, p, max(self.nbytes, 8))

    def numpy(self) -> np.ndarray:
        out = np.empty(self.count, dtype=np.float64)
        _lib.call("vr_memcpy_d2h", self.ctx.handle, out.ctypes.data, self.ptr, self.nbytes)
        d = self.ctx.local_dims
        if self.spectrum:
            c = out.view(np.complex128)
            return c.reshape((self.nfields, d[0], d[1], self.ctx.nh)) if self.nfields > 1 else c.reshape(d[0], d[1], self.ctx.nh)
        return out.reshape((self.nfields,) + d) if self.nfields > 1 else out.reshape(d)

    def upload(self, arr):
        a = np.ascontiguousarray(arr, dtype=np.complex128 if self.spectrum else np.float64)
        if a.nbytes != self.nbytes:
            raise DimensionError("upload: size mismatch")
        _lib.call("vr_memcpy_h2d", self.ctx.handle, self.ptr, a.ctypes.data, a.nbytes)

    def field(self, i: int) -> C.c_void_p:
        per = self.count // self.nfields
        return C.c_void_p(self.ptr.value + 8 * per * i)

    def free(self):
        if getattr(self, "ptr", None) is not None and self.ctx._h:
            _lib.call("vr_device_free", self.ctx.handle, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _dev(ctx, a, nfields: Optional[int] = None):
    """Device view of `a` (host arrays are uploaded). With `nfields`, the argument must hold
    exactly that many real fields of this context's grid: the C ABI takes bare pointers and
    would otherwise read or write past a short buffer (DimensionError before any call)."""
    if isinstance(a, DeviceArray):
        if nfields is not None and (a.nfields != nfields or a.spectrum or a.ctx.N != ctx.N):
            raise DimensionError(f"expected a device array of {nfields} real field(s) of {ctx.local_dims}, got "
                                 f"{a.nfields} {'spectra' if a.spectrum else 'field(s)'} of {a.ctx.local_dims}")
        return a
    if nfields is not None and np.size(a) != nfields * ctx.N:
        raise DimensionError(f"expected {nfields} field(s) of {ctx.local_dims} ({nfields * ctx.N} values), "
                             f"got an array of shape {np.shape(a)}")
    return ctx.to_device(a)


def _host_buf(ctx, a, nfields: int, name: str, writeable: bool = False):
    """Host buffer for the *_host entry points: float64, C-contiguous, exactly nfields*N
    values (the C side copies nfields*N*8 bytes from / to the raw pointer)."""
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
        raise DimensionError(f"{name}: need a C-contiguous float64 numpy array")
    if a.size != nfields * ctx.N:
        raise DimensionError(f"{name}: need {nfields * ctx.N} values ({nfields} field(s) of {ctx.local_dims}), "
                             f"got {a.size}")
    if writeable and not a.flags.writeable:
        raise DimensionError(f"{name}: output array is read-only")
    return a.ctypes.data


def _ret(out: DeviceArray, host: bool):
    return out.numpy() if host else out


def _is_host(*arrs):
    return any(not isinstance(a, DeviceArray) for a in arrs)


# ---- BLAS-1 / quadrature (field_ops.hpp, spectral.cpp:47-62) ------------------
def inner_product(ctx, a, b) -> float:
    da = _dev(ctx, a)
    db = _dev(ctx, b, da.nfields)
    r = C.c_double()
    _lib.call("vr_inner_product", ctx.handle, da.ptr, db.ptr, da.nfields, C.byref(r))
    return r.value


def dot_l2(ctx, a, b) -> float:
    da = _dev(ctx, a)
    db = _dev(ctx, b, da.nfields)
    r = C.c_double()
    _lib.call("vr_dot_l2", ctx.handle, da.ptr, db.ptr, da.nfields, C.byref(r))
    return r.value


def norm_l2(ctx, a) -> float:
    return float(np.sqrt(dot_l2(ctx, a, a)))


def max_abs(ctx, a) -> float:
    da = _dev(ctx, a)
    r = C.c_double()
    _lib.call("vr_max_abs", ctx.handle, da.ptr, da.nfields, C.byref(r))
    return r.value


def max_magnitude(ctx, v) -> float:
    dv = _dev(ctx, v, 3)
    r = C.c_double()
    _lib.call("vr_max_magnitude", ctx.handle, dv.ptr, C.byref(r))
    return r.value


# ---- spectral ----------------------------------------------------------------
def fft_forward(ctx, f):
    """fft_forward_raw (fft.cpp:66-73): unnormalized half spectrum (n1, n2, n3/2+1)."""
    df = _dev(ctx, f, 1)
    out = ctx.empty(1, complex_spectrum=True)
    _lib.call("vr_fft_r2c", ctx.handle, df.ptr, out.ptr)
    return _ret(out, _is_host(f))


def fft_inverse(ctx, spec):
    """fft_inverse_raw (fft.cpp:75-83), includes the 1/N scale."""
    if isinstance(spec, DeviceArray):
        ds = spec
    else:
        ds = ctx.empty(1, complex_spectrum=True)
        ds.upload(spec)
    out = ctx.empty(1)
    _lib.call("vr_fft_c2r", ctx.handle, ds.ptr, out.ptr)
    return _ret(out, _is_host(spec))


def gradient(ctx, f):
    df = _dev(ctx, f, 1)
    out = ctx.empty(3)
    _lib.call("vr_gradient", ctx.handle, df.ptr, out.ptr)
    return _ret(out, _is_host(f))


def divergence(ctx, v):
    dv = _dev(ctx, v, 3)
    out = ctx.empty(1)
    _lib.call("vr_divergence", ctx.handle, dv.ptr, out.ptr)
    return _ret(out, _is_host(v))


def laplacian(ctx, f):
    df = _dev(ctx, f)
    out = ctx.empty(df.nfields)
    _lib.call("vr_laplacian", ctx.handle, df.ptr, out.ptr, df.nfields)
    return _ret(out, _is_host(f))


def helmholtz1_apply(ctx, f):
    df = _dev(ctx, f, 1)
    out = ctx.empty(1)
    _lib.call("vr_helmholtz1_apply", ctx.handle, df.ptr, out.ptr)
    return _ret(out, _is_host(f))


def gaussian_smooth(ctx, f, sigma_voxels: Sequence[float]):
    df = _dev(ctx, f)
    out = ctx.empty(df.nfields)
    sig = (C.c_double * 3)(*[float(s) for s in sigma_voxels])
    _lib.call("vr_gaussian_smooth", ctx.handle, df.ptr, out.ptr, df.nfields, sig)
    return _ret(out, _is_host(f))


def apply_reg_operator(ctx, v, norm=None, mode="apply", beta=1.0):
    dv = _dev(ctx, v, 3)
    out = ctx.empty(3)
    norm = norm if norm is not None else make_norm()
    _lib.call("vr_apply_reg_operator", ctx.handle, dv.ptr, out.ptr, C.byref(norm),
              _enum(_MODE, mode), beta)
    return _ret(out, _is_host(v))


def apply_projection(ctx, v, kind="incompressible", beta_v=0.0, beta_w=0.0):
    dv = _dev(ctx, v, 3)
    out = ctx.empty(3)
    _lib.call("vr_apply_projection", ctx.handle, dv.ptr, out.ptr, _enum(_PROJ, kind), beta_v, beta_w)
    return _ret(out, _is_host(v))


def rescale_intensity(ctx, f):
    df = _dev(ctx, f, 1)
    out = ctx.empty(1)
    deg = C.c_int()
    _lib.call("vr_rescale_intensity", ctx.handle, df.ptr, out.ptr, C.byref(deg))
    return _ret(out, _is_host(f)), bool(deg.value)


# ---- transport -------------------------------------------------------------------
def tricubic_interpolate(ctx, f, points):
    df, dp = _dev(ctx, f), _dev(ctx, points, 3)
    if df.nfields not in (1, 2, 3):
        raise DimensionError(f"tricubic_interpolate: 1, 2 or 3 fields, got {df.nfields}")
    out = ctx.empty(df.nfields)
    _lib.call("vr_tricubic_interpolate", ctx.handle, df.ptr, dp.ptr, out.ptr, df.nfields)
    return _ret(out, _is_host(f, points))


def trace_characteristics(ctx, v, nt, direction="backward"):
    dv = _dev(ctx, v, 3)
    out = ctx.empty(3)
    d = _lib.TRACE_BACKWARD if direction == "backward" else _lib.TRACE_FORWARD
    _lib.call("vr_trace_characteristics", ctx.handle, dv.ptr, nt, d, out.ptr)
    return _ret(out, _is_host(v))


def continuity_factor(ctx, div_v, departure, dt):
    dd, dp = _dev(ctx, div_v, 1), _dev(ctx, departure, 3)
    out = ctx.empty(1)
    _lib.call("vr_continuity_factor", ctx.handle, dd.ptr, dp.ptr, dt, out.ptr)
    return _ret(out, _is_host(div_v, departure))


def solve_state(ctx, m_T, v, nt):
    dm, dv = _dev(ctx, m_T, 1), _dev(ctx, v, 3)
    out = ctx.empty(nt + 1)
    _lib.call("vr_solve_state", ctx.handle, dm.ptr, dv.ptr, nt, out.ptr)
    return _ret(out, _is_host(m_T, v))


def solve_adjoint(ctx, terminal, v, nt, needs_history=False):
    dt_, dv = _dev(ctx, terminal, 1), _dev(ctx, v, 3)
    init = ctx.empty(1)
    hist = ctx.empty(nt + 1) if needs_history else None
    _lib.call("vr_solve_adjoint", ctx.handle, dt_.ptr, dv.ptr, nt, hist.ptr if hist else None, init.ptr)
    host = _is_host(terminal, v)
    return _ret(init, host), (_ret(hist, host) if hist else None)


def solve_inc_adjoint(ctx, terminal, v, nt, needs_history=False):
    dt_, dv = _dev(ctx, terminal, 1), _dev(ctx, v, 3)
    init = ctx.empty(1)
    hist = ctx.empty(nt + 1) if needs_history else None
    _lib.call("vr_solve_inc_adjoint", ctx.handle, dt_.ptr, dv.ptr, nt, hist.ptr if hist else None, init.ptr)
    host = _is_host(terminal, v)
    return _ret(init, host), (_ret(hist, host) if hist else None)


def gradient_dot(ctx, f, w):
    df, dw = _dev(ctx, f, 1), _dev(ctx, w, 3)
    out = ctx.empty(1)
    _lib.call("vr_gradient_dot", ctx.handle, df.ptr, dw.ptr, out.ptr)
    return _ret(out, _is_host(f, w))


def solve_inc_state(ctx, m_history, v, v_tilde, nt):
    dm, dv, dvt = _dev(ctx, m_history, nt + 1), _dev(ctx, v, 3), _dev(ctx, v_tilde, 3)
    out = ctx.empty(nt + 1)
    _lib.call("vr_solve_inc_state", ctx.handle, dm.ptr, dv.ptr, dvt.ptr, nt, out.ptr)
    return _ret(out, _is_host(m_history, v, v_tilde))


def generate_synthetic(ctx, nt, amplitude=1.0, host=True):
    """generate_synthetic (synthetic.cpp:16-34) on the device: (m_R, m_T, v_star)."""
    mR, mT, vs = ctx.empty(1), ctx.empty(1), ctx.empty(3)
    _lib.call("vr_generate_synthetic", ctx.handle, nt, amplitude, mR.ptr, mT.ptr, vs.ptr)
    return (mR.numpy(), mT.numpy(), vs.numpy()) if host else (mR, mT, vs)


# ---- objective -----------------------------------------------------------------
class EvalState:
    """EvalState<T> (objective.hpp:37-54); device resident."""

    def __init__(self, obj: "Objective", handle):
        self.obj = obj
        self._h = handle

    def _scalars(self):
        J, mis, rel = C.c_double(), C.c_double(), C.c_double()
        hg, hc = C.c_int(), C.c_int()
        _lib.call("vr_state_scalars", self._h, C.byref(J), C.byref(mis), C.byref(rel), C.byref(hg), C.byref(hc))
        return J.value, mis.value, rel.value, bool(hg.value), bool(hc.value)

    objective = property(lambda s: s._scalars()[0])
    mismatch = property(lambda s: s._scalars()[1])
    mismatch_rel = property(lambda s: s._scalars()[2])
    has_gradient = property(lambda s: s._scalars()[3])
    has_adjoint_ctx = property(lambda s: s._scalars()[4])

    def get(self, which: int, host=True):
        ctx = self.obj.ctx
        nt = self.obj.model.nt
        nf = {_lib.STATE_V: 3, _lib.STATE_X_BWD: 3, _lib.STATE_X_FWD: 3, _lib.STATE_FACTOR: 1,
              _lib.STATE_M_HISTORY: nt + 1, _lib.STATE_GRADIENT: 3,
              _lib.STATE_GRAD_M: 3 * (nt + 1), _lib.STATE_LAMBDA_HISTORY: nt + 1}[which]
        out = ctx.empty(nf)
        _lib.call("vr_state_get", self._h, which, out.ptr)
        return out.numpy() if host else out

    @property
    def gradient(self):
        return self.get(_lib.STATE_GRADIENT)

    @property
    def m_history(self):
        return self.get(_lib.STATE_M_HISTORY)

    def close(self):
        # the C state points at its objective and context: only destroy it while both live
        if getattr(self, "_h", None):
            if getattr(self.obj, "_h", None) and getattr(self.obj.ctx, "_h", None):
                _lib.call("vr_state_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Objective:
    """Objective<double> (objective.hpp:56-102) over device-resident images."""

    def __init__(self, ctx: Context, m_R, m_T, model=None):
        self.ctx = ctx
        self.model = model if model is not None else make_model()
        self._mR = _dev(ctx, m_R, 1)  # kept alive: the C object holds non-owning pointers
        self._mT = _dev(ctx, m_T, 1)
        h = C.c_void_p()
        _lib.call("vr_objective_create", ctx.handle, self._mR.ptr, self._mT.ptr, C.byref(self.model), C.byref(h))
        self._h = h

    @property
    def handle(self):
        return self._h

    def initial_mismatch(self) -> float:
        r = C.c_double()
        _lib.call("vr_objective_initial_mismatch", self._h, C.byref(r))
        return r.value

    def counters(self) -> dict:
        c = _lib.Counters()
        _lib.call("vr_objective_counters", self._h, C.byref(c))
        return {k: getattr(c, k) for k, _ in _lib.Counters._fields_}

    def evaluate(self, v) -> EvalState:
        dv = _dev(self.ctx, v, 3)
        h = C.c_void_p()
        _lib.call("vr_evaluate", self._h, dv.ptr, C.byref(h))
        return EvalState(self, h)

    def compute_gradient(self, state: EvalState):
        _lib.call("vr_compute_gradient", self._h, state._h, None)

    def hessian_matvec(self, state: EvalState, v_tilde, out: Optional[DeviceArray] = None):
        dv = _dev(self.ctx, v_tilde, 3)
        o = _dev(self.ctx, out, 3) if out is not None else self.ctx.empty(3)
        _lib.call("vr_hessian_matvec", self._h, state._h, dv.ptr, o.ptr)
        return _ret(o, _is_host(v_tilde) and out is None)

    def split_matvec(self, state: EvalState, w):
        """Objective::split_matvec (objective.cpp:158-176): (I + R H_data R) w, R = (beta_v A)^-1/2."""
        dw = _dev(self.ctx, w, 3)
        o = self.ctx.empty(3)
        _lib.call("vr_split_matvec", self._h, state._h, dw.ptr, o.ptr)
        return _ret(o, _is_host(w))

    def hessian_data_matvec(self, state: EvalState, v_tilde):
        dv = _dev(self.ctx, v_tilde, 3)
        o = self.ctx.empty(3)
        _lib.call("vr_hessian_data_matvec", self._h, state._h, dv.ptr, o.ptr)
        return _ret(o, _is_host(v_tilde))

    def hessian_matvec_host(self, state: EvalState, vt_host: np.ndarray, out_host: np.ndarray):
        """End-to-end entry: host buffers in/out (H2D + matvec + D2H)."""
        _lib.call("vr_hessian_matvec_host", self._h, state._h, _host_buf(self.ctx, vt_host, 3, "vt_host"),
                  _host_buf(self.ctx, out_host, 3, "out_host", writeable=True))
        return out_host

    def hessian_matvec_host_async(self, state: EvalState, vt_host: np.ndarray, out_host: np.ndarray):
        """Pipelined host-buffer matvec (vr_hessian_matvec_host_async); results are valid
        after wait(). Keep both arrays alive and vt_host unchanged until then."""
        _lib.call("vr_hessian_matvec_host_async", self._h, state._h, _host_buf(self.ctx, vt_host, 3, "vt_host"),
                  _host_buf(self.ctx, out_host, 3, "out_host", writeable=True))
        return out_host

    def wait(self):
        _lib.call("vr_objective_wait", self._h)

    def apply_reg(self, u, mode="apply"):
        du = _dev(self.ctx, u, 3)
        o = self.ctx.empty(3)
        _lib.call("vr_objective_apply_reg", self._h, du.ptr, _enum(_MODE, mode), o.ptr)
        return _ret(o, _is_host(u))

    def apply_K(self, u):
        du = _dev(self.ctx, u, 3)
        o = self.ctx.empty(3)
        _lib.call("vr_objective_apply_K", self._h, du.ptr, o.ptr)
        return _ret(o, _is_host(u))

    def close(self):
        if getattr(self, "_h", None):
            if getattr(self.ctx, "_h", None):
                _lib.call("vr_objective_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- solvers --------------------------------------------------------------------
def compute_forcing(grad_norm, grad0_norm) -> float:
    r = C.c_double()
    _lib.call("vr_compute_forcing", grad_norm, grad0_norm, C.byref(r))
    return r.value


def pcg_solve(obj: Objective, state: EvalState, rhs, rel_tol, max_iter, precond="spectral"):
    ctx = obj.ctx
    drhs = _dev(ctx, rhs)
    x = ctx.empty(3)
    st = _lib.PcgStats()
    pc = _lib.PRECOND_SPECTRAL if precond == "spectral" else _lib.PRECOND_NONE
    _lib.call("vr_pcg_solve", obj.handle, state._h, drhs.ptr, rel_tol, max_iter, pc, x.ptr, C.byref(st))
    stats = {k: getattr(st, k) for k, _ in _lib.PcgStats._fields_}
    return _ret(x, _is_host(rhs)), stats


@dataclass
class SolveResult:
    v: np.ndarray
    report: dict
    records: List[dict] = field(default_factory=list)
    csv: str = ""  # SolveReport::write_csv (solver.cpp:29-47) of this solve


def solve_report_csv(rep, recs, comment: Optional[str] = None) -> str:
    """The reference's SolveReport CSV (vr_solve_report_csv) of a raw report / records."""
    need = C.c_size_t()
    cm = comment.encode() if comment is not None else None
    _lib.call("vr_solve_report_csv", C.byref(rep), recs, cm, None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    _lib.call("vr_solve_report_csv", C.byref(rep), recs, cm, buf, need.value, None)
    return buf.value.decode()


def _report_dict(r: _lib.SolveReport) -> dict:
    d = {k: getattr(r, k) for k, _ in _lib.SolveReport._fields_ if k not in ("fine", "coarse")}
    d["stop_name"] = _lib.STOP_NAMES[r.stop]
    for nm in ("fine", "coarse"):
        c = getattr(r, nm)
        d[nm] = {k: getattr(c, k) for k, _ in _lib.Counters._fields_}
    return d


def _records(recs, n) -> List[dict]:
    return [{k: getattr(recs[i], k) for k, _ in _lib.IterationRecord._fields_} for i in range(n)]


_PRECOND = {"none": _lib.PRECOND_NONE, "spectral": _lib.PRECOND_SPECTRAL,
            "two_level": _lib.PRECOND_TWO_LEVEL}


def gauss_newton_solve(ctx, m_R, m_T, v0, model=None, params=None, precond="spectral",
                       max_records=512, twolevel=None):
    """gauss_newton_solve (solver.hpp:159-164) with the C++ host driver. precond:
    "spectral" (SpectralPreconditioner), "none", or "two_level" (TwoLevelPreconditioner,
    options from make_twolevel_options / `twolevel`)."""
    model = model if model is not None else make_model()
    params = params if params is not None else make_params()
    dR, dT, dv0 = _dev(ctx, m_R), _dev(ctx, m_T), _dev(ctx, v0)
    vout = ctx.empty(3)
    rep = _lib.SolveReport()
    recs = (_lib.IterationRecord * max_records)()
    pc = _enum(_PRECOND, precond)
    if pc == _lib.PRECOND_TWO_LEVEL:
        opts = twolevel if twolevel is not None else make_twolevel_options()
        _lib.call("vr_gauss_newton_solve_two_level", ctx.handle, dR.ptr, dT.ptr, dv0.ptr,
                  C.byref(model), C.byref(params), C.byref(opts), vout.ptr, C.byref(rep), recs,
                  max_records)
    else:
        _lib.call("vr_gauss_newton_solve", ctx.handle, dR.ptr, dT.ptr, dv0.ptr, C.byref(model),
                  C.byref(params), pc, vout.ptr, C.byref(rep), recs, max_records)
    return SolveResult(_ret(vout, _is_host(m_R, m_T, v0)), _report_dict(rep),
                       _records(recs, min(rep.n_records, max_records)), solve_report_csv(rep, recs, "gpu"))


# ---- two-level preconditioner and grid transfer (precond.hpp, spectral.cpp:228-385) ----
def make_twolevel_options(**kw):
    """TwoLevelOptions (precond.hpp:46-53) with keyword overrides; inner "pcg" or "cheb"."""
    o = _lib.TwoLevelOptions()
    _lib.load().vr_twolevel_options_default(C.byref(o))
    for k, v in kw.items():
        if k == "inner":
            v = {"pcg": _lib.INNER_PCG, "cheb": _lib.INNER_CHEB}.get(v, v)
        if not hasattr(o, k):
            raise ArgumentError(f"TwoLevelOptions has no field {k}")
        setattr(o, k, v)
    return o


def spectral_resample(src: Context, f, dst: Context):
    """spectral_resample (spectral.cpp:340-356): field on src's grid -> dst's grid."""
    df = _dev(src, f)
    nc = df.nfields
    out = dst.empty(nc)
    _lib.call("vr_spectral_resample", src.handle, df.ptr, nc, dst.handle, out.ptr)
    return _ret(out, _is_host(f))


def frequency_filter(ctx: Context, f, band, cutoff):
    """frequency_filter (spectral.cpp:358-385): band "low" (F_L) or "high" (F_H)."""
    df = _dev(ctx, f)
    out = ctx.empty(df.nfields)
    cut = (C.c_int * 3)(*((cutoff,) * 3 if isinstance(cutoff, int) else cutoff))
    b = {"low": 0, "high": 1}.get(band, band)
    _lib.call("vr_frequency_filter", ctx.handle, df.ptr, df.nfields, b, cut, out.ptr)
    return _ret(out, _is_host(f))


class TwoLevelPreconditioner:
    """TwoLevelPreconditioner / TwoLevelContext (precond.hpp:55-110) on the device."""

    def __init__(self, options=None, **kw):
        self.options = options if options is not None else make_twolevel_options(**kw)
        h = C.c_void_p()
        _lib.call("vr_twolevel_create", C.byref(self.options), C.byref(h))
        self._h = h
        self.fine = None

    def rebuild(self, obj: Objective, state: EvalState, eps_H: float):
        self.fine = obj.ctx
        _lib.call("vr_twolevel_rebuild", self._h, obj.handle, state._h, eps_H)

    def apply(self, r):
        dr = _dev(self.fine, r)
        z = self.fine.empty(3)
        _lib.call("vr_twolevel_apply", self._h, self.fine.handle, dr.ptr, z.ptr)
        return _ret(z, _is_host(r))

    def info(self) -> dict:
        dims = (C.c_int * 3)()
        runs, div = C.c_int(), C.c_int()
        b = (C.c_double * 2)()
        c = _lib.Counters()
        _lib.call("vr_twolevel_info", self._h, dims, C.byref(runs), C.byref(div), b, C.byref(c))
        return {"coarse_dims": tuple(dims), "lanczos_runs": runs.value,
                "inner_diverged": bool(div.value), "bounds": (b[0], b[1]),
                "coarse": {k: getattr(c, k) for k, _ in _lib.Counters._fields_}}

    def coarse_matvec(self, u: np.ndarray) -> np.ndarray:
        """Split-form GN matvec on the coarse grid (host arrays of the coarse shape)."""
        dims = self.info()["coarse_dims"]
        u = np.ascontiguousarray(u, dtype=np.float64).reshape((3,) + dims)
        nb = 8 * u.size
        ptr, out = C.c_void_p(), C.c_void_p()
        _lib.call("vr_device_alloc", self.fine.handle, nb, C.byref(ptr))
        _lib.call("vr_device_alloc", self.fine.handle, nb, C.byref(out))
        try:
            _lib.call("vr_memcpy_h2d", self.fine.handle, ptr, u.ctypes.data, nb)
            _lib.call("vr_twolevel_coarse_matvec", self._h, ptr, out)
            res = np.empty((3,) + dims)
            _lib.call("vr_memcpy_d2h", self.fine.handle, res.ctypes.data, out, nb)
        finally:
            _lib.call("vr_device_free", self.fine.handle, ptr)
            _lib.call("vr_device_free", self.fine.handle, out)
        return res

    def close(self):
        if getattr(self, "_h", None):
            _lib.call("vr_twolevel_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def parameter_continuation(ctx, m_R, m_T, v0, model=None, params=None, precond="spectral",
                           max_levels=16, max_records=1024):
    """beta_v continuation 1, 1e-1, ..., target with warm starts."""
    model = model if model is not None else make_model()
    params = params if params is not None else make_params()
    dR, dT, dv0 = _dev(ctx, m_R), _dev(ctx, m_T), _dev(ctx, v0)
    vout = ctx.empty(3)
    reps = (_lib.SolveReport * max_levels)()
    recs = (_lib.IterationRecord * max_records)()
    nl = C.c_int()
    pc = _enum(_PRECOND, precond)
    _lib.call("vr_parameter_continuation", ctx.handle, dR.ptr, dT.ptr, dv0.ptr, C.byref(model),
              C.byref(params), pc, vout.ptr, reps, max_levels, C.byref(nl), recs, max_records)
    reports = [_report_dict(reps[i]) for i in range(min(nl.value, max_levels))]
    nrec = sum(r["n_records"] for r in reports)
    return _ret(vout, _is_host(m_R, m_T, v0)), reports, _records(recs, min(nrec, max_records))


def _levels(ctx, fn, args, max_levels, max_records):
    vout = ctx.empty(3)
    reps = (_lib.SolveReport * max_levels)()
    recs = (_lib.IterationRecord * max_records)()
    nl = C.c_int()
    _lib.call(fn, *args, vout.ptr, reps, max_levels, C.byref(nl), recs, max_records)
    reports = [_report_dict(reps[i]) for i in range(min(nl.value, max_levels))]
    nrec = sum(r["n_records"] for r in reports)
    return vout.numpy(), reports, _records(recs, min(nrec, max_records))


def grid_continuation(ctx, m_R, m_T, v0, levels, model=None, params=None, precond="spectral",
                      max_levels=16, max_records=1024):
    """Coarse-to-fine solves over `levels` grids (vr_grid_continuation)."""
    model = model if model is not None else make_model()
    params = params if params is not None else make_params()
    dR, dT, dv0 = _dev(ctx, m_R), _dev(ctx, m_T), _dev(ctx, v0)
    return _levels(ctx, "vr_grid_continuation",
                   (ctx.handle, dR.ptr, dT.ptr, dv0.ptr, C.byref(model), C.byref(params),
                    _enum(_PRECOND, precond), int(levels)), max_levels, max_records)


def scale_continuation(ctx, m_R, m_T, v0, sigmas, model=None, params=None, precond="spectral",
                       max_levels=16, max_records=1024):
    """Warm-started solves on images smoothed by decreasing sigmas."""
    model = model if model is not None else make_model()
    params = params if params is not None else make_params()
    dR, dT, dv0 = _dev(ctx, m_R), _dev(ctx, m_T), _dev(ctx, v0)
    sg = (C.c_double * len(sigmas))(*[float(x) for x in sigmas])
    vout = ctx.empty(3)
    reps = (_lib.SolveReport * max_levels)()
    recs = (_lib.IterationRecord * max_records)()
    nl = C.c_int()
    _lib.call("vr_scale_continuation", ctx.handle, dR.ptr, dT.ptr, dv0.ptr, C.byref(model),
              C.byref(params), _enum(_PRECOND, precond), sg, len(sigmas), vout.ptr, reps,
              max_levels, C.byref(nl), recs, max_records)
    reports = [_report_dict(reps[i]) for i in range(min(nl.value, max_levels))]
    nrec = sum(r["n_records"] for r in reports)
    return vout.numpy(), reports, _records(recs, min(nrec, max_records))


def beta_search_params(**kw) -> _lib.BetaSearchParams:
    p = _lib.BetaSearchParams()
    _lib.load().vr_beta_search_params_default(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def _trial_dict(t) -> dict:
    return {"beta": t.beta, "feasible": bool(t.feasible), "det_min": t.det.min,
            "det_mean": t.det.mean, "det_max": t.det.max, "report": _report_dict(t.report)}


def beta_search(ctx, m_R, m_T, v0, model=None, params=None, precond="spectral", search=None,
                max_trials=64):
    """Smallest feasible beta_v by bisection on log10 beta (vr_beta_search).
    Returns (beta, v, trials); NumericError (with .trials attached) when beta_hi is infeasible."""
    model = model if model is not None else make_model()
    params = params if params is not None else make_params()
    search = search if search is not None else beta_search_params()
    dR, dT, dv0 = _dev(ctx, m_R), _dev(ctx, m_T), _dev(ctx, v0)
    vout = ctx.empty(3)
    trials = (_lib.BetaTrial * max_trials)()
    nt_ = C.c_int()
    beta = C.c_double()
    try:
        _lib.call("vr_beta_search", ctx.handle, dR.ptr, dT.ptr, dv0.ptr, C.byref(model),
                  C.byref(params), _enum(_PRECOND, precond), C.byref(search), C.byref(beta), vout.ptr,
                  trials, max_trials, C.byref(nt_))
    except _lib.NumericError as e:
        e.trials = [_trial_dict(trials[i]) for i in range(min(nt_.value, max_trials))]
        raise
    return beta.value, vout.numpy(), [_trial_dict(trials[i]) for i in range(min(nt_.value, max_trials))]


# ---- fp32 lane: float fields, fp64 stencil arithmetic --------------
class DeviceBufferF32:
    """Raw fp32 device buffer (host round trips by explicit copies)."""

    def __init__(self, ctx: Context, count: int):
        self.ctx, self.count = ctx, int(count)
        p = C.c_void_p()
        _lib.call("vr_device_alloc", ctx.handle, 4 * self.count, C.byref(p))
        self.ptr = p

    @classmethod
    def from_host(cls, ctx, a):
        a = np.ascontiguousarray(a, dtype=np.float32)
        b = cls(ctx, a.size)
        _lib.call("vr_memcpy_h2d", ctx.handle, b.ptr, a.ctypes.data, 4 * a.size)
        return b

    def numpy(self, shape):
        out = np.empty(shape, dtype=np.float32)
        _lib.call("vr_memcpy_d2h", self.ctx.handle, out.ctypes.data, self.ptr, 4 * out.size)
        return out

    def free(self):
        if getattr(self, "ptr", None):
            _lib.call("vr_device_free", self.ctx.handle, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def tricubic_interpolate_f32(ctx, f, points):
    """tricubic_interpolate{,2,3}<float> (interp.hpp:80-126) on host float32 arrays."""
    f = np.ascontiguousarray(f, dtype=np.float32)
    nf = 1 if f.ndim == 3 else f.shape[0]
    df, dp = DeviceBufferF32.from_host(ctx, f), DeviceBufferF32.from_host(ctx, points)
    out = DeviceBufferF32(ctx, f.size)
    _lib.call("vr_tricubic_interpolate_f32", ctx.handle, df.ptr, dp.ptr, out.ptr, nf)
    return out.numpy(f.shape)


def trace_characteristics_f32(ctx, v, nt, direction="backward"):
    """trace_characteristics<float> (transport.cpp:11-42): fp32 departure points."""
    v = np.ascontiguousarray(v, dtype=np.float32)
    dv = DeviceBufferF32.from_host(ctx, v)
    out = DeviceBufferF32(ctx, v.size)
    _lib.call("vr_trace_characteristics_f32", ctx.handle, dv.ptr, nt,
              _lib.TRACE_BACKWARD if direction == "backward" else _lib.TRACE_FORWARD, out.ptr)
    return out.numpy(v.shape)


def solve_state_f32(ctx, m_T, v, nt):
    """solve_state<float> (transport.cpp:72-86): the fp32 state history (nt + 1 fields)."""
    m = np.ascontiguousarray(m_T, dtype=np.float32)
    dm, dv = DeviceBufferF32.from_host(ctx, m), DeviceBufferF32.from_host(ctx, v)
    out = DeviceBufferF32(ctx, (nt + 1) * m.size)
    _lib.call("vr_solve_state_f32", ctx.handle, dm.ptr, dv.ptr, nt, out.ptr)
    return out.numpy((nt + 1,) + m.shape)


class StateF32:
    """EvalState<float> (device resident)."""

    def __init__(self, obj, handle):
        self.obj, self._h = obj, handle

    def _scalars(self):
        J, mis, rel = C.c_double(), C.c_double(), C.c_double()
        _lib.call("vr_state_f32_scalars", self._h, C.byref(J), C.byref(mis), C.byref(rel))
        return J.value, mis.value, rel.value

    objective = property(lambda s: s._scalars()[0])
    mismatch = property(lambda s: s._scalars()[1])
    mismatch_rel = property(lambda s: s._scalars()[2])

    def close(self):
        if getattr(self, "_h", None) and getattr(self.obj, "_h", None):
            _lib.call("vr_state_f32_destroy", self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ObjectiveF32:
    """Objective<float> (objective.hpp:56-102, T = float; Gauss-Newton, one GPU) on host
    float32 arrays: fp32 fields, fp64 stencils / transforms / reductions."""

    def __init__(self, ctx: Context, m_R, m_T, model=None):
        self.ctx = ctx
        self.model = model if model is not None else make_model()
        self.shape = tuple(np.shape(m_R))
        self._mR = DeviceBufferF32.from_host(ctx, m_R)
        self._mT = DeviceBufferF32.from_host(ctx, m_T)
        h = C.c_void_p()
        _lib.call("vr_objective_f32_create", ctx.handle, self._mR.ptr, self._mT.ptr, C.byref(self.model),
                  C.byref(h))
        self._h = h

    def counters(self) -> dict:
        c = _lib.Counters()
        _lib.call("vr_objective_f32_counters", self._h, C.byref(c))
        return {k: getattr(c, k) for k, _ in _lib.Counters._fields_}

    def evaluate(self, v) -> StateF32:
        dv = DeviceBufferF32.from_host(self.ctx, v)
        h = C.c_void_p()
        _lib.call("vr_evaluate_f32", self._h, dv.ptr, C.byref(h))
        return StateF32(self, h)

    def compute_gradient(self, state: StateF32):
        g = DeviceBufferF32(self.ctx, 3 * int(np.prod(self.shape)))
        _lib.call("vr_compute_gradient_f32", self._h, state._h, g.ptr)
        return g.numpy((3,) + self.shape)

    def hessian_matvec(self, state: StateF32, v_tilde):
        dv = DeviceBufferF32.from_host(self.ctx, v_tilde)
        out = DeviceBufferF32(self.ctx, 3 * int(np.prod(self.shape)))
        _lib.call("vr_hessian_matvec_f32", self._h, state._h, dv.ptr, out.ptr)
        return out.numpy((3,) + self.shape)

    def close(self):
        if getattr(self, "_h", None):
            _lib.call("vr_objective_f32_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gauss_newton_solve_f32(ctx, m_R, m_T, v0, model=None, params=None, precond="spectral",
                           max_records=512, twolevel=None):
    """gauss_newton_solve<float> (solver.cpp:154-269) on host float32 arrays; precond
    "two_level" takes TwoLevelOptions in `twolevel`."""
    model = model if model is not None else make_model()
    params = params if params is not None else make_params()
    dR, dT, dv0 = (DeviceBufferF32.from_host(ctx, a) for a in (m_R, m_T, v0))
    v0 = np.asarray(v0)
    vout = DeviceBufferF32(ctx, v0.size)
    rep = _lib.SolveReport()
    recs = (_lib.IterationRecord * max_records)()
    if precond == "two_level":
        _lib.call("vr_gauss_newton_solve_two_level_f32", ctx.handle, dR.ptr, dT.ptr, dv0.ptr, C.byref(model),
                  C.byref(params), C.byref(twolevel) if twolevel is not None else None, vout.ptr,
                  C.byref(rep), recs, max_records)
    else:
        _lib.call("vr_gauss_newton_solve_f32", ctx.handle, dR.ptr, dT.ptr, dv0.ptr, C.byref(model),
                  C.byref(params), _enum(_PRECOND, precond), vout.ptr, C.byref(rep), recs, max_records)
    return SolveResult(vout.numpy(v0.shape), _report_dict(rep), _records(recs, min(rep.n_records, max_records)))


def parameter_continuation_f32(ctx, m_R, m_T, v0, model=None, params=None, precond="spectral",
                               max_levels=16, max_records=1024):
    """beta_v continuation over the fp32 solve on host float32 arrays, or on
    DeviceBufferF32 inputs (then the result stays on the device)."""
    model = model if model is not None else make_model()
    params = params if params is not None else make_params()
    bufs = [a if isinstance(a, DeviceBufferF32) else DeviceBufferF32.from_host(ctx, a) for a in (m_R, m_T, v0)]
    host = not isinstance(v0, DeviceBufferF32)
    n3 = bufs[2].count
    vout = DeviceBufferF32(ctx, n3)
    reps = (_lib.SolveReport * max_levels)()
    recs = (_lib.IterationRecord * max_records)()
    nl = C.c_int()
    _lib.call("vr_parameter_continuation_f32", ctx.handle, bufs[0].ptr, bufs[1].ptr, bufs[2].ptr,
              C.byref(model), C.byref(params), _enum(_PRECOND, precond), vout.ptr, reps, max_levels,
              C.byref(nl), recs, max_records)
    reports = [_report_dict(reps[i]) for i in range(min(nl.value, max_levels))]
    nrec = sum(r["n_records"] for r in reports)
    v = vout.numpy(np.shape(v0)) if host else vout
    return v, reports, _records(recs, min(nrec, max_records))


def _f32_op(ctx, fn, a, nout, *extra):
    a = np.ascontiguousarray(a, dtype=np.float32)
    din = DeviceBufferF32.from_host(ctx, a)
    n = a.size if a.ndim == 3 else a[0].size
    out = DeviceBufferF32(ctx, nout * n)
    _lib.call(fn, ctx.handle, din.ptr, out.ptr, *extra)
    shape = a.shape if a.ndim == 3 else a.shape[1:]
    return out.numpy(((nout,) if nout > 1 else ()) + tuple(shape))


def gradient_f32(ctx, f):
    """gradient<float> (spectral.cpp:108-122): fp64 transforms, fp32 fields."""
    return _f32_op(ctx, "vr_gradient_f32", f, 3)


def divergence_f32(ctx, v):
    return _f32_op(ctx, "vr_divergence_f32", v, 1)


def apply_reg_operator_f32(ctx, v, norm=None, mode="apply", beta=1.0):
    norm = norm if norm is not None else make_norm()
    return _f32_op(ctx, "vr_apply_reg_operator_f32", v, 3, C.byref(norm), _enum(_MODE, mode), float(beta))


def apply_projection_f32(ctx, v, kind="incompressible", beta_v=0.0, beta_w=0.0):
    return _f32_op(ctx, "vr_apply_projection_f32", v, 3, _enum(_PROJ, kind), float(beta_v), float(beta_w))


def gaussian_smooth_f32(ctx, f, sigma_voxels):
    f = np.ascontiguousarray(f, dtype=np.float32)
    nc = 1 if f.ndim == 3 else f.shape[0]
    sg = (C.c_double * 3)(*[float(x) for x in sigma_voxels])
    return _f32_op(ctx, "vr_gaussian_smooth_f32", f, nc, nc, sg)


def fft_forward_f32(ctx, f):
    """fft_forward<float> (fft.hpp:28-29): complex128 half spectrum of an fp32 field."""
    f = np.ascontiguousarray(f, dtype=np.float32)
    din = DeviceBufferF32.from_host(ctx, f)
    out = ctx.empty(1, complex_spectrum=True)
    _lib.call("vr_fft_r2c_f32", ctx.handle, din.ptr, out.ptr)
    return out.numpy()


def fft_inverse_f32(ctx, spec):
    """fft_inverse<float> (fft.hpp:31-32): fp32 field from a complex128 half spectrum."""
    ds = ctx.empty(1, complex_spectrum=True)
    ds.upload(spec)
    n1, n2, nh = np.shape(spec)
    out = DeviceBufferF32(ctx, n1 * n2 * 2 * (nh - 1))
    _lib.call("vr_fft_c2r_f32", ctx.handle, ds.ptr, out.ptr)
    return out.numpy((n1, n2, 2 * (nh - 1)))


# ---- postprocess (postprocess.hpp:9-56) -----------------------------------------
def det_deformation_gradient(ctx, v, nt):
    """det grad y by continuity transport (postprocess.cpp:13-29)."""
    dv = _dev(ctx, v)
    out = ctx.empty(1)
    _lib.call("vr_det_deformation_gradient", ctx.handle, dv.ptr, nt, out.ptr)
    return _ret(out, _is_host(v))


def deformation_map(ctx, v, nt, absolute=False):
    """Displacement u(., 1), or y = wrap(x + u) (postprocess.cpp:31-60)."""
    dv = _dev(ctx, v)
    out = ctx.empty(3)
    _lib.call("vr_deformation_map", ctx.handle, dv.ptr, nt, 1 if absolute else 0, out.ptr)
    return _ret(out, _is_host(v))


def det_stats(ctx, det, foreground=None, threshold=0.05) -> dict:
    """min / mean / max of det grad y, optionally on the foreground (postprocess.cpp:62-81)."""
    dd = _dev(ctx, det)
    fg = _dev(ctx, foreground) if foreground is not None else None
    st = _lib.DetSummary()
    _lib.call("vr_det_stats", ctx.handle, dd.ptr, fg.ptr if fg is not None else None, float(threshold),
              C.byref(st))
    return {"min": st.min, "mean": st.mean, "max": st.max}


def transport_labels(ctx, labels, v, nt):
    """Per-code label transport (postprocess.cpp:83-120)."""
    dl, dv = _dev(ctx, labels), _dev(ctx, v)
    out = ctx.empty(1)
    _lib.call("vr_transport_labels", ctx.handle, dl.ptr, dv.ptr, nt, out.ptr)
    return _ret(out, _is_host(labels))


def _ov(o) -> dict:
    return {"dice": o.dice, "false_positive_rate": o.false_positive_rate,
            "false_negative_rate": o.false_negative_rate}


def overlap_scores(ctx, reference, test, mask=None, max_labels=4096) -> dict:
    """Dice / error rates per label and for the union (postprocess.cpp:122-165)."""
    da, db = _dev(ctx, reference), _dev(ctx, test)
    dm = _dev(ctx, mask) if mask is not None else None
    n = C.c_int()
    codes = (C.c_int * max_labels)()
    per = (_lib.Overlap * max_labels)()
    uni = _lib.Overlap()
    _lib.call("vr_overlap_scores", ctx.handle, da.ptr, db.ptr, dm.ptr if dm is not None else None,
              max_labels, C.byref(n), codes, per, C.byref(uni))
    k = min(n.value, max_labels)
    return {"per_label": {codes[i]: _ov(per[i]) for i in range(k)}, "union": _ov(uni),
            "n_labels": n.value}


# ---- x1-slab decomposition ---------------------------------
SLAB_FIELDS = ("planes", "first_plane", "halo", "n2s", "k2_off", "points", "spectrum",
               "padded_stride", "global_points")


def slab_layout(dims, rank: int, nranks: int, halo: int) -> dict:
    """x1-slab geometry of `rank` (host only, no GPU): vr_slab_layout."""
    n1, n2, n3 = (dims,) * 3 if isinstance(dims, int) else tuple(dims)
    out = (C.c_longlong * len(SLAB_FIELDS))()
    _lib.call("vr_slab_layout", n1, n2, n3, rank, nranks, halo, out)
    return dict(zip(SLAB_FIELDS, (int(x) for x in out)))


def slab_halo_required(vmax_x1: float, nt: int, n1: int) -> int:
    """Halo planes a velocity with max |v_1| = vmax_x1 needs (vr_slab_halo_required)."""
    planes = C.c_int()
    _lib.call("vr_slab_halo_required", float(vmax_x1), nt, n1, C.byref(planes))
    return planes.value


def nccl_unique_id() -> bytes:
    """NCCL unique id for vr_ctx_create_dist (create on one rank, broadcast)."""
    buf = C.create_string_buffer(128)
    _lib.call("vr_nccl_unique_id", buf)
    return buf.raw


class DistContext(Context):
    """This process's x1 slab of a grid decomposed over `nranks` GPUs (NCCL)."""

    def __init__(self, dims, rank: int, nranks: int, uid: bytes, device: int = 0, halo: int = 16):
        if isinstance(dims, int):
            dims = (dims, dims, dims)
        self.dims = tuple(int(d) for d in dims)
        h = C.c_void_p()
        _lib.call("vr_ctx_create_dist", self.dims[0], self.dims[1], self.dims[2], device, rank,
                  nranks, uid, halo, C.byref(h))
        self._h = h
        vals = [C.c_int() for _ in range(5)]
        _lib.call("vr_ctx_slab", h, *[C.byref(x) for x in vals])
        self.rank, self.nranks, self.planes, self.first_plane, self.halo = (x.value for x in vals)
        self.local_dims = (self.planes, self.dims[1], self.dims[2])
        self.N = self.planes * self.dims[1] * self.dims[2]
        self.nh = self.dims[2] // 2 + 1

    def slab(self, arr):
        """This rank's planes of a global host array (scalar or vector field)."""
        a = np.asarray(arr)
        sl = slice(self.first_plane, self.first_plane + self.planes)
        return np.ascontiguousarray(a[..., sl, :, :])


def dist_selftest_objective(P, m_R, m_T, v, vt, model=None, halo=8, device=0):
    """Evaluate + gradient + Hessian matvec + apply_reg on P virtual slab ranks on
    one GPU; returns (gradient, matvec, reg, scalars) assembled over all slabs."""
    dims = tuple(np.shape(m_R))
    model = model if model is not None else make_model()
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in (m_R, m_T, v, vt)]
    g, mv, rg = (np.empty((3,) + dims) for _ in range(3))
    sc = np.empty(5)
    _lib.call("vr_dist_selftest_objective", P, dims[0], dims[1], dims[2], device, halo,
              C.byref(model), *[x.ctypes.data for x in a], g.ctypes.data, mv.ctypes.data,
              rg.ctypes.data, sc.ctypes.data)
    return g, mv, rg, dict(objective=sc[0], mismatch=sc[1], mismatch_rel=sc[2], grad_norm=sc[3],
                           vt_H_vt=sc[4])


def dist_selftest_postprocess(P, v, nt, halo=8, device=0):
    """det grad y, the absolute deformation map and det_stats on P virtual slab ranks."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    dims = v.shape[1:]
    det, ymap, st = np.empty(dims), np.empty((3,) + dims), np.empty(3)
    _lib.call("vr_dist_selftest_postprocess", P, dims[0], dims[1], dims[2], device, halo, v.ctypes.data, nt,
              det.ctypes.data, ymap.ctypes.data, st.ctypes.data)
    return det, ymap, {"min": st[0], "max": st[1], "mean": st[2]}


def dist_selftest_labels(P, labels, v, nt, halo=8, device=0, max_labels=256):
    """transport_labels + overlap_scores(labels, warped) on P virtual slab ranks."""
    labels = np.ascontiguousarray(labels, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    dims = labels.shape
    warped = np.empty(dims)
    n = C.c_int()
    codes = (C.c_int * max_labels)()
    per = (_lib.Overlap * max_labels)()
    uni = _lib.Overlap()
    _lib.call("vr_dist_selftest_labels", P, dims[0], dims[1], dims[2], device, halo, labels.ctypes.data,
              v.ctypes.data, nt, warped.ctypes.data, max_labels, C.byref(n), codes, per, C.byref(uni))
    k = min(n.value, max_labels)
    return warped, {"per_label": {codes[i]: _ov(per[i]) for i in range(k)}, "union": _ov(uni),
                    "n_labels": n.value}


def dist_selftest_solve(P, m_R, m_T, v0, model=None, params=None, halo=8, device=0, precond="spectral",
                        two_level=None):
    """A full GN solve on P virtual slab ranks on one GPU (precond: none / spectral / two_level)."""
    dims = tuple(np.shape(m_R))
    model = model if model is not None else make_model()
    params = params if params is not None else make_params()
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in (m_R, m_T, v0)]
    vout = np.empty((3,) + dims)
    rep = _lib.SolveReport()
    pc = {"none": 0, "spectral": 1, "two_level": 2}[precond]
    _lib.call("vr_dist_selftest_solve_precond", P, dims[0], dims[1], dims[2], device, halo,
              C.byref(model), C.byref(params), pc, C.byref(two_level) if two_level is not None else None,
              *[x.ctypes.data for x in a], vout.ctypes.data, C.byref(rep))
    return vout, _report_dict(rep)
