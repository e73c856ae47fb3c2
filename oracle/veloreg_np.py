"""oracle/veloreg_np.py -- TEST INFRASTRUCTURE ONLY: CPU restatement of the reference.

A numpy restatement of the reference veloreg hot path (/root/reference/proj),
used only as a checker by tests/ (never by the product, which has no CPU path).
Each function cites the reference file:line it follows. Pinned against the
compiled reference (oracle/_ref, tests/test_oracle.py) and against the golden
vectors in tests/golden/ generated from it.

FFT: numpy.fft.rfftn / irfftn (pocketfft) have FFTW's r2c layout
(n1, n2, n3/2+1), an unnormalized forward and a 1/N inverse -- the exact
convention of proj/src/fft.cpp:66-83. Arrays: scalar (n1,n2,n3), vector
(3,n1,n2,n3), time series (nt+1,n1,n2,n3), float64.
"""
from __future__ import annotations

import math

import numpy as np

TWO_PI = 2.0 * math.pi

H1, H2, H3, HELMHOLTZ = 0, 1, 2, 3
APPLY, INVERSE, INVERSE_SQRT = 0, 1, 2
IDENTITY, INCOMPRESSIBLE, NEAR_INCOMPRESSIBLE = 0, 1, 2


# ---- grid (grid.hpp:20-71) -----------------------------------------------------
def spacing(shape):
    return tuple(TWO_PI / n for n in shape)


def cell_volume(shape):
    h = spacing(shape)
    return h[0] * h[1] * h[2]


def fft_freq(n):
    """grid.hpp:60: 0..n/2, -(n/2-1)..-1."""
    i = np.arange(n)
    return np.where(2 * i <= n, i, i - n).astype(np.float64)


def deriv_freq(n):
    """grid.hpp:64: the Nyquist mode of an even axis gets 0."""
    k = fft_freq(n)
    if n % 2 == 0:
        k[n // 2] = 0.0
    return k


def wrap_coord(x):
    """grid.hpp:66-71."""
    y = x - TWO_PI * np.floor(x / TWO_PI)
    y = np.where(y >= TWO_PI, y - TWO_PI, y)
    return np.where(y >= 0.0, y, 0.0)


def coords(shape):
    h = spacing(shape)
    return [h[a] * np.arange(shape[a], dtype=np.float64) for a in range(3)]


def _kgrids(shape, deriv=False):
    f = deriv_freq if deriv else fft_freq
    n1, n2, n3 = shape
    k1 = f(n1)[:, None, None]
    k2 = f(n2)[None, :, None]
    k3 = (deriv_freq(n3) if deriv else fft_freq(n3))[: n3 // 2 + 1][None, None, :]
    return k1, k2, k3


# ---- FFT (fft.cpp:66-115) ---------------------------------------------------------
def fft_forward(f):
    return np.fft.rfftn(f)


def fft_inverse(spec, shape):
    return np.fft.irfftn(spec, s=shape, axes=(0, 1, 2))


# ---- spectral operators (spectral.cpp) --------------------------------------------
def inner_product(a, b):
    """spectral.cpp:47-62 (vector: per-component sums times h^3, added in order)."""
    vol = cell_volume(a.shape[-3:])
    if a.ndim == 4:
        return sum(float(np.sum(a[c] * b[c])) * vol for c in range(3))
    return float(np.sum(a * b)) * vol


def dot_l2(a, b):
    """field_ops.hpp:51-64 (unweighted)."""
    if a.ndim == 4:
        return sum(float(np.sum(a[c] * b[c])) for c in range(3))
    return float(np.sum(a * b))


def norm_l2(a):
    return math.sqrt(dot_l2(a, a))


def _k2_full(shape):
    k1, k2, k3 = _kgrids(shape)
    return k1 * k1 + k2 * k2 + k3 * k3


def _scalar_multiplier(f, m):
    """spectral.cpp:30-39."""
    return fft_inverse(fft_forward(f) * m, f.shape)


def gradient(f):
    """spectral.cpp:108-122."""
    c = fft_forward(f)
    k = _kgrids(f.shape, deriv=True)
    return np.stack([fft_inverse(1j * k[a] * c, f.shape) for a in range(3)])


def divergence(v):
    """spectral.cpp:124-140."""
    shape = v.shape[1:]
    k = _kgrids(shape, deriv=True)
    acc = np.zeros((shape[0], shape[1], shape[2] // 2 + 1), dtype=np.complex128)
    for a in range(3):
        acc = acc + 1j * k[a] * fft_forward(v[a])
    return fft_inverse(acc, shape)


def laplacian(f):
    """spectral.cpp:142-147."""
    return _scalar_multiplier(f, -_k2_full(f.shape))


def helmholtz1_apply(f):
    """spectral.cpp:155-160."""
    return _scalar_multiplier(f, _k2_full(f.shape) + 1.0)


def gaussian_smooth(f, sigma):
    """spectral.cpp:84-99."""
    h = spacing(f.shape)
    k1, k2, k3 = _kgrids(f.shape)
    e = (sigma[0] * sigma[0] * h[0] * h[0] * k1 * k1 + sigma[1] * sigma[1] * h[1] * h[1] * k2 * k2
         + sigma[2] * sigma[2] * h[2] * h[2] * k3 * k3)
    return _scalar_multiplier(f, np.exp(-0.5 * e))


def reg_symbol(kind, k2, gamma=1.0, helmholtz_squared=True):
    """RegNorm::symbol (spectral.hpp:89-101)."""
    if kind == H1:
        return k2
    if kind == H2:
        return k2 * k2
    if kind == H3:
        return k2 * k2 * k2
    s = k2 + gamma
    return s * s if helmholtz_squared else s


def apply_reg_operator(v, kind=H2, mode=APPLY, beta=1.0, gamma=1.0, helmholtz_squared=True):
    """spectral.cpp:166-184 (zero singular values -> 1 before inversion)."""
    s = reg_symbol(kind, _k2_full(v.shape[1:]), gamma, helmholtz_squared)
    if mode == APPLY:
        m = beta * s
    elif mode == INVERSE:
        m = 1.0 / (beta * np.where(s == 0.0, 1.0, s))
    else:
        m = 1.0 / np.sqrt(beta * np.where(s == 0.0, 1.0, s))
    return np.stack([_scalar_multiplier(v[c], m) for c in range(3)])


def apply_projection(f, kind, beta_v=0.0, beta_w=0.0):
    """spectral.cpp:190-214 (deriv_freq wavenumbers, |k|^2 = 0 passes through)."""
    if kind == IDENTITY:
        return f.copy()
    shape = f.shape[1:]
    k = _kgrids(shape, deriv=True)
    kk = k[0] * k[0] + k[1] * k[1] + k[2] * k[2]
    c = [fft_forward(f[a]) for a in range(3)]
    s = 1.0
    if kind == NEAR_INCOMPRESSIBLE:
        s = beta_w * (kk + 1.0) / (beta_v + beta_w * (kk + 1.0))
    kdotf = k[0] * c[0] + k[1] * c[1] + k[2] * c[2]
    with np.errstate(divide="ignore", invalid="ignore"):
        corr = np.where(kk == 0.0, 0.0, kdotf * (s / kk))
    return np.stack([fft_inverse(c[a] - k[a] * corr, shape) for a in range(3)])


# ---- tricubic interpolation (interp.hpp:12-97) -------------------------------------
def cubic_weights(s):
    """interp.hpp:12-18."""
    sm1, sm2, sp1 = s - 1.0, s - 2.0, s + 1.0
    return [-s * sm1 * sm2 * (1.0 / 6.0), sp1 * sm1 * sm2 * 0.5, -sp1 * s * sm2 * 0.5,
            sp1 * s * sm1 * (1.0 / 6.0)]


def _axis_stencil(x, h, n):
    """TricubicStencil ctor (interp.hpp:32-53)."""
    u = x / h
    r = np.rint(u)
    u = np.where(np.abs(u - r) < 1e-12, r, u)
    fl = np.floor(u)
    s = u - fl
    base = np.mod(fl.astype(np.int64) - 1, n)
    idx = [np.where(base + t < n, base + t, base + t - n) for t in range(4)]
    return idx, cubic_weights(s)


def tricubic_interpolate(f, pts):
    """interp.hpp:55-89: sum_a w0 sum_b w1 sum_c w2 f, accumulated in that order."""
    shape = f.shape[-3:]
    h = spacing(shape)
    st = [_axis_stencil(pts[a], h[a], shape[a]) for a in range(3)]
    flat = f.reshape(-1)
    n2, n3 = shape[1], shape[2]
    acc = np.zeros(pts.shape[1:])
    for a in range(4):
        o1 = st[0][0][a] * n2
        acc1 = np.zeros_like(acc)
        for b in range(4):
            o2 = (o1 + st[1][0][b]) * n3
            acc2 = np.zeros_like(acc)
            for c in range(4):
                acc2 = acc2 + st[2][1][c] * flat[o2 + st[2][0][c]]
            acc1 = acc1 + st[1][1][b] * acc2
        acc = acc + st[0][1][a] * acc1
    return acc


# ---- transport (transport.cpp) --------------------------------------------------------
def trace_characteristics(v, nt, direction="backward"):
    """transport.cpp:11-42."""
    shape = v.shape[1:]
    dt = 1.0 / nt
    sign = -1.0 if direction == "backward" else 1.0
    x = np.meshgrid(*coords(shape), indexing="ij")
    mid = np.stack([wrap_coord(x[c] + sign * 0.5 * dt * v[c]) for c in range(3)])
    return np.stack([wrap_coord(x[c] + sign * dt * tricubic_interpolate(v[c], mid)) for c in range(3)])


def continuity_factor(div_v, departure, dt):
    """transport.cpp:44-55."""
    return np.exp(0.5 * dt * (div_v + tricubic_interpolate(div_v, departure)))


def solve_state(m_T, v, nt, bwd=None):
    """transport.cpp:72-86."""
    bwd = trace_characteristics(v, nt, "backward") if bwd is None else bwd
    hist = [m_T.copy()]
    for _ in range(nt):
        hist.append(tricubic_interpolate(hist[-1], bwd))
    return np.stack(hist)


def sweep_continuity(terminal, fwd, factor, nt, observe=None):
    """transport.cpp:88-113 (no-history branch); returns the slices j = nt..0."""
    cur = terminal
    out = {nt: cur}
    if observe:
        observe(nt, cur)
    for j in range(nt - 1, -1, -1):
        cur = tricubic_interpolate(cur, fwd) * factor
        out[j] = cur
        if observe:
            observe(j, cur)
    return out


def solve_adjoint(terminal, v, nt):
    """transport.cpp:115-124; returns the history (nt+1, ...)."""
    fwd = trace_characteristics(v, nt, "forward")
    factor = continuity_factor(divergence(v), fwd, 1.0 / nt)
    sl = sweep_continuity(terminal, fwd, factor, nt)
    return np.stack([sl[j] for j in range(nt + 1)])


def gradient_dot(f, w):
    """transport.cpp:126-148: ((0 + d0 w0) + d1 w1) + d2 w2."""
    g = gradient(f)
    out = np.zeros_like(f)
    for a in range(3):
        out = out + g[a] * w[a]
    return out


def solve_inc_state(m_hist, v, vt, nt, bwd=None):
    """transport.cpp:150-180."""
    bwd = trace_characteristics(v, nt, "backward") if bwd is None else bwd
    hdt = 0.5 / nt
    mt = [np.zeros_like(m_hist[0])]
    q_prev = gradient_dot(m_hist[0], vt)
    for j in range(nt):
        q_next = gradient_dot(m_hist[j + 1], vt)
        tmp = 1.0 * mt[j] + (-hdt) * q_prev
        nxt = tricubic_interpolate(tmp, bwd)
        mt.append(nxt + (-hdt) * q_next)
        q_prev = q_next
    return np.stack(mt)


# ---- objective (objective.cpp) --------------------------------------------------------
class Objective:
    """Objective<double> (objective.cpp:35-186), Gauss-Newton."""

    def __init__(self, m_R, m_T, kind=H2, beta_v=1e-2, nt=4, projection=IDENTITY, gamma=1.0,
                 helmholtz_squared=True, div_penalty=False, beta_w=1e-4):
        self.m_R, self.m_T = m_R, m_T
        self.kind, self.beta_v, self.nt, self.projection = kind, beta_v, nt, projection
        self.gamma, self.hsq, self.div_penalty, self.beta_w = gamma, helmholtz_squared, div_penalty, beta_w
        d = 1.0 * m_T + (-1.0) * m_R
        self.initial_mismatch = inner_product(d, d)
        self.counters = dict(objective_evals=0, gradient_evals=0, hessian_matvecs=0, pde_solves=0)

    def reg(self, u, mode=APPLY, beta=None):
        return apply_reg_operator(u, self.kind, mode, self.beta_v if beta is None else beta,
                                  self.gamma, self.hsq)

    def K(self, u):
        return apply_projection(u, self.projection, self.beta_v, self.beta_w)

    def evaluate(self, v):
        """objective.cpp:47-75."""
        if not np.all(np.isfinite(v)):
            raise FloatingPointError("evaluate_objective: non-finite velocity")
        s = {"v": v.copy()}
        s["bwd"] = trace_characteristics(v, self.nt, "backward")
        s["m_history"] = solve_state(self.m_T, v, self.nt, bwd=s["bwd"])
        self.counters["pde_solves"] += 1
        diff = 1.0 * s["m_history"][-1] + (-1.0) * self.m_R
        s["mismatch"] = inner_product(diff, diff)
        s["mismatch_rel"] = s["mismatch"] / self.initial_mismatch if self.initial_mismatch > 0 else 0.0
        reg = 0.5 * self.beta_v * inner_product(self.reg(v, APPLY, 1.0), v)
        pen = 0.0
        if self.div_penalty:
            w = divergence(v)
            pen = 0.5 * self.beta_w * inner_product(helmholtz1_apply(w), w)
        s["objective"] = 0.5 * s["mismatch"] + reg + pen
        self.counters["objective_evals"] += 1
        return s

    def _ctx(self, s):
        """prepare_adjoint_ctx (objective.cpp:77-84)."""
        if "fwd" not in s:
            s["fwd"] = trace_characteristics(s["v"], self.nt, "forward")
            s["factor"] = continuity_factor(divergence(s["v"]), s["fwd"], 1.0 / self.nt)

    def _accumulate(self, b, f, lam, w):
        """accumulate_weighted_grad (objective.cpp:9-32)."""
        g = gradient(f)
        for a in range(3):
            b[a] = b[a] + w * lam * g[a]

    def compute_gradient(self, s):
        """objective.cpp:86-112."""
        self._ctx(s)
        nt, dt = self.nt, 1.0 / self.nt
        terminal = 1.0 * self.m_R + (-1.0) * s["m_history"][-1]
        b = np.zeros((3,) + self.m_R.shape)

        def obs(j, lam):
            w = 0.5 * dt if (j == 0 or j == nt) else dt
            self._accumulate(b, s["m_history"][j], lam, w)

        sweep_continuity(terminal, s["fwd"], s["factor"], nt, obs)
        self.counters["pde_solves"] += 1
        b = self.K(b)
        s["gradient"] = b + 1.0 * self.reg(s["v"])
        self.counters["gradient_evals"] += 1
        return s["gradient"]

    def hessian_data_matvec(self, s, vt):
        """objective.cpp:123-156 (GN)."""
        if "fwd" not in s:
            raise RuntimeError("hessian_matvec: compute the gradient first")
        nt, dt = self.nt, 1.0 / self.nt
        mt = solve_inc_state(s["m_history"], s["v"], vt, nt, bwd=s["bwd"])
        self.counters["pde_solves"] += 1
        b = np.zeros((3,) + self.m_R.shape)

        def obs(j, lam):
            w = 0.5 * dt if (j == 0 or j == nt) else dt
            self._accumulate(b, s["m_history"][j], lam, w)

        sweep_continuity(-mt[-1], s["fwd"], s["factor"], nt, obs)
        self.counters["pde_solves"] += 1
        b = self.K(b)
        self.counters["hessian_matvecs"] += 1
        return b

    def hessian_matvec(self, s, vt):
        """objective.cpp:114-121."""
        return self.hessian_data_matvec(s, vt) + 1.0 * self.reg(vt)


# ---- solver (solver.cpp) -----------------------------------------------------------
def compute_forcing(g, g0):
    """solver.cpp:23-27."""
    return min(0.5, math.sqrt(g / g0))


def pcg_solve(apply, rhs, rel_tol, max_iter, precond):
    """solver.cpp:51-100."""
    x = np.zeros_like(rhs)
    r0 = norm_l2(rhs)
    st = dict(iterations=0, rel_residual=1.0, converged=False, negative_curvature=False)
    if r0 == 0.0:
        st.update(converged=True, rel_residual=0.0)
        return x, st
    target = rel_tol * r0
    r = rhs.copy()
    z = precond(r)
    s = z.copy()
    rz = dot_l2(r, z)
    for it in range(max_iter):
        Hs = apply(s)
        sHs = dot_l2(s, Hs)
        if sHs <= 0.0:
            st["negative_curvature"] = True
            if it == 0:
                x = z
            st.update(iterations=it + 1, rel_residual=norm_l2(r) / r0)
            return x, st
        kappa = rz / sHs
        x = x + kappa * s
        r = r + (-kappa) * Hs
        st["iterations"] = it + 1
        rn = norm_l2(r)
        st["rel_residual"] = rn / r0
        if rn < target:
            st["converged"] = True
            return x, st
        z = precond(r)
        rz_new = dot_l2(r, z)
        mu = rz_new / rz
        rz = rz_new
        s = 1.0 * z + mu * s
    return x, st


def gauss_newton_solve(m_R, m_T, v0, obj_kwargs, eps_opt=5e-2, abs_grad_tol=1e-6, max_newton=50,
                       max_krylov=100, c1=1e-4, backtrack=0.5, max_trials=20):
    """solver.cpp:154-269 with the spectral preconditioner (solver.hpp:139-150)."""
    obj = Objective(m_R, m_T, **obj_kwargs)
    s = obj.evaluate(v0)
    g = obj.compute_gradient(s)
    g0 = norm_l2(g)
    recs = [dict(k=0, objective=s["objective"], grad_rel=1.0, inner_iterations=0)]
    stop = "zero_gradient" if g0 == 0.0 else None
    gk, k = g0, 0
    while stop is None:
        if gk * gk <= eps_opt * g0 * g0:
            stop = "converged_rel"
            break
        if gk <= abs_grad_tol:
            stop = "converged_abs"
            break
        if k >= max_newton:
            stop = "max_iterations"
            break
        eps_h = compute_forcing(gk, g0)
        d, st = pcg_solve(lambda u: obj.hessian_matvec(s, u), -1.0 * s["gradient"], eps_h, max_krylov,
                          lambda r: obj.reg(r, INVERSE))
        slope = inner_product(s["gradient"], d)
        if slope >= 0.0:
            stop = "line_search_failure"
            break
        alpha, ok = 1.0, False
        for _ in range(max_trials):
            trial = obj.evaluate(1.0 * s["v"] + alpha * d)
            if trial["objective"] <= s["objective"] + c1 * alpha * slope:
                ok = True
                break
            alpha *= backtrack
        if not ok:
            stop = "line_search_failure"
            break
        s = trial
        gk = norm_l2(obj.compute_gradient(s))
        k += 1
        recs.append(dict(k=k, objective=s["objective"], grad_rel=gk / g0, inner_iterations=st["iterations"],
                         step_length=alpha))
    return dict(v=s["v"], stop=stop, outer_iterations=k, final_mismatch_rel=s["mismatch_rel"],
                final_grad_rel=gk / g0 if g0 > 0 else 0.0, records=recs, counters=obj.counters)


def generate_synthetic(shape, nt, amplitude=1.0):
    """synthetic.cpp:16-34."""
    x1, x2, x3 = np.meshgrid(*coords(shape), indexing="ij")
    s1, s2, s3 = np.sin(x1), np.sin(x2), np.sin(x3)
    m_T = (s1 * s1 + s2 * s2 + s3 * s3) / 3.0
    v = np.stack([amplitude * (np.sin(x3) * np.cos(x2) * np.sin(x2)),
                  amplitude * (np.sin(x1) * np.cos(x3) * np.sin(x3)),
                  amplitude * (np.sin(x2) * np.cos(x1) * np.sin(x1))])
    m_R = solve_state(m_T, v, nt)[-1]
    return m_R, m_T, v
