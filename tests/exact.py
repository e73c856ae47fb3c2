"""Test infrastructure: the regularisation operator beta * A^{1, -1, -1/2} evaluated in
extended precision, as the exact answer the fp64 GPU path and the fp64 reference are both
measured against.

The operator is the Fourier multiplier of proj/src/spectral.cpp:166-184 (symbol
RegNorm::symbol, proj/include/veloreg/spectral.hpp:91-101, on |k|^2 = k2_full with the
fft_freq convention of proj/include/veloreg/grid.hpp:58-60; zero singular values replaced by
one before inversion). Here the transforms run in x87 long double (64-bit mantissa, eps
1.1e-19, scipy.fft's pocketfft long-double path) on the SAME fp64 input array, so the result
is the exact image of that input up to ~1e-18 -- including the input's own round-off in
the empty high modes, which the H2 symbol |k|^4 amplifies by up to ~2.4e9 at 256^3. An fp64
FFT pair adds its own ~1e-16 round-off in every mode on top of that; the parity criterion is
that the GPU's error against this exact answer is no worse than the reference's (1.5x).
"""
from __future__ import annotations

import os

import numpy as np


def _fft_freq(n):
    # grid.hpp:58-60: 0..n/2, -(n/2-1)..-1 (Nyquist +n/2)
    k = np.arange(n, dtype=np.longdouble)
    return np.where(k <= n // 2, k, k - n)


def _symbol(kind, k2, gamma=1.0, helmholtz_squared=True):
    if kind == "h1":
        return k2
    if kind == "h2":
        return k2 * k2
    if kind == "h3":
        return k2 * k2 * k2
    s = k2 + np.longdouble(gamma)
    return s * s if helmholtz_squared else s


def exact_reg(v, kind="h2", beta=1e-2, mode="apply", gamma=1.0, helmholtz_squared=True):
    """beta A v (mode 'apply'), (beta A)^-1 v ('inverse') or (beta A)^-1/2 v ('inverse_sqrt')
    per component of a (3, n1, n2, n3) or (n1, n2, n3) fp64 (or long double) array, in
    long double; returns long double."""
    import scipy.fft as sf
    a = np.asarray(v)
    if a.dtype != np.longdouble:
        a = a.astype(np.float64)  # the fp64 input both sides receive, taken as exact
    comps = a if a.ndim == 4 else a[None]
    n1, n2, n3 = comps.shape[1:]
    k1 = _fft_freq(n1)[:, None, None]
    k2 = _fft_freq(n2)[None, :, None]
    k3 = np.arange(n3 // 2 + 1, dtype=np.longdouble)[None, None, :]
    s = _symbol(kind, k1 * k1 + k2 * k2 + k3 * k3, gamma, helmholtz_squared)
    b = np.longdouble(beta)
    if mode == "apply":
        m = b * s
    else:
        s = np.where(s == 0, np.longdouble(1), s)
        m = 1 / (b * s) if mode == "inverse" else 1 / np.sqrt(b * s)
    w = os.cpu_count() or 1
    out = np.empty(comps.shape, dtype=np.longdouble)
    for c in range(comps.shape[0]):
        spec = sf.rfftn(comps[c].astype(np.longdouble), workers=w)
        spec *= m
        out[c] = sf.irfftn(spec, s=(n1, n2, n3), workers=w)
        del spec
    return out if a.ndim == 4 else out[0]


def rel_err(x, exact):
    """||x - exact|| / ||exact|| in long double."""
    x = np.asarray(x, dtype=np.longdouble)
    e = np.asarray(exact, dtype=np.longdouble)
    return float(np.sqrt(((x - e) ** 2).sum()) / np.sqrt((e * e).sum()))


def sampled_max_err(x, exact, count=100_000, seed=5):
    """max |x - exact| / max |exact| over `count` seeded grid points."""
    e = np.asarray(exact).reshape(-1)
    idx = np.random.default_rng(seed).integers(0, e.size, count)
    d = np.abs(np.asarray(x).reshape(-1)[idx].astype(np.longdouble) - e[idx])
    return float(d.max() / np.abs(e).max())


# GPU error vs exact must not exceed the reference's by more than this factor; below the
# floor both are at round-off level and the ratio carries no information (1000x under the
# north star's 1e-10 parity bar)
RATIO = 1.5
FLOOR = 1e-13


def no_worse_than_reference(e_gpu, e_ref, ratio=RATIO, floor=FLOOR):
    return e_gpu <= max(ratio * e_ref, floor)
