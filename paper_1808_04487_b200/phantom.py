"""Seeded synthetic inputs for BASELINE configs 3-5 (host, numpy; not on the hot path).

The reference ships only the analytic section-4.2 pair (proj/src/synthetic.cpp:10-34).
Configs 3-5 ask for a "neuro-sized" phantom instead of NIREP MRI data, which is
not available here: a sum of seeded random ellipsoids, Gaussian-smoothed and
normalised to [0, 1], and a seeded band-limited stationary velocity scaled to a
given maximum displacement. Both arms of every
comparison receive the same arrays.
"""
from __future__ import annotations

import numpy as np

TWO_PI = 2.0 * np.pi


def _quat_to_mat(q):
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def _freq(n):
    # fft_freq convention (grid.hpp:58-60): 0..n/2, -(n/2-1)..-1
    return np.fft.fftfreq(n, 1.0 / n)


def gaussian_smooth_np(f, sigma_voxels):
    """Spectral Gaussian exp(-1/2 sum sigma_d^2 h_d^2 k_d^2) (spectral.cpp:84-99)."""
    n1, n2, n3 = f.shape
    k1 = _freq(n1)[:, None, None]
    k2 = _freq(n2)[None, :, None]
    k3 = np.arange(n3 // 2 + 1, dtype=np.float64)[None, None, :]
    h = (TWO_PI / n1, TWO_PI / n2, TWO_PI / n3)
    s = sigma_voxels
    e = (s[0] * s[0] * h[0] * h[0]) * k1 * k1 + (s[1] * s[1] * h[1] * h[1]) * k2 * k2 + (s[2] * s[2] * h[2] * h[2]) * k3 * k3
    return np.fft.irfftn(np.fft.rfftn(f) * np.exp(-0.5 * e), s=f.shape, axes=(0, 1, 2))


def ellipsoid_phantom(n, count=40, seed=1808, sigma_voxels=2.0):
    """Sum of `count` random ellipsoids: centres U[0,2pi)^3, semi-axes U[0.1,0.6] rad,
    uniform random rotation, intensities U[0.2,1]; periodic minimum-image distance;
    Gaussian-smoothed (sigma in voxels) and rescaled to [0, 1]."""
    rng = np.random.default_rng(seed)
    h = TWO_PI / n
    img = np.zeros((n, n, n))
    for _ in range(count):
        c = rng.uniform(0.0, TWO_PI, 3)
        ax = rng.uniform(0.1, 0.6, 3)
        q = rng.standard_normal(4)
        q /= np.linalg.norm(q)
        R = _quat_to_mat(q)
        inten = rng.uniform(0.2, 1.0)
        r = ax.max()
        idx = []
        for a in range(3):
            lo = int(np.floor((c[a] - r) / h)) - 1
            hi = int(np.ceil((c[a] + r) / h)) + 1
            idx.append(np.arange(lo, hi + 1))
        d = [(i * h - c[a]) for a, i in enumerate(idx)]  # unwrapped offsets = minimum image (r < pi)
        D0, D1, D2 = np.meshgrid(d[0], d[1], d[2], indexing="ij")
        Y = np.einsum("ji,j...->i...", R, np.stack([D0, D1, D2]))  # R^T d
        inside = (Y[0] / ax[0]) ** 2 + (Y[1] / ax[1]) ** 2 + (Y[2] / ax[2]) ** 2 <= 1.0
        w = [np.mod(i, n) for i in idx]
        img[np.ix_(w[0], w[1], w[2])] += inten * inside
    img = gaussian_smooth_np(img, (sigma_voxels,) * 3)
    lo, hi = img.min(), img.max()
    return (img - lo) / (hi - lo) if hi > lo else np.zeros_like(img)


def bandlimited_velocity(n, kmax, max_disp, seed=4487):
    """Per component c: i.i.d. N(0,1) real/imag half-spectrum coefficients on integer
    wavevectors 0 < |k|_2 <= kmax (seed + 7919 (c+1)), c2r, then one common scale so
    that max_x |v(x)|_2 = max_disp (max_magnitude, field_ops.hpp:91-97)."""
    k1 = _freq(n)[:, None, None]
    k2 = _freq(n)[None, :, None]
    k3 = np.arange(n // 2 + 1, dtype=np.float64)[None, None, :]
    mask = (k1 * k1 + k2 * k2 + k3 * k3) <= kmax * kmax
    mask[0, 0, 0] = False
    nnz = int(mask.sum())
    v = np.empty((3, n, n, n))
    for c in range(3):
        rng = np.random.default_rng(seed + 7919 * (c + 1))
        spec = np.zeros((n, n, n // 2 + 1), dtype=np.complex128)
        spec[mask] = rng.standard_normal(nnz) + 1j * rng.standard_normal(nnz)
        v[c] = np.fft.irfftn(spec, s=(n, n, n), axes=(0, 1, 2))
    mag = np.sqrt((v * v).sum(axis=0)).max()
    return v * (max_disp / mag)


def bandlimited_direction(n, kmax_inf=2, seed=142):
    """Matvec probe (SURVEY 8(d) 'Matvec bench inputs'): per component N(0,1)
    coefficients on |k|_inf <= kmax_inf (seed 142 + 7919 (c+1)), each component
    scaled to max |vt_c| = 1."""
    k1 = _freq(n)[:, None, None]
    k2 = _freq(n)[None, :, None]
    k3 = np.arange(n // 2 + 1, dtype=np.float64)[None, None, :]
    mask = (np.abs(k1) <= kmax_inf) & (np.abs(k2) <= kmax_inf) & (k3 <= kmax_inf)
    mask[0, 0, 0] = False
    nnz = int(mask.sum())
    out = np.empty((3, n, n, n))
    for c in range(3):
        rng = np.random.default_rng(seed + 7919 * (c + 1))
        spec = np.zeros((n, n, n // 2 + 1), dtype=np.complex128)
        spec[mask] = rng.standard_normal(nnz) + 1j * rng.standard_normal(nnz)
        f = np.fft.irfftn(spec, s=(n, n, n), axes=(0, 1, 2))
        out[c] = f / np.abs(f).max()
    return out


CONFIGS = {
    # BASELINE.json configs[2..4]: (grid, |k| band limit, max displacement)
    3: dict(n=256, kmax=6, disp=0.08 * TWO_PI),
    4: dict(n=512, kmax=10, disp=0.08 * TWO_PI),
    5: dict(n=1024, kmax=16, disp=0.05 * TWO_PI),
}


def make_config_inputs(config=3, n=None):
    """(m_T, v) for BASELINE config 3/4/5 (optionally at another grid size n)."""
    c = CONFIGS[config]
    n = n or c["n"]
    m_T = ellipsoid_phantom(n)
    v = bandlimited_velocity(n, c["kmax"], c["disp"])
    return m_T, v
