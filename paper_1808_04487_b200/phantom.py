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


# ---------------------------------------------------------------------------
# Per-slab generation (x1 slabs, one rank each): the same fields as the global
# generators above, restricted to planes [first, first + planes), without ever
# materialising the global grid (1024^3 fp64 is 8 GiB per field). Global max /
# min come from caller-supplied reductions (torch.distributed all_reduce on the
# bench ranks, identity on one process).

def _ident(x):
    return x


def _slab_irfftn(spec_rows, k1_rows, n, first, planes):
    """Planes [first, first+planes) of irfftn(spec) where spec is zero outside the x1
    wavenumbers k1_rows: the x1 inverse DFT evaluated directly on the slab's planes, then
    numpy's axis-1 ifft and axis-2 irfft (irfftn's own order, so the Hermitian handling
    of the k3 = 0 / Nyquist bins is the same)."""
    x1 = (first + np.arange(planes)) % n
    ph = np.exp(2j * np.pi * ((x1[:, None] * np.asarray(k1_rows)[None, :]) % n) / n) / n
    s = np.tensordot(ph, spec_rows, axes=(1, 0))  # (planes, n2, n3/2+1)
    s = np.fft.ifft(s, axis=1)
    return np.fft.irfft(s, n=n, axis=2) * n * n  # numpy's ifft/irfft scale 1/n each; x1 already 1/n


def _band_rows(n, kmax_box):
    """x1 row indices (fftfreq order) with |k1| <= kmax_box, ascending."""
    return np.nonzero(np.abs(_freq(n)) <= kmax_box)[0]


def _masked_rows_spec(n, rows, row_mask, seed):
    """spec[rows] of the global generators' `spec[mask] = N(0,1) + i N(0,1)` fill without
    the global array: mask nonzeros outside `rows` do not exist, so C order over the
    restricted rows draws the same values in the same order."""
    k1 = _freq(n)[rows][:, None, None]
    k2 = _freq(n)[None, :, None]
    k3 = np.arange(n // 2 + 1, dtype=np.float64)[None, None, :]
    mask = row_mask(k1, k2, k3)
    if rows[0] == 0:
        mask[0, 0, 0] = False  # the k = 0 mode
    nnz = int(mask.sum())
    rng = np.random.default_rng(seed)
    spec = np.zeros((len(rows), n, n // 2 + 1), dtype=np.complex128)
    spec[mask] = rng.standard_normal(nnz) + 1j * rng.standard_normal(nnz)
    return spec


def bandlimited_velocity_slab(n, kmax, max_disp, first, planes, seed=4487, allreduce_max=_ident):
    """Planes [first, first+planes) of bandlimited_velocity(n, kmax, max_disp, seed) (equal to
    round-off); the common scale uses allreduce_max(max over this slab of |v|_2). Returns
    (v_slab, global max |v_1|) -- the latter sizes the semi-Lagrangian halo."""
    rows = _band_rows(n, kmax)
    k1_rows = _freq(n)[rows].astype(np.int64)
    v = np.empty((3, planes, n, n))
    for c in range(3):
        spec = _masked_rows_spec(n, rows, lambda a, b, d: (a * a + b * b + d * d) <= kmax * kmax,
                                 seed + 7919 * (c + 1))
        v[c] = _slab_irfftn(spec, k1_rows, n, first, planes)
    mag = float(allreduce_max(float(np.sqrt((v * v).sum(axis=0)).max())))
    v *= max_disp / mag
    return v, float(allreduce_max(float(np.abs(v[0]).max())))


def bandlimited_direction_slab(n, first, planes, kmax_inf=2, seed=142, allreduce_max=_ident):
    """Planes [first, first+planes) of bandlimited_direction(n, kmax_inf, seed)."""
    rows = _band_rows(n, kmax_inf)
    k1_rows = _freq(n)[rows].astype(np.int64)
    out = np.empty((3, planes, n, n))
    for c in range(3):
        spec = _masked_rows_spec(n, rows, lambda a, b, d: (np.abs(a) <= kmax_inf) & (np.abs(b) <= kmax_inf)
                                 & (d <= kmax_inf), seed + 7919 * (c + 1))
        f = _slab_irfftn(spec, k1_rows, n, first, planes)
        out[c] = f / float(allreduce_max(float(np.abs(f).max())))
    return out


def ellipsoid_phantom_slab(n, first, planes, count=40, seed=1808, sigma_voxels=2.0, margin=None,
                           allreduce_max=_ident, allreduce_min=_ident):
    """Planes [first, first+planes) of ellipsoid_phantom(n, count, seed, sigma_voxels).

    The indicator sum is built on the slab plus `margin` planes each side (same RNG
    stream, so every rank places the same ellipsoids); the x2/x3 Gaussian is spectral
    as in the global generator, the x1 Gaussian is the same periodic kernel applied as a
    spatial convolution truncated at +-margin planes. The spectral multiplier is still
    exp(-19.7) at the Nyquist bin (sigma = 2 voxels at any n), so that kernel has a flat
    ~1e-9/n tail: the slab image equals the global one to ~1e-10 absolute, not to
    round-off (synthetic input only; both arms of a comparison get the same arrays). The
    [0, 1] rescale uses the global min / max from the reductions."""
    margin = int(np.ceil(12 * sigma_voxels)) if margin is None else int(margin)
    margin = min(margin, (n - 1) // 2)  # one period of the periodic kernel, no image counted twice
    rng = np.random.default_rng(seed)
    h = TWO_PI / n
    W = planes + 2 * margin
    plane_of = (first - margin + np.arange(W)) % n
    where = {}
    for q, p in enumerate(plane_of):
        where.setdefault(int(p), []).append(q)
    img = np.zeros((W, n, n))
    for _ in range(count):
        c = rng.uniform(0.0, TWO_PI, 3)
        ax = rng.uniform(0.1, 0.6, 3)
        qv = rng.standard_normal(4)
        qv /= np.linalg.norm(qv)
        R = _quat_to_mat(qv)
        inten = rng.uniform(0.2, 1.0)
        r = ax.max()
        idx = []
        for a in range(3):
            lo = int(np.floor((c[a] - r) / h)) - 1
            hi = int(np.ceil((c[a] + r) / h)) + 1
            idx.append(np.arange(lo, hi + 1))
        sel = [(j, q) for j, i0 in enumerate(idx[0]) for q in where.get(int(i0 % n), [])]
        if not sel:
            continue
        js = np.array([s[0] for s in sel])
        qs = np.array([s[1] for s in sel])
        d0 = idx[0][js] * h - c[0]
        d = [d0, idx[1] * h - c[1], idx[2] * h - c[2]]
        D0, D1, D2 = np.meshgrid(d[0], d[1], d[2], indexing="ij")
        Y = np.einsum("ji,j...->i...", R, np.stack([D0, D1, D2]))
        inside = (Y[0] / ax[0]) ** 2 + (Y[1] / ax[1]) ** 2 + (Y[2] / ax[2]) ** 2 <= 1.0
        w1, w2 = np.mod(idx[1], n), np.mod(idx[2], n)
        for t, q in enumerate(qs):
            img[q][np.ix_(w1, w2)] += inten * inside[t]
    # x2/x3: spectral Gaussian (spectral.cpp:84-99 multiplier restricted to those axes)
    s = sigma_voxels
    k2 = _freq(n)[None, :, None]
    k3 = np.arange(n // 2 + 1, dtype=np.float64)[None, None, :]
    e = (s * s * h * h) * k2 * k2 + (s * s * h * h) * k3 * k3
    img = np.fft.irfftn(np.fft.rfftn(img, axes=(1, 2)) * np.exp(-0.5 * e), s=(n, n), axes=(1, 2))
    # x1: the periodic kernel g(d) = ifft(exp(-1/2 s^2 h^2 k1^2))(d), truncated at +-margin
    g = np.fft.ifft(np.exp(-0.5 * (s * s * h * h) * _freq(n) ** 2)).real
    out = np.zeros((planes, n, n))
    for dd in range(-margin, margin + 1):
        out += g[dd % n] * img[margin - dd: margin - dd + planes]
    lo = float(allreduce_min(float(out.min())))
    hi = float(allreduce_max(float(out.max())))
    return (out - lo) / (hi - lo) if hi > lo else np.zeros_like(out)


def make_config_inputs_slab(config, first, planes, n=None, allreduce_max=_ident, allreduce_min=_ident):
    """(m_T slab, v slab, vt slab, global max |v_1|) for BASELINE config 3/4/5 on planes
    [first, first+planes)."""
    c = CONFIGS[config]
    n = n or c["n"]
    m_T = ellipsoid_phantom_slab(n, first, planes, allreduce_max=allreduce_max, allreduce_min=allreduce_min)
    v, vmax1 = bandlimited_velocity_slab(n, c["kmax"], c["disp"], first, planes, allreduce_max=allreduce_max)
    vt = bandlimited_direction_slab(n, first, planes, allreduce_max=allreduce_max)
    return m_T, v, vt, vmax1
