"""GPU parity: FFT and spectral operators vs the compiled reference (oracle/_ref).

Reference: proj/src/fft.cpp:66-115, proj/src/spectral.cpp:84-222.
Bar: relative L2 <= 1e-10 (fp64, BASELINE north star), most land near 1e-15.
"""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-10
GRIDS = [(16, 16, 16), (8, 16, 32), (32, 8, 16), (64, 64, 64), (4, 4, 4)]
# the longest supported axis in every position (1024: four 256-row groups per TMA box and
# 2-column tiles in the strided passes, M = 512 row transforms) and 512 (two row groups)
LONG_AXES = [(1024, 4, 8), (4, 1024, 8), (8, 4, 1024), (512, 8, 4), (4, 512, 16)]


@pytest.mark.parametrize("dims", GRIDS + LONG_AXES)
def test_fft_r2c_c2r(vr, ref, ctx, dims):
    c = ctx(dims)
    f = ref.random_rough_scalar(dims, 11)
    s_ref = ref.fft_forward(f)
    s_gpu = vr.fft_forward(c, f)
    assert s_gpu.shape == s_ref.shape
    assert rel_l2(s_gpu.view(np.float64), s_ref.view(np.float64)) < 1e-13
    back_ref = ref.fft_inverse(s_ref, dims)
    back_gpu = vr.fft_inverse(c, s_ref)
    assert rel_l2(back_gpu, back_ref) < 1e-13
    assert rel_l2(back_gpu, f) < 1e-13


@pytest.mark.parametrize("dims", [(16, 16, 16), (8, 16, 32), (64, 32, 16)] + LONG_AXES)
def test_gradient_divergence_laplacian(vr, ref, ctx, dims):
    c = ctx(dims)
    f = ref.random_smooth_scalar(dims, 3, 5, 1.0) + 0.1 * ref.random_rough_scalar(dims, 6)
    assert rel_l2(vr.gradient(c, f), ref.gradient(f)) < TOL
    v = ref.random_smooth_vector(dims, 3, 7, 1.0)
    assert rel_l2(vr.divergence(c, v), ref.divergence(v)) < TOL
    assert rel_l2(vr.laplacian(c, f), ref.laplacian(f)) < TOL
    assert rel_l2(vr.helmholtz1_apply(c, f), ref.helmholtz1_apply(f)) < TOL


def test_derivatives_exact_on_pure_modes(vr, ctx):
    # test_fields.cpp:103-142 analogue on the GPU path
    n = 16
    c = ctx(n)
    x = 2 * np.pi * np.arange(n) / n
    X1, X2, X3 = np.meshgrid(x, x, x, indexing="ij")
    g = vr.gradient(c, np.sin(X1))
    assert np.abs(g[0] - np.cos(X1)).max() < 1e-12
    assert np.abs(g[1]).max() < 1e-12 and np.abs(g[2]).max() < 1e-12
    for k in [(3, 2, 1), (5, 0, 7), (1, 6, 4)]:
        mode = np.sin(k[0] * X1 + k[1] * X2 + k[2] * X3)
        gm = vr.gradient(c, mode)
        dc = np.cos(k[0] * X1 + k[1] * X2 + k[2] * X3)
        for a in range(3):
            assert np.abs(gm[a] - k[a] * dc).max() < 1e-12 * max(1, k[a])


@pytest.mark.parametrize("kind", ["h1", "h2", "h3", "helmholtz"])
@pytest.mark.parametrize("mode", ["apply", "inverse", "inverse_sqrt"])
def test_reg_operator(vr, ref, ctx, kind, mode):
    dims = (16, 32, 16)
    c = ctx(dims)
    v = ref.random_smooth_vector(dims, 4, 21, 1.0) + 0.01 * np.stack([ref.random_rough_scalar(dims, s) for s in (1, 2, 3)])
    norm = vr.make_norm(kind, gamma=0.7, helmholtz_squared=(kind != "helmholtz" or True))
    m = {"apply": 0, "inverse": 1, "inverse_sqrt": 2}[mode]
    out_g = vr.apply_reg_operator(c, v, norm, mode, beta=3e-2)
    out_r = ref.apply_reg_operator(v, norm, m, 3e-2)
    assert rel_l2(out_g, out_r) < TOL


def test_reg_operator_helmholtz_single(vr, ref, ctx):
    dims = (16, 16, 16)
    c = ctx(dims)
    v = ref.random_smooth_vector(dims, 4, 31, 1.0)
    norm = vr.make_norm("helmholtz", gamma=2.0, helmholtz_squared=False)
    assert rel_l2(vr.apply_reg_operator(c, v, norm, "inverse", 0.5), ref.apply_reg_operator(v, norm, 1, 0.5)) < TOL


@pytest.mark.parametrize("kind,bv,bw", [("incompressible", 0.0, 0.0), ("near_incompressible", 1e-3, 1e-4)])
def test_projection(vr, ref, ctx, kind, bv, bw):
    dims = (32, 16, 16)
    c = ctx(dims)
    v = ref.random_smooth_vector(dims, 5, 41, 1.0)
    k = {"incompressible": 1, "near_incompressible": 2}[kind]
    out_g = vr.apply_projection(c, v, kind, bv, bw)
    assert rel_l2(out_g, ref.apply_projection(v, k, bv, bw)) < TOL
    if kind == "incompressible":
        # Leray: idempotent and divergence free (test_fields.cpp:182-208)
        assert rel_l2(vr.apply_projection(c, out_g, kind), out_g) < 1e-12
        assert np.abs(vr.divergence(c, out_g)).max() < 1e-10


def test_gaussian_smooth(vr, ref, ctx):
    dims = (32, 32, 32)
    c = ctx(dims)
    f = ref.random_rough_scalar(dims, 11)
    for sig in [(0.0, 0.0, 0.0), (1.5, 2.0, 1.0), (2.0, 2.0, 2.0)]:
        assert rel_l2(vr.gaussian_smooth(c, f, sig), ref.gaussian_smooth(f, sig)) < TOL


def test_inner_products_and_rescale(vr, ref, ctx):
    dims = (16, 16, 32)
    c = ctx(dims)
    a = ref.random_rough_scalar(dims, 1)
    b = ref.random_rough_scalar(dims, 2)
    assert abs(vr.inner_product(c, a, b) - ref.inner_product(a, b)) < 1e-12 * abs(ref.inner_product(a, a))
    va = np.stack([a, b, a * b])
    assert abs(vr.dot_l2(c, va, va) - ref.dot_l2(va, va)) < 1e-12 * ref.dot_l2(va, va)
    assert abs(vr.max_magnitude(c, va) - ref.max_magnitude(va)) < 1e-14
    rg, dg = vr.rescale_intensity(c, a)
    rr, dr = ref.rescale_intensity(a)
    assert dg == dr and rel_l2(rg, rr) < 1e-14
    konst = np.full(dims, 5.0)
    _, deg = vr.rescale_intensity(c, konst)
    assert deg


def test_errors(vr, ctx):
    c = ctx(16)
    with pytest.raises(vr.ArgumentError):
        vr.apply_reg_operator(c, np.zeros((3, 16, 16, 16)), vr.make_norm(), "apply", beta=0.0)
    with pytest.raises(vr.ArgumentError):
        vr.apply_reg_operator(c, np.zeros((3, 16, 16, 16)), vr.make_norm("helmholtz", gamma=0.0), "apply")
    with pytest.raises(vr.ArgumentError):
        vr.apply_projection(c, np.zeros((3, 16, 16, 16)), "near_incompressible", 0.0, 1.0)
    with pytest.raises(vr.DimensionError):
        vr.Context((3, 8, 8))
