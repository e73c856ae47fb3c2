"""GPU parity: tricubic interpolation and semi-Lagrangian transport vs the compiled reference.

Reference: proj/include/veloreg/interp.hpp:10-126, proj/src/transport.cpp:11-237.
"""
import numpy as np
import pytest

from conftest import periodic_diff, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-10


def grid_points(dims):
    axes = [2 * np.pi * np.arange(n) / n for n in dims]
    return np.stack(np.meshgrid(*axes, indexing="ij"))


@pytest.mark.parametrize("dims", [(8, 16, 32), (16, 16, 16), (32, 32, 32)])
def test_tricubic_random_points(vr, ref, ctx, dims):
    c = ctx(dims)
    rng = np.random.default_rng(3)
    f = ref.random_rough_scalar(dims, 3)
    # arbitrary real coordinates, including negative and > 2pi (wrapped by index arithmetic)
    pts = rng.uniform(-3.0, 10.0, size=(3,) + dims)
    assert rel_l2(vr.tricubic_interpolate(c, f, pts), ref.tricubic_interpolate(f, pts)) < TOL
    f3 = np.stack([f, f * 2 + 1, np.cos(f)])
    assert rel_l2(vr.tricubic_interpolate(c, f3, pts), ref.tricubic_interpolate(f3, pts)) < TOL
    f2 = f3[:2].copy()
    assert rel_l2(vr.tricubic_interpolate(c, f2, pts), ref.tricubic_interpolate(f2, pts)) < TOL


def test_tricubic_reproduces_grid_values(vr, ref, ctx):
    dims = (8, 12 if False else 16, 16)
    c = ctx(dims)
    f = ref.random_rough_scalar(dims, 3)
    out = vr.tricubic_interpolate(c, f, grid_points(dims))
    assert np.abs(out - f).max() < 1e-12


@pytest.mark.parametrize("direction", ["backward", "forward"])
@pytest.mark.parametrize("nt", [1, 4, 8])
def test_trace_characteristics(vr, ref, ctx, direction, nt):
    dims = (32, 32, 32)
    c = ctx(dims)
    _, _, vs = ref.generate_synthetic(dims, 4)
    vs = vs * 1.7 + 0.2 * ref.random_smooth_vector(dims, 2, 9, 1.0)
    g = vr.trace_characteristics(c, vs, nt, direction)
    r = ref.trace_characteristics(vs, nt, direction)
    assert periodic_diff(g, r).max() < 1e-12
    assert g.min() >= 0.0 and g.max() < 2 * np.pi


def test_trace_zero_and_constant(vr, ctx):
    dims = (16, 16, 16)
    c = ctx(dims)
    ch = vr.trace_characteristics(c, np.zeros((3,) + dims), 4)
    assert np.array_equal(ch, grid_points(dims))
    v = np.zeros((3,) + dims)
    v[0] = 0.7
    chb = vr.trace_characteristics(c, v, 4, "backward")
    x = grid_points(dims)[0]
    assert periodic_diff(chb[0], x - 0.7 / 4).max() < 1e-12


def test_state_adjoint_inc_solves(vr, ref, ctx):
    dims = (32, 32, 32)
    nt = 4
    c = ctx(dims)
    mR, mT, vs = ref.generate_synthetic(dims, nt)
    hist_g = vr.solve_state(c, mT, vs, nt)
    hist_r = ref.solve_state(mT, vs, nt)
    assert rel_l2(hist_g, hist_r) < TOL

    term = ref.random_smooth_scalar(dims, 2, 31, 1.0)
    ig, hg = vr.solve_adjoint(c, term, vs, nt, needs_history=True)
    ir, hr = ref.solve_adjoint(term, vs, nt, needs_history=True)
    assert rel_l2(ig, ir) < TOL and rel_l2(hg, hr) < TOL

    ig2, _ = vr.solve_inc_adjoint(c, term, vs, nt)
    ir2, _ = ref.solve_inc_adjoint(term, vs, nt)
    assert rel_l2(ig2, ir2) < TOL

    w = ref.random_smooth_vector(dims, 2, 101, 0.3)
    assert rel_l2(vr.gradient_dot(c, mT, w), ref.gradient_dot(mT, w)) < TOL
    mt_g = vr.solve_inc_state(c, hist_r, vs, w, nt)
    mt_r = ref.solve_inc_state(hist_r, vs, w, nt)
    assert rel_l2(mt_g[1:], mt_r[1:]) < TOL
    assert np.abs(mt_g[0]).max() == 0.0


def test_continuity_factor(vr, ref, ctx):
    dims = (16, 32, 16)
    c = ctx(dims)
    _, _, vs = ref.generate_synthetic(dims, 4)
    v = vs + 0.3 * ref.random_smooth_vector(dims, 2, 3, 1.0)
    xf = ref.trace_characteristics(v, 4, "forward")
    d = ref.divergence(v)
    assert rel_l2(vr.continuity_factor(c, d, xf, 0.25), ref.continuity_factor(d, xf, 0.25)) < TOL


def test_nonfinite_velocity_raises(vr, ctx):
    dims = (16, 16, 16)
    c = ctx(dims)
    v = np.zeros((3,) + dims)
    v[1, 3, 4, 5] = np.nan
    with pytest.raises(vr.NumericError):
        vr.trace_characteristics(c, v, 4)
