"""fp32 lane: the semi-Lagrangian operators of the reference's
Objective<float> -- fields and departure points stored in fp32, stencil weights and
sums in fp64, results rounded to fp32 (interp.hpp:55-126, transport.cpp:11-42, :72-86,
T = float) -- against the reference's own float instantiations. Bar (BASELINE north
star): relative L2 <= 1e-5 when the reference is fp32; observed: equal to the last bit
for almost every value (same fp64 arithmetic, one rounding to fp32).
"""
import numpy as np
import pytest

from conftest import periodic_diff, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [16, 32, 64])
@pytest.mark.parametrize("nf", [1, 3])
def test_tricubic_f32(vr, ref, ctx, n, nf):
    dims = (n, n, n)
    c = ctx(dims)
    mR, mT, vs = ref.generate_synthetic(dims, 4)
    f = vs if nf == 3 else mT
    # departure points incl. values outside [0, 2pi) (any real value is wrapped)
    pts = ref.trace_characteristics(vs, 4) + 0.3 * ref.random_smooth_vector(dims, 2, 77, 1.0)
    g = vr.tricubic_interpolate_f32(c, f, pts)
    r = ref.tricubic_interpolate_f32(f, pts)
    assert g.dtype == np.float32
    assert rel_l2(g, r) <= 1e-5
    assert np.mean(g == r) > 0.99


@pytest.mark.parametrize("direction", ["backward", "forward"])
def test_trace_f32(vr, ref, ctx, direction):
    dims = (32, 32, 32)
    c = ctx(dims)
    _, _, vs = ref.generate_synthetic(dims, 4)
    g = vr.trace_characteristics_f32(c, vs, 4, direction)
    r = ref.trace_characteristics_f32(vs, 4, direction)
    assert periodic_diff(g, r).max() <= 1e-5 * 2 * np.pi


def test_solve_state_f32(vr, ref, ctx):
    dims = (32, 32, 32)
    c = ctx(dims)
    _, mT, vs = ref.generate_synthetic(dims, 4)
    g = vr.solve_state_f32(c, mT, vs, 4)
    r = ref.solve_state_f32(mT, vs, 4)
    assert rel_l2(g, r) <= 1e-5
    # and against the fp64 lane: the fp32 rounding of fields and points only
    d = ref.solve_state(mT, vs, 4)
    assert rel_l2(g.astype(np.float64), d) <= 1e-5
    bad = vs.copy()
    bad[0, 1, 2, 3] = np.inf
    with pytest.raises(vr.NumericError):
        vr.solve_state_f32(c, mT, bad, 4)


@pytest.mark.parametrize("n", [16, 32])
def test_spectral_f32(vr, ref, ctx, n):
    # the reference's float instantiations of the spectral module (spectral.cpp:84-222):
    # fp32 fields, fp64 transforms, one rounding at the end
    dims = (n, n, n)
    c = ctx(dims)
    _, mT, vs = ref.generate_synthetic(dims, 4)
    w = ref.random_smooth_vector(dims, 3, 55, 1.0)
    model = vr.make_model()
    cases = [
        (vr.gradient_f32(c, mT), ref.gradient_f32(mT)),
        (vr.divergence_f32(c, w), ref.divergence_f32(w)),
        (vr.apply_projection_f32(c, w, "incompressible"), ref.apply_projection_f32(w, 1)),
        (vr.gaussian_smooth_f32(c, mT, (1.0, 2.0, 0.5)), ref.gaussian_smooth_f32(mT, (1.0, 2.0, 0.5))),
    ]
    for mode, m in (("apply", 0), ("inverse", 1), ("inverse_sqrt", 2)):
        cases.append((vr.apply_reg_operator_f32(c, w, model.norm, mode, 1e-2),
                      ref.apply_reg_operator_f32(w, model.norm, m, 1e-2)))
    for g, r in cases:
        assert g.dtype == np.float32 and g.shape == r.shape
        assert rel_l2(g, r) <= 1e-5
    spec_g, spec_r = vr.fft_forward_f32(c, mT), ref.fft_forward_f32(mT)
    # fp64 transform of the same fp32 input (compared as (re, im) pairs)
    assert rel_l2(np.ascontiguousarray(spec_g).view(np.float64), spec_r.view(np.float64)) <= 1e-10
    assert rel_l2(vr.fft_inverse_f32(c, spec_r), ref.fft_inverse_f32(spec_r, dims)) <= 1e-5
