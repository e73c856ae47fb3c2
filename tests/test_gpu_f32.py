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


@pytest.mark.parametrize("n", [16, 32])
@pytest.mark.parametrize("kind", ["h2", "h1div", "h2_full_newton"])
def test_objective_f32(vr, ref, ctx, n, kind):
    # Objective<float> (objective.cpp:35-156, T = float): J, mismatch, reduced gradient and
    # GN Hessian matvec against the reference's float instantiation, same PDE-solve counts
    dims = (n, n, n)
    c = ctx(dims)
    mR, mT, vs = ref.generate_synthetic(dims, 4)
    if kind == "h2":
        model = vr.make_model()
    elif kind == "h2_full_newton":  # transport.cpp:192-226, objective.cpp:143-148 with T = float
        model = vr.make_model(gauss_newton=False)
    else:
        model = vr.make_model("h1", beta_v=1e-3, nt=4, div_penalty=True, beta_w=1e-4,
                              projection="near_incompressible")
    o = vr.ObjectiveF32(c, mR, mT, model)
    ro = ref.ObjectiveF32(mR, mT, model)
    vt = ref.random_smooth_vector(dims, 2, 142, 1.0)
    for v in (0.5 * vs, np.zeros_like(vs)):
        s, rs = o.evaluate(v), ro.evaluate(v)
        sc = rs.scalars()
        assert abs(s.objective - sc["objective"]) <= 1e-5 * abs(sc["objective"])
        assert abs(s.mismatch_rel - sc["mismatch_rel"]) <= 1e-5 * max(abs(sc["mismatch_rel"]), 1e-30)
        g, g_ref = o.compute_gradient(s), ro.compute_gradient(rs)
        assert g.dtype == np.float32
        assert rel_l2(g, g_ref) <= 1e-5
        h, h_ref = o.hessian_matvec(s, vt), ro.hessian_matvec(rs, vt)
        assert rel_l2(h, h_ref) <= 1e-5
    assert o.counters() == ro.counters()
    # and against the fp64 lane at the same inputs: fp32 storage only
    o64 = vr.Objective(c, mR, mT, model)
    s64 = o64.evaluate(0.5 * vs)
    o64.compute_gradient(s64)
    s32 = o.evaluate(0.5 * vs)
    o.compute_gradient(s32)
    assert rel_l2(o.hessian_matvec(s32, vt), o64.hessian_matvec(s64, vt)) <= 1e-4


@pytest.mark.parametrize("n,gn", [(16, True), (32, True), (16, False)])
def test_gn_solve_f32(vr, ref, ctx, n, gn):
    # gauss_newton_solve<float> (gn = False: the full-Newton Hessian): Newton iterations +-1,
    # final mismatch and |g| within 1 %
    dims = (n, n, n)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model, params = vr.make_model(gauss_newton=gn), vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3,) + dims)
    res = vr.gauss_newton_solve_f32(c, mR, mT, v0, model, params)
    v_ref, rep, _ = ref.gauss_newton_solve_f32(mR, mT, v0, model, params)
    g = res.report
    assert res.v.dtype == np.float32 and g["success"]
    assert g["stop"] == rep["stop"]
    assert abs(g["outer_iterations"] - rep["outer_iterations"]) <= 1
    assert abs(g["final_mismatch_rel"] - rep["final_mismatch_rel"]) <= 1e-2 * rep["final_mismatch_rel"]
    assert abs(g["final_grad_rel"] - rep["final_grad_rel"]) <= 1e-2 * rep["final_grad_rel"]
    if g["outer_iterations"] == rep["outer_iterations"]:
        assert rel_l2(res.v, v_ref) <= 1e-4
    # the fp64 lane reaches the same iterate (the paper: fp32 converges identically)
    r64 = vr.gauss_newton_solve(c, mR, mT, v0, model, params)
    assert abs(r64.report["outer_iterations"] - g["outer_iterations"]) <= 1


def test_parameter_continuation_f32(vr, ref, ctx):
    # beta continuation over the fp32 solve vs the restatement over gauss_newton_solve<float>
    dims = (32, 32, 32)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model, params = vr.make_model(), vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3,) + dims)
    vg, rg, _ = vr.parameter_continuation_f32(c, mR, mT, v0, model, params)
    vref, rr = ref.parameter_continuation_f32(mR, mT, v0, model, params)
    assert len(rg) == len(rr) == 3
    for a, b in zip(rg, rr):
        assert abs(a["outer_iterations"] - b["outer_iterations"]) <= 1
        assert abs(a["final_mismatch_rel"] - b["final_mismatch_rel"]) <= 1e-2 * b["final_mismatch_rel"]
    assert vg.dtype == np.float32 and rel_l2(vg, vref) <= 1e-3


@pytest.mark.parametrize("n,inner", [(16, "pcg"), (32, "pcg"), (32, "cheb")])
def test_two_level_solve_f32(vr, ref, ctx, n, inner):
    """gauss_newton_solve<float> with TwoLevelPreconditioner<float> (precond.cpp:153-249,
    solver.cpp:208-221): the GPU runs the fp32 Newton / split-system PCG with the coarse-grid
    machinery in fp64; Newton iterations +-1, final mismatch and |g| within 1 % of the
    reference's float instantiation, coarse work recorded."""
    dims = (n, n, n)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model, params = vr.make_model("h2", beta_v=1e-2, nt=4), vr.make_params(eps_opt=1e-2)
    opts = vr.make_twolevel_options(inner=inner)
    v0 = np.zeros((3,) + dims)
    res = vr.gauss_newton_solve_f32(c, mR, mT, v0, model, params, precond="two_level", twolevel=opts)
    v_ref, rep, _ = ref.gauss_newton_solve_two_level_f32(mR, mT, v0, model, params, opts)
    g = res.report
    assert res.v.dtype == np.float32 and g["success"] and g["stop"] == rep["stop"]
    assert abs(g["outer_iterations"] - rep["outer_iterations"]) <= 1
    assert abs(g["final_mismatch_rel"] - rep["final_mismatch_rel"]) <= 1e-2 * rep["final_mismatch_rel"]
    assert abs(g["final_grad_rel"] - rep["final_grad_rel"]) <= 1e-2 * rep["final_grad_rel"]
    assert g["coarse"]["hessian_matvecs"] > 0
    if g["outer_iterations"] == rep["outer_iterations"]:
        assert rel_l2(res.v, v_ref) <= 1e-3
