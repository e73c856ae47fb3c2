"""GPU: the full-Newton Hessian (RegModel::gauss_newton = false) vs the compiled reference
(SURVEY 8(f) #2).

Reference: proj/src/transport.cpp:182-226 (solve_inc_adjoint full-Newton branch: sources
r_j = div(lambda_j vt), two-field gathers), proj/src/objective.cpp:100-102 (adjoint history
kept by the gradient) and :141-148 (the extra (w lambda_j) grad mt_j observer term).
"""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-10

MODELS = {
    "h2": dict(kind="h2", beta_v=1e-2, nt=4),
    "h1div_nearinc": dict(kind="h1", beta_v=1e-3, nt=4, div_penalty=True, beta_w=1e-4,
                          projection="near_incompressible"),
    "helmholtz_nt2": dict(kind="helmholtz", gamma=0.5, beta_v=5e-2, nt=2),
}


def _pair(ref, dims):
    a = 0.5 + ref.random_smooth_scalar(dims, 2, 91, 0.3)
    b = 0.5 + ref.random_smooth_scalar(dims, 2, 92, 0.3)
    return a, b


@pytest.mark.parametrize("name", list(MODELS))
@pytest.mark.parametrize("dims", [(16, 16, 16), (8, 16, 32)])
def test_full_newton_matvec(vr, ref, ctx, name, dims):
    model = vr.make_model(gauss_newton=False, **MODELS[name])
    mR, mT = _pair(ref, dims)
    v = ref.random_smooth_vector(dims, 2, 120, 0.3)
    vt = ref.random_smooth_vector(dims, 2, 142, 1.0)
    ro, go = ref.Objective(mR, mT, model), vr.Objective(ctx(dims), mR, mT, model)
    rs, gs = ro.evaluate(v), go.evaluate(v)
    go.compute_gradient(gs)
    assert rel_l2(gs.gradient, ro.compute_gradient(rs)) < TOL
    assert rel_l2(go.hessian_matvec(gs, vt), ro.hessian_matvec(rs, vt)) < TOL
    assert rel_l2(go.hessian_data_matvec(gs, vt), ro.hessian_data_matvec(rs, vt)) < TOL
    assert go.counters() == ro.counters()
    # the full-Newton term changes the operator (vs the GN matvec of the same state)
    gn = vr.make_model(gauss_newton=True, **MODELS[name])
    og = vr.Objective(ctx(dims), mR, mT, gn)
    sg = og.evaluate(v)
    og.compute_gradient(sg)
    assert rel_l2(og.hessian_data_matvec(sg, vt), go.hessian_data_matvec(gs, vt)) > 1e-6


def test_full_newton_adjoint_history_and_errors(vr, ref, ctx):
    from paper_1808_04487_b200._lib import LogicError
    dims = (16, 16, 16)
    model = vr.make_model(gauss_newton=False)
    mR, mT = _pair(ref, dims)
    v = ref.random_smooth_vector(dims, 2, 120, 0.3)
    go = vr.Objective(ctx(dims), mR, mT, model)
    gs = go.evaluate(v)
    with pytest.raises(LogicError):
        go.hessian_matvec(gs, v)
    go.compute_gradient(gs)
    lam = gs.get(vr._lib.STATE_LAMBDA_HISTORY)
    # lambda_nt = m_R - m_nt (objective.cpp:91-92)
    assert np.abs(lam[-1] - (mR - gs.m_history[-1])).max() < 1e-14


@pytest.mark.parametrize("precond", ["spectral", "two_level"])
def test_full_newton_solve(vr, ref, ctx, precond):
    dims = (16, 16, 16)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model = vr.make_model("h2", beta_v=1e-2, nt=4, gauss_newton=False)
    params = vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3,) + dims)
    res = vr.gauss_newton_solve(c, mR, mT, v0, model, params, precond=precond)
    if precond == "spectral":
        _, rep_r, recs_r = ref.gauss_newton_solve(mR, mT, v0, model, params)
    else:
        _, rep_r, recs_r = ref.gauss_newton_solve_two_level(mR, mT, v0, model, params,
                                                            vr.make_twolevel_options())
    g = res.report
    assert g["stop"] == rep_r["stop"]
    assert abs(g["outer_iterations"] - rep_r["outer_iterations"]) <= 1
    assert abs(g["final_mismatch_rel"] - rep_r["final_mismatch_rel"]) <= 1e-2 * rep_r["final_mismatch_rel"]
    assert abs(g["final_grad_rel"] - rep_r["final_grad_rel"]) <= 1e-2 * rep_r["final_grad_rel"]
    if g["outer_iterations"] == rep_r["outer_iterations"]:
        for a, b in zip(res.records, recs_r):
            assert a["inner_iterations"] == b["inner_iterations"]
