"""GPU end-to-end: Gauss-Newton-Krylov solves vs the compiled reference.

Reference: proj/src/solver.cpp:23-269; tests proj/tests/test_solver.cpp.
Bar (BASELINE north star): Newton iterations +-1; final relative mismatch and
relative gradient norm within 1%.
"""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _compare(rep_g, rep_r):
    assert rep_g["stop"] == rep_r["stop"]
    assert abs(rep_g["outer_iterations"] - rep_r["outer_iterations"]) <= 1
    assert abs(rep_g["final_mismatch_rel"] - rep_r["final_mismatch_rel"]) <= 1e-2 * rep_r["final_mismatch_rel"]
    assert abs(rep_g["final_grad_rel"] - rep_r["final_grad_rel"]) <= 1e-2 * rep_r["final_grad_rel"]


@pytest.mark.parametrize("n", [16, 32, 64])
def test_config1_synthetic_solve(vr, ref, ctx, n):
    # BASELINE config 1 (64^3) and smaller: H2, beta 1e-2, n_t 4, spectral precond, eps 1e-2
    dims = (n, n, n)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model = vr.make_model("h2", beta_v=1e-2, nt=4)
    params = vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3,) + dims)
    res = vr.gauss_newton_solve(c, mR, mT, v0, model, params)
    vr_ref, rep_r, recs_r = ref.gauss_newton_solve(mR, mT, v0, model, params)
    _compare(res.report, rep_r)
    assert res.report["success"]
    if res.report["outer_iterations"] == rep_r["outer_iterations"]:
        assert rel_l2(res.v, vr_ref) < 1e-6
        for a, b in zip(res.records, recs_r):
            assert a["inner_iterations"] == b["inner_iterations"]
            assert abs(a["objective"] - b["objective"]) <= 1e-8 * abs(b["objective"])
    f = res.report["fine"]
    assert f["pde_solves"] == f["objective_evals"] + f["gradient_evals"] + 2 * f["hessian_matvecs"]


def test_h1div_solve(vr, ref, ctx):
    # test_solver.cpp:138-178 configuration (H1-div, near-incompressible K)
    dims = (16, 16, 16)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model = vr.make_model("h1", beta_v=1e-3, nt=4, div_penalty=True, beta_w=1e-4,
                          projection="near_incompressible")
    params = vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3,) + dims)
    res = vr.gauss_newton_solve(c, mR, mT, v0, model, params)
    _, rep_r, _ = ref.gauss_newton_solve(mR, mT, v0, model, params)
    _compare(res.report, rep_r)
    assert res.report["final_mismatch_rel"] < 0.2
    objs = [r["objective"] for r in res.records]
    assert all(b < a for a, b in zip(objs, objs[1:]))


def test_identical_images_stop_immediately(vr, ref, ctx):
    dims = (16, 16, 16)
    c = ctx(dims)
    m = 0.5 + ref.random_smooth_scalar(dims, 2, 700, 0.3)
    res = vr.gauss_newton_solve(c, m, m, np.zeros((3,) + dims), vr.make_model(beta_v=1e-3))
    assert res.report["stop_name"] == "zero_gradient" and res.report["outer_iterations"] == 0


def test_pcg_matches_reference(vr, ref, ctx):
    dims = (16, 16, 16)
    c = ctx(dims)
    mR, mT, vs = ref.generate_synthetic(dims, 4)
    model = vr.make_model()
    go, ro = vr.Objective(c, mR, mT, model), ref.Objective(mR, mT, model)
    gs, rs = go.evaluate(0.5 * vs), ro.evaluate(0.5 * vs)
    go.compute_gradient(gs)
    g = ro.compute_gradient(rs)
    xg, stg = vr.pcg_solve(go, gs, -g, 1e-6, 50)
    xr, str_ = ro.pcg_solve(rs, -g, 1e-6, 50)
    assert stg["iterations"] == str_["iterations"]
    assert rel_l2(xg, xr) < 1e-8


def test_parameter_continuation(vr, ref, ctx):
    dims = (16, 16, 16)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model = vr.make_model("h2", beta_v=1e-2, nt=4)
    params = vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3,) + dims)
    vg, reps_g, _ = vr.parameter_continuation(c, mR, mT, v0, model, params)
    vref_, reps_r, _ = ref.parameter_continuation(mR, mT, v0, model, params)
    assert len(reps_g) == len(reps_r) == 3
    for a, b in zip(reps_g, reps_r):
        _compare(a, b)


def test_solve_report_csv_matches_reference(vr, ref, ctx):
    """SolveReport::write_csv (solver.cpp:29-47): the GPU solve's CSV has the reference's
    header and one row per iteration with the same integer columns (iter, inner iterations,
    cumulative matvecs / PDE solves) and the same floats to 1e-8 relative; wall time is the
    only column that differs by construction."""
    dims = (16, 16, 16)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model, params = vr.make_model("h2", beta_v=1e-2, nt=4), vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3,) + dims)
    res = vr.gauss_newton_solve(c, mR, mT, v0, model, params)
    cpu = ref.gauss_newton_solve_csv(mR, mT, v0, model, params)
    g_lines, r_lines = res.csv.strip().splitlines(), cpu.strip().splitlines()
    assert g_lines[0] == "# gpu" and r_lines[0] == "# reference"
    assert g_lines[1] == r_lines[1]  # header
    assert len(g_lines) == len(r_lines)
    cols = r_lines[1].split(",")
    for gl, rl in zip(g_lines[2:], r_lines[2:]):
        for name, a, b in zip(cols, gl.split(","), rl.split(",")):
            if name == "wall_time_s":
                continue
            if name in ("iter", "inner_iterations", "fine_matvecs", "coarse_matvecs", "pde_solves"):
                assert a == b, (name, a, b)
            else:
                fa, fb = float(a), float(b)
                assert abs(fa - fb) <= 1e-8 * max(abs(fb), 1e-300), (name, fa, fb)
