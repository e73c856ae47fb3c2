"""GPU vs the committed golden vectors (generated from the compiled reference by
tests/golden/make_golden.py) -- runs even where the reference sources are absent."""
import os

import numpy as np
import pytest

from conftest import periodic_diff, rel_l2

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-10


@pytest.fixture(scope="module", params=["16", "8x16x32"])
def gold(request):
    return dict(np.load(os.path.join(GOLD, f"golden_{request.param}.npz")))


def test_gpu_operators_vs_golden(vr, ctx, gold):
    f, v = gold["f"], gold["v"]
    c = ctx(f.shape)
    assert rel_l2(vr.fft_forward(c, f).view(np.float64), gold["fft_r2c"].view(np.float64)) < 1e-13
    assert rel_l2(vr.gradient(c, f), gold["gradient"]) < TOL
    assert rel_l2(vr.divergence(c, v), gold["divergence"]) < TOL
    assert rel_l2(vr.laplacian(c, f), gold["laplacian"]) < TOL
    assert rel_l2(vr.gaussian_smooth(c, f, (1.0, 2.0, 1.5)), gold["gaussian_1_2_1p5"]) < TOL
    for kind in ("h1", "h2", "h3", "helmholtz"):
        n = vr.make_norm(kind, gamma=0.7)
        for mode in ("apply", "inverse", "inverse_sqrt"):
            assert rel_l2(vr.apply_reg_operator(c, v, n, mode, 3e-2), gold[f"reg_{kind}_{mode}"]) < TOL
    assert rel_l2(vr.apply_projection(c, v, "incompressible"), gold["leray"]) < TOL
    assert rel_l2(vr.apply_projection(c, v, "near_incompressible", 1e-3, 1e-4), gold["nearinc"]) < TOL
    assert rel_l2(vr.tricubic_interpolate(c, f, gold["pts"]), gold["tricubic"]) < TOL
    assert periodic_diff(vr.trace_characteristics(c, gold["syn_v"], 4, "backward"), gold["trace_bwd"]).max() < 1e-12
    assert periodic_diff(vr.trace_characteristics(c, gold["syn_v"], 4, "forward"), gold["trace_fwd"]).max() < 1e-12
    assert rel_l2(vr.solve_state(c, gold["syn_mT"], gold["syn_v"], 4), gold["state"]) < TOL


@pytest.mark.parametrize("name,kw", [("h2", dict()),
                                     ("h1div", dict(kind="h1", beta_v=1e-3, projection="near_incompressible",
                                                    div_penalty=True))])
def test_gpu_objective_vs_golden(vr, ctx, gold, name, kw):
    c = ctx(gold["syn_mR"].shape)
    o = vr.Objective(c, gold["syn_mR"], gold["syn_mT"], vr.make_model(**kw))
    s = o.evaluate(0.5 * gold["syn_v"])
    J, mis, rel = gold[f"obj_{name}_J"]
    assert abs(s.objective - J) <= 1e-10 * abs(J)
    o.compute_gradient(s)
    assert rel_l2(s.gradient, gold[f"obj_{name}_grad"]) < TOL
    assert rel_l2(o.hessian_matvec(s, gold["vt"]), gold[f"obj_{name}_matvec"]) < TOL


def test_gpu_gn_solve_vs_golden(vr, ctx, gold):
    c = ctx(gold["syn_mR"].shape)
    res = vr.gauss_newton_solve(c, gold["syn_mR"], gold["syn_mT"], np.zeros_like(gold["syn_v"]),
                                vr.make_model(), vr.make_params(eps_opt=1e-2))
    it, mis, grel, nmv, npde = gold["gn_report"]
    assert abs(res.report["outer_iterations"] - int(it)) <= 1
    assert abs(res.report["final_mismatch_rel"] - mis) <= 1e-2 * mis
    assert abs(res.report["final_grad_rel"] - grel) <= 1e-2 * grel
