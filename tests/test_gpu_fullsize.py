"""GPU parity and size-independent properties at BASELINE's full single-GPU sizes.

* config 3 (256^3, the bench workload): one evaluate + reduced gradient + GN
  Hessian matvec (at half the generating velocity) against the compiled reference run on the host cores (the
  reference's own objective.cpp:47-156 on the same arrays), relative L2 <= 1e-10.
* config 3 and config 4 (512^3 on one GPU): size-independent properties of the
  GN Hessian -- linearity, symmetry of the Gauss-Newton operator in the weighted
  inner product (test_objective.cpp:186-215), positive semi-definiteness, zero in
  -> zero out -- and of the spectral layer (FFT round trip, A^-1 A = I on
  mean-free fields, spectral.cpp:166-184).
Inputs are the seeded synthetic phantoms of BASELINE configs 3/4
(paper_1808_04487_b200/phantom.py); they stand in for the paper's MRI data.
"""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _inputs(vr, ctx, config):
    from paper_1808_04487_b200 import phantom
    n = phantom.CONFIGS[config]["n"]
    m_T, v = phantom.make_config_inputs(config)
    c = ctx(n)
    m_R = np.asarray(vr.solve_state(c, m_T, v, 4))[4]  # m_T transported by v (config definition)
    return c, n, m_R, m_T, v


def test_config3_reference_parity(vr, ref, ctx):
    """Data parts at 1e-10. The beta_v A terms are compared at 2e-9: the H2 symbol |k|^4
    reaches (128 sqrt 3)^4 ~ 2.4e9 at 256^3, so the O(1e-16) round-off two correct fp64
    FFTs leave in the empty high modes of a band-limited field is amplified to ~1e-10 of
    ||beta A v|| (measured 1.9e-10; 2e-15 at v = 0 where the term vanishes)."""
    from paper_1808_04487_b200 import phantom
    c, n, m_R, m_T, v = _inputs(vr, ctx, 3)
    vt = phantom.bandlimited_direction(n)
    model = vr.make_model()
    o = vr.Objective(c, m_R, m_T, model)
    v_eval = 0.5 * v  # halfway to the generating velocity: non-trivial mismatch and adjoint
    s = o.evaluate(v_eval)
    o.compute_gradient(s)
    hv = o.hessian_matvec(s, vt)
    hdv = o.hessian_data_matvec(s, vt)
    ro = ref.Objective(m_R, m_T, model)
    rs = ro.evaluate(v_eval)
    g_ref = ro.compute_gradient(rs)
    hv_ref = ro.hessian_matvec(rs, vt)
    hdv_ref = ro.hessian_data_matvec(rs, vt)
    sc = rs.scalars()
    assert abs(s.objective - sc["objective"]) <= 1e-12 * abs(sc["objective"])
    assert abs(s.mismatch_rel - sc["mismatch_rel"]) <= 1e-12 * abs(sc["mismatch_rel"])
    reg = np.asarray(vr.apply_reg_operator(c, v_eval, model.norm, "apply", model.beta_v))
    reg_ref = ref.apply_reg_operator(v_eval, model.norm, 0, model.beta_v)
    assert rel_l2(s.gradient - reg, g_ref - reg_ref) <= 1e-10
    assert rel_l2(reg, reg_ref) <= 2e-9
    assert rel_l2(s.gradient, g_ref) <= 2e-9
    assert rel_l2(hdv, hdv_ref) <= 1e-10
    assert rel_l2(hv, hv_ref) <= 2e-9
    assert o.counters()["pde_solves"] == ro.counters()["pde_solves"]


def _probe(n, seed):
    from paper_1808_04487_b200 import phantom
    return phantom.bandlimited_direction(n, kmax_inf=3, seed=seed)


@pytest.mark.parametrize("config", [3, 4])
def test_fullsize_gn_properties(vr, ctx, config):
    """test_objective.cpp:186-215 at full size: exact symmetry / PSD at v = 0 (1e-6), the
    O(discretization) optimize-then-discretize asymmetry at a generic v (< 5e-3, the
    reference's bound); linearity of the data matvec to round-off (the beta_v A term
    at the conditioning-scaled 2e-9 (n/256)^4 of test_config3_reference_parity)."""
    c, n, m_R, m_T, v = _inputs(vr, ctx, config)
    o = vr.Objective(c, m_R, m_T, vr.make_model())
    u, w = c.to_device(_probe(n, 7)), c.to_device(_probe(n, 8))
    for v_eval, sym_tol in ((np.zeros_like(v), 1e-6), (0.5 * v, 5e-3)):
        s = o.evaluate(v_eval)
        o.compute_gradient(s)
        assert np.isfinite(s.objective) and 0.0 < s.mismatch_rel <= 1.0
        Hu, Hw = o.hessian_matvec(s, u), o.hessian_matvec(s, w)
        a, b = vr.inner_product(c, Hu, w), vr.inner_product(c, u, Hw)
        assert abs(a - b) <= sym_tol * max(abs(a), abs(b))
        assert vr.inner_product(c, Hu, u) > 0.0
    # linearity: H(2u - 3w) = 2 Hu - 3 Hw
    comb = c.to_device(2.0 * u.numpy() - 3.0 * w.numpy())
    lhs = o.hessian_data_matvec(s, comb).numpy()
    rhs = 2.0 * o.hessian_data_matvec(s, u).numpy() - 3.0 * o.hessian_data_matvec(s, w).numpy()
    assert rel_l2(lhs, rhs) <= 1e-12
    lhs = o.hessian_matvec(s, comb).numpy()
    rhs = 2.0 * Hu.numpy() - 3.0 * Hw.numpy()
    assert rel_l2(lhs, rhs) <= 2e-9 * (n / 256) ** 4  # |k|^4 amplification grows as n^4
    # zero in -> zero out
    z = c.to_device(np.zeros((3, n, n, n)))
    assert vr.max_abs(c, o.hessian_matvec(s, z)) == 0.0


@pytest.mark.parametrize("config", [3, 4])
def test_fullsize_spectral_round_trips(vr, ctx, config):
    from paper_1808_04487_b200 import phantom
    n = phantom.CONFIGS[config]["n"]
    c = ctx(n)
    f = _probe(n, 11)
    spec = vr.fft_forward(c, c.to_device(f[0]))
    back = vr.fft_inverse(c, spec)
    assert rel_l2(np.asarray(back.numpy() if hasattr(back, "numpy") else back), f[0]) <= 1e-13
    model = vr.make_model()
    au = vr.apply_reg_operator(c, c.to_device(f), model.norm, "apply", model.beta_v)
    rt = vr.apply_reg_operator(c, au, model.norm, "inverse", model.beta_v)
    fm = f - f.mean(axis=(1, 2, 3), keepdims=True)  # A^-1 maps the zero mode to itself / beta
    rtn = rt.numpy() if hasattr(rt, "numpy") else rt
    rtm = rtn - rtn.mean(axis=(1, 2, 3), keepdims=True)
    assert rel_l2(rtm, fm) <= 1e-11


@pytest.mark.skipif(not __import__("os").environ.get("VR_FULLSIZE_512"),
                    reason="~10 min of reference CPU time and ~90 GB host RAM; set VR_FULLSIZE_512=1")
def test_config4_reference_parity(vr, ref, ctx):
    """Config 4 (512^3) on one GPU against the reference on the host cores: one evaluate +
    gradient + data matvec (same bars as config 3; run on demand, result in DESIGN.md)."""
    from paper_1808_04487_b200 import phantom
    c, n, m_R, m_T, v = _inputs(vr, ctx, 4)
    vt = phantom.bandlimited_direction(n)
    model = vr.make_model()
    o = vr.Objective(c, m_R, m_T, model)
    v_eval = 0.5 * v
    s = o.evaluate(v_eval)
    o.compute_gradient(s)
    g, hdv = s.gradient, o.hessian_data_matvec(s, vt)
    ro = ref.Objective(m_R, m_T, model)
    rs = ro.evaluate(v_eval)
    g_ref = ro.compute_gradient(rs)
    hdv_ref = ro.hessian_data_matvec(rs, vt)
    sc = rs.scalars()
    reg = np.asarray(vr.apply_reg_operator(c, v_eval, model.norm, "apply", model.beta_v))
    reg_ref = ref.apply_reg_operator(v_eval, model.norm, 0, model.beta_v)
    errs = {"objective": abs(s.objective - sc["objective"]) / abs(sc["objective"]),
            "gradient_data": rel_l2(g - reg, g_ref - reg_ref), "reg": rel_l2(reg, reg_ref),
            "data_matvec": rel_l2(hdv, hdv_ref)}
    print("config4 parity", errs)
    assert errs["objective"] <= 1e-12
    assert errs["gradient_data"] <= 1e-10 and errs["data_matvec"] <= 1e-10
    assert errs["reg"] <= 2e-9 * (n / 256) ** 4


@pytest.mark.skipif(not __import__("os").environ.get("VR_FULLSIZE_SOLVE"),
                    reason="~10 min of reference CPU time; set VR_FULLSIZE_SOLVE=1")
def test_config3_solve_vs_reference(vr, ref, ctx):
    """Config 3 end to end: beta continuation 1 -> 1e-1 -> 1e-2 on the GPU
    and in the reference on the host cores; per level Newton iterations +-1, final mismatch
    and gradient norm within 1 % (BASELINE north star). On demand; result in DESIGN.md."""
    c, n, m_R, m_T, v = _inputs(vr, ctx, 3)
    model, params = vr.make_model(), vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3, n, n, n))
    vg, rg, _ = vr.parameter_continuation(c, m_R, m_T, v0, model, params)
    vref, rr, _ = ref.parameter_continuation(m_R, m_T, v0, model, params)
    print("config3 solve GPU", [(r["outer_iterations"], r["final_mismatch_rel"], r["final_grad_rel"]) for r in rg])
    print("config3 solve REF", [(r["outer_iterations"], r["final_mismatch_rel"], r["final_grad_rel"]) for r in rr])
    print("config3 solve v rel", rel_l2(vg, vref))
    assert len(rg) == len(rr)
    for a, b in zip(rg, rr):
        assert abs(a["outer_iterations"] - b["outer_iterations"]) <= 1
    assert abs(rg[-1]["final_mismatch_rel"] - rr[-1]["final_mismatch_rel"]) <= 1e-2 * rr[-1]["final_mismatch_rel"]
    assert abs(rg[-1]["final_grad_rel"] - rr[-1]["final_grad_rel"]) <= 1e-2 * rr[-1]["final_grad_rel"]
