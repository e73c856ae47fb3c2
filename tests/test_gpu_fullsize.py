"""GPU parity and size-independent properties at BASELINE's full single-GPU sizes.

* config 3 (256^3, the bench workload): one evaluate + reduced gradient + GN
  Hessian matvec (at half the generating velocity) against the compiled reference run on
  the host cores (the reference's own objective.cpp:47-156 on the same arrays): data parts
  relative L2 <= 1e-10; the beta_v A terms against the exact (long-double) operator, GPU
  error <= 1.5x the reference's (tests/exact.py).
* the regularisation operator in all three modes at 256^3 and 512^3 against exact.
* config 2 (128^3) full solve (reference live on the host cores) and config 3 (256^3)
  beta-continuation solve (reference results from the committed fixture
  tests/golden/config3_solve.npz; live with VR_LIVE_CONFIG3=1): Newton iterations +-1,
  final mismatch and gradient within 1 %.
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
    """Config 3 (the bench workload) against the reference on the host cores and against the
    exact answer. Data parts (state, mismatch, the adjoint/incremental sweeps) GPU vs
    reference at 1e-10. The beta_v A terms (proj/src/spectral.cpp:166-184) are measured
    against beta_v A evaluated in long double on the same input (tests/exact.py): the H2
    symbol |k|^4 reaches (128 sqrt 3)^4 ~ 2.4e9 at 256^3 and amplifies the round-off of any
    fp64 FFT pair to ~1e-10 of ||beta A v||, the reference's included (measured: 1.4e-10 vs
    exact). Bar: the GPU's error against exact is at most 1.5x the reference's."""
    from exact import exact_reg, no_worse_than_reference, rel_err, sampled_max_err
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
    reg_ex = exact_reg(v_eval, "h2", model.beta_v)
    vt_ex = exact_reg(vt, "h2", model.beta_v)
    # data parts: GPU vs reference
    assert rel_l2(s.gradient - reg, g_ref - reg_ref) <= 1e-10
    assert rel_l2(hdv, hdv_ref) <= 1e-10
    # beta_v A terms vs exact: the operator itself, the gradient (data part + beta_v A v) and
    # the full matvec (data part + beta_v A vt), each GPU vs reference error against exact
    g_ex = (g_ref - reg_ref) + reg_ex
    hv_ex = hdv_ref + vt_ex
    errs = {"reg": (rel_err(reg, reg_ex), rel_err(reg_ref, reg_ex)),
            "gradient": (rel_err(s.gradient, g_ex), rel_err(g_ref, g_ex)),
            "matvec": (rel_err(hv, hv_ex), rel_err(hv_ref, hv_ex)),
            "reg_sampled_max": (sampled_max_err(reg, reg_ex), sampled_max_err(reg_ref, reg_ex))}
    print("config3 (gpu, reference) error vs exact:", errs)
    for k, (eg, er) in errs.items():
        assert no_worse_than_reference(eg, er), (k, eg, er)
    assert o.counters()["pde_solves"] == ro.counters()["pde_solves"]


@pytest.mark.parametrize("config", [3, 4])
def test_fullsize_reg_operator_vs_exact(vr, ref, ctx, config):
    """beta_v A, (beta_v A)^-1 and (beta_v A)^-1/2 (spectral.cpp:166-184; H2, beta 1e-2) of
    the config's velocity and of the matvec probe at 256^3, and beta_v A of both at 512^3
    (the |k|^4-amplified mode; the inverse modes sit at 2-3e-16 on both sides): GPU and
    reference errors against the long-double answer (tests/exact.py); GPU <= 1.5x reference."""
    from exact import exact_reg, no_worse_than_reference, rel_err
    from paper_1808_04487_b200 import phantom
    n = phantom.CONFIGS[config]["n"]
    c = ctx(n)
    cfg = phantom.CONFIGS[config]
    norm = vr.make_norm("h2")
    modes = (("apply", 0), ("inverse", 1), ("inverse_sqrt", 2)) if n <= 256 else (("apply", 0),)
    for name, f in (("v", phantom.bandlimited_velocity(n, cfg["kmax"], cfg["disp"])),
                    ("vt", phantom.bandlimited_direction(n))):
        if n > 256:
            f = f[:1]  # one component: the operator acts per component
        for mode, code in modes:
            ex = exact_reg(f, "h2", 1e-2, mode)
            full = np.concatenate([f, f, f]) if f.shape[0] == 1 else f
            eg = rel_err(np.asarray(vr.apply_reg_operator(c, full, norm, mode, 1e-2))[: f.shape[0]], ex)
            er = rel_err(ref.apply_reg_operator(full, norm, code, 1e-2)[: f.shape[0]], ex)
            print(f"config{config} {name} {mode}: gpu {eg:.3e} reference {er:.3e}")
            assert no_worse_than_reference(eg, er), (name, mode, eg, er)
            del ex


def _probe(n, seed):
    from paper_1808_04487_b200 import phantom
    return phantom.bandlimited_direction(n, kmax_inf=3, seed=seed)


@pytest.mark.parametrize("config", [3, 4])
def test_fullsize_gn_properties(vr, ctx, config):
    """test_objective.cpp:186-215 at full size: exact symmetry / PSD at v = 0 (1e-6), the
    O(discretization) optimize-then-discretize asymmetry at a generic v (< 5e-3, the
    reference's bound); linearity of the data matvec to round-off and of the full matvec
    within the measured exact-operator error of its beta_v A term (256^3; at 512^3 the
    exact operator's cost keeps that check to test_fullsize_reg_operator_vs_exact)."""
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
    # linearity: H(2u - 3w) = 2 Hu - 3 Hw. The data matvec to round-off; the full matvec up to
    # its beta_v A term's measured distance from the exact (long-double) operator, which is
    # linear: |D| <= |D_data| + e(2u - 3w) + 2 e(u) + 3 e(w), e(x) = ||beta A_gpu x - beta A x||
    from exact import exact_reg
    comb = c.to_device(2.0 * u.numpy() - 3.0 * w.numpy())
    lhs = o.hessian_data_matvec(s, comb).numpy()
    rhs = 2.0 * o.hessian_data_matvec(s, u).numpy() - 3.0 * o.hessian_data_matvec(s, w).numpy()
    assert rel_l2(lhs, rhs) <= 1e-12
    # zero in -> zero out
    z = c.to_device(np.zeros((3, n, n, n)))
    assert vr.max_abs(c, o.hessian_matvec(s, z)) == 0.0
    if n > 256:  # the exact-operator bound below costs ~1 min of long-double FFTs at 512^3
        return
    d_data = np.linalg.norm((lhs - rhs).ravel())
    bound = d_data
    for x, k in ((comb, 1.0), (u, 2.0), (w, 3.0)):
        xa = x.numpy()
        gx = np.asarray(vr.apply_reg_operator(c, x, vr.make_norm("h2"), "apply", 1e-2).numpy())
        bound += k * float(np.sqrt(((gx - exact_reg(xa, "h2", 1e-2)) ** 2).sum()))
    lhs = o.hessian_matvec(s, comb).numpy()
    rhs = 2.0 * Hu.numpy() - 3.0 * Hw.numpy()
    assert np.linalg.norm((lhs - rhs).ravel()) <= 1.01 * bound + 1e-14 * np.linalg.norm(rhs.ravel())


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
    from exact import exact_reg, no_worse_than_reference, rel_err
    reg = np.asarray(vr.apply_reg_operator(c, v_eval, model.norm, "apply", model.beta_v))
    reg_ref = ref.apply_reg_operator(v_eval, model.norm, 0, model.beta_v)
    reg_ex = exact_reg(v_eval, "h2", model.beta_v)
    errs = {"objective": abs(s.objective - sc["objective"]) / abs(sc["objective"]),
            "gradient_data": rel_l2(g - reg, g_ref - reg_ref), "data_matvec": rel_l2(hdv, hdv_ref),
            "reg_vs_exact": (rel_err(reg, reg_ex), rel_err(reg_ref, reg_ex))}
    print("config4 parity", errs)
    assert errs["objective"] <= 1e-12
    assert errs["gradient_data"] <= 1e-10 and errs["data_matvec"] <= 1e-10
    assert no_worse_than_reference(*errs["reg_vs_exact"])


def _check_solve_levels(rg, ref_iters, ref_mismatch, ref_grad):
    assert len(rg) == len(ref_iters)
    for a, it in zip(rg, ref_iters):
        assert abs(a["outer_iterations"] - int(it)) <= 1
    assert abs(rg[-1]["final_mismatch_rel"] - ref_mismatch[-1]) <= 1e-2 * ref_mismatch[-1]
    assert abs(rg[-1]["final_grad_rel"] - ref_grad[-1]) <= 1e-2 * ref_grad[-1]


def test_config3_solve_vs_reference(vr, ref, ctx):
    """Config 3 end to end: beta continuation 1 -> 1e-1 -> 1e-2 on the GPU
    against the reference's own solve of the same arrays (proj/src/solver.cpp:154-269): per
    level Newton iterations +-1, final mismatch and gradient norm within 1 % (BASELINE north
    star), final velocity equal on the stored sub-grid. The reference solve takes ~6.5 min on
    16 host cores, so its results are the committed fixture tests/golden/config3_solve.npz
    (tests/golden/make_config3_solve.py, generated from the compiled reference);
    VR_LIVE_CONFIG3=1 also runs the reference live on this box's host cores."""
    import os
    c, n, m_R, m_T, v = _inputs(vr, ctx, 3)
    model, params = vr.make_model(), vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3, n, n, n))
    vg, rg, _ = vr.parameter_continuation(c, m_R, m_T, v0, model, params)
    print("config3 solve GPU", [(r["outer_iterations"], r["final_mismatch_rel"], r["final_grad_rel"]) for r in rg])
    gold = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "config3_solve.npz"))
    print("config3 solve REF (fixture)", list(zip(gold["outer_iterations"], gold["final_mismatch_rel"],
                                                  gold["final_grad_rel"])))
    # same problem: the reference's transported image equals the GPU's on the stored sub-grid
    assert rel_l2(m_R[::8, ::8, ::8], gold["m_R_sub8"]) <= 1e-10
    _check_solve_levels(rg, gold["outer_iterations"], gold["final_mismatch_rel"], gold["final_grad_rel"])
    for a, st in zip(rg, gold["stop"]):
        assert a["stop"] == int(st)
    dv = rel_l2(vg[:, ::8, ::8, ::8], gold["v_sub8"])
    print("config3 solve v rel (sub-grid)", dv)
    assert dv <= 1e-8
    assert abs(np.linalg.norm(vg.ravel()) - float(gold["v_norm"])) <= 1e-8 * float(gold["v_norm"])
    if os.environ.get("VR_LIVE_CONFIG3"):
        vref, rr, _ = ref.parameter_continuation(m_R, m_T, v0, model, params)
        print("config3 solve REF (live)", [(r["outer_iterations"], r["final_mismatch_rel"], r["final_grad_rel"]) for r in rr])
        print("config3 solve v rel", rel_l2(vg, vref))
        _check_solve_levels(rg, [r["outer_iterations"] for r in rr], [r["final_mismatch_rel"] for r in rr],
                            [r["final_grad_rel"] for r in rr])
        assert rel_l2(vg, vref) <= 1e-8


def test_config2_solve_vs_reference(vr, ref, ctx):
    """Config 2 (128^3 section-4.2 problem, proj/src/synthetic.cpp:16-34): full GN-Krylov
    solve on the GPU and in the reference; Newton iterations +-1, final mismatch and gradient
    norm within 1 %, same stop reason (proj/src/solver.cpp:154-269)."""
    n = 128
    c = ctx(n)
    m_R, m_T, _ = ref.generate_synthetic((n, n, n), 4)
    model, params = vr.make_model(), vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3, n, n, n))
    res = vr.gauss_newton_solve(c, m_R, m_T, v0, model, params)
    vref, rr, _ = ref.gauss_newton_solve(m_R, m_T, v0, model, params)
    rg = res.report
    print("config2 solve GPU", rg["outer_iterations"], rg["final_mismatch_rel"], rg["final_grad_rel"],
          "REF", rr["outer_iterations"], rr["final_mismatch_rel"], rr["final_grad_rel"])
    assert rg["stop"] == rr["stop"]
    assert abs(rg["outer_iterations"] - rr["outer_iterations"]) <= 1
    assert abs(rg["final_mismatch_rel"] - rr["final_mismatch_rel"]) <= 1e-2 * rr["final_mismatch_rel"]
    assert abs(rg["final_grad_rel"] - rr["final_grad_rel"]) <= 1e-2 * rr["final_grad_rel"]
    assert rel_l2(res.v, vref) <= 1e-6
