"""CPU-only: pin the oracle before trusting it.

1. The reference's own doctest suite (proj/tests, compiled unmodified against the
   FFTW/doctest shims into oracle/_ref) passes: this pins the FFTW shim and the
   compiled reference by the reference's known-answer and property tests.
2. The numpy restatement (oracle/veloreg_np.py) reproduces the golden vectors
   generated from the compiled reference (tests/golden/make_golden.py).
3. Where the compiled reference is present, the restatement matches it on
   fresh seeded inputs too.
"""
import os
import subprocess

import numpy as np
import pytest

from conftest import periodic_diff, rel_l2
from oracle import veloreg_np as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref")
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.mark.parametrize("suite", ["test_fields", "test_transport", "test_objective", "test_solver",
                                   "test_precond"])
def test_reference_suite_passes(suite):
    exe = os.path.join(REF_BIN, suite)
    if not os.path.exists(exe):
        pytest.skip("reference test binaries not built (make -C oracle tests)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout


def test_reference_postprocess_suite_known_failures():
    # 2 of the 7 postprocess cases fail with the reference's own tolerances:
    # test_postprocess.cpp:66 (det grad y vs the RK4/FD trajectory oracle: 1.38e-2 > 1e-2 at
    # 16^3, n_t = 4; 2.6e-3 at 32^3 -- discretisation error of the algorithm) and :142 (80
    # boundary voxels of two small balls flip under smoothing + arg-max at v = 0, bound 14).
    # Both reproduce identically on the GPU path, whose FFT is independent of the oracle's
    # FFTW shim (tests/test_gpu_postprocess.py::test_reference_postprocess_failures_are_not_
    # the_fft_shim), so they are not shim artefacts; pinned here
    exe = os.path.join(REF_BIN, "test_postprocess")
    if not os.path.exists(exe):
        pytest.skip("reference test binaries not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert "test cases: 7 | 5 passed | 2 failed" in r.stdout


@pytest.fixture(scope="module", params=["16", "8x16x32"])
def gold(request):
    return dict(np.load(os.path.join(GOLD, f"golden_{request.param}.npz")))


def test_np_fft_and_spectral_vs_golden(gold):
    f, v = gold["f"], gold["v"]
    assert rel_l2(O.fft_forward(f).view(np.float64), gold["fft_r2c"].view(np.float64)) < 1e-13
    assert rel_l2(O.gradient(f), gold["gradient"]) < 1e-12
    assert rel_l2(O.divergence(v), gold["divergence"]) < 1e-12
    assert rel_l2(O.laplacian(f), gold["laplacian"]) < 1e-12
    assert rel_l2(O.gaussian_smooth(f, (1.0, 2.0, 1.5)), gold["gaussian_1_2_1p5"]) < 1e-12
    for kind, nm in ((0, "h1"), (1, "h2"), (2, "h3"), (3, "helmholtz")):
        for mode, mn in ((0, "apply"), (1, "inverse"), (2, "inverse_sqrt")):
            out = O.apply_reg_operator(v, kind, mode, 3e-2, gamma=0.7)
            assert rel_l2(out, gold[f"reg_{nm}_{mn}"]) < 1e-12, (nm, mn)
    assert rel_l2(O.apply_projection(v, O.INCOMPRESSIBLE), gold["leray"]) < 1e-12
    assert rel_l2(O.apply_projection(v, O.NEAR_INCOMPRESSIBLE, 1e-3, 1e-4), gold["nearinc"]) < 1e-12


def test_np_transport_vs_golden(gold):
    assert rel_l2(O.tricubic_interpolate(gold["f"], gold["pts"]), gold["tricubic"]) < 1e-13
    mT, vs = gold["syn_mT"], gold["syn_v"]
    assert periodic_diff(O.trace_characteristics(vs, 4, "backward"), gold["trace_bwd"]).max() < 1e-13
    assert periodic_diff(O.trace_characteristics(vs, 4, "forward"), gold["trace_fwd"]).max() < 1e-13
    assert rel_l2(O.solve_state(mT, vs, 4), gold["state"]) < 1e-13


@pytest.mark.parametrize("name,kw", [("h2", dict()),
                                     ("h1div", dict(kind=O.H1, beta_v=1e-3, projection=O.NEAR_INCOMPRESSIBLE,
                                                    div_penalty=True))])
def test_np_objective_vs_golden(gold, name, kw):
    o = O.Objective(gold["syn_mR"], gold["syn_mT"], **kw)
    s = o.evaluate(0.5 * gold["syn_v"])
    J, mis, rel = gold[f"obj_{name}_J"]
    assert abs(s["objective"] - J) <= 1e-12 * abs(J)
    assert abs(s["mismatch"] - mis) <= 1e-12 * abs(mis)
    g = o.compute_gradient(s)
    assert rel_l2(g, gold[f"obj_{name}_grad"]) < 1e-11
    assert rel_l2(s["factor"], gold[f"obj_{name}_factor"]) < 1e-12
    assert rel_l2(o.hessian_matvec(s, gold["vt"]), gold[f"obj_{name}_matvec"]) < 1e-11
    assert o.counters["pde_solves"] == 4


def test_np_gn_solve_vs_golden(gold):
    res = O.gauss_newton_solve(gold["syn_mR"], gold["syn_mT"], np.zeros_like(gold["syn_v"]), dict(), eps_opt=1e-2)
    it, mis, grel, nmv, npde = gold["gn_report"]
    assert res["outer_iterations"] == int(it)
    assert abs(res["final_mismatch_rel"] - mis) <= 1e-6 * mis
    assert abs(res["final_grad_rel"] - grel) <= 1e-6 * grel
    assert [r["inner_iterations"] for r in res["records"]] == list(gold["gn_inner"])
    assert res["counters"]["hessian_matvecs"] == int(nmv) and res["counters"]["pde_solves"] == int(npde)
    assert rel_l2(res["v"], gold["gn_v"]) < 1e-9


def test_np_vs_compiled_reference_fresh_inputs(ref):
    shape = (16, 8, 16)
    f = ref.random_rough_scalar(shape, 99)
    v = ref.random_smooth_vector(shape, 2, 77, 0.6)
    assert rel_l2(O.gradient(f), ref.gradient(f)) < 1e-12
    assert rel_l2(O.solve_state(f, v, 3), ref.solve_state(f, v, 3)) < 1e-12
    hist = ref.solve_state(f, v, 4)
    vt = ref.random_smooth_vector(shape, 2, 78, 1.0)
    assert rel_l2(O.solve_inc_state(hist, v, vt, 4)[1:], ref.solve_inc_state(hist, v, vt, 4)[1:]) < 1e-11
    term = ref.random_smooth_scalar(shape, 2, 31, 1.0)
    init, hist_r = ref.solve_adjoint(term, v, 4, needs_history=True)
    assert rel_l2(O.solve_adjoint(term, v, 4), hist_r) < 1e-12


# ---- continuation restatements (oracle/ref_capi.cpp) ------------------
def _ref_or_skip():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref/libveloreg_ref.so not built (make -C oracle lib)")
    return ref


def _pods():
    from paper_1808_04487_b200 import _lib as L
    m = L.Model(L.RegNorm(L.REG_H2, 1.0, 1, 0, 1e-4), L.PROJ_IDENTITY, 1e-2, 4, 1)
    p = L.SolverParams(1e-2, 1e-6, 50, 100, 1e-4, 0.5, 20, 1)
    return L, m, p


def test_oracle_single_level_continuations_equal_plain_solve():
    ref = _ref_or_skip()
    L, m, p = _pods()
    dims = (16, 16, 16)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    v0 = np.zeros((3,) + dims)
    plain, rep, _ = ref.gauss_newton_solve(mR, mT, v0, m, p)
    vg, rg, _ = ref.grid_continuation(mR, mT, v0, 1, m, p)
    vs, rs, _ = ref.scale_continuation(mR, mT, v0, [0.0], m, p)
    assert np.array_equal(vg, plain) and np.array_equal(vs, plain)
    assert rg[0]["outer_iterations"] == rs[0]["outer_iterations"] == rep["outer_iterations"]


def test_oracle_grid_continuation_quality():
    # two levels 16^3 -> 32^3 end within 1.5x of the single-level mismatch
    ref = _ref_or_skip()
    L, m, p = _pods()
    dims = (32, 32, 32)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    v0 = np.zeros((3,) + dims)
    _, rep, _ = ref.gauss_newton_solve(mR, mT, v0, m, p)
    _, reps, _ = ref.grid_continuation(mR, mT, v0, 2, m, p)
    assert len(reps) == 2 and all(r["success"] for r in reps)
    assert reps[-1]["final_mismatch_rel"] <= 1.5 * rep["final_mismatch_rel"]


def test_oracle_beta_search_contract():
    ref = _ref_or_skip()
    L, m, p = _pods()
    dims = (16, 16, 16)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    v0 = np.zeros((3,) + dims)
    sp = L.BetaSearchParams(0.9, 1e-5, 1.0, 10, 0.25)
    beta, v, trials = ref.beta_search(mR, mT, v0, m, p, sp)
    assert trials[0]["beta"] == 1.0 and trials[0]["feasible"]
    assert trials[1]["beta"] == 1e-5 and not trials[1]["feasible"]
    feas = [t["beta"] for t in trials if t["feasible"]]
    assert beta == min(feas)
    infeas_above = [t["beta"] for t in trials if not t["feasible"] and t["beta"] > beta]
    assert not infeas_above  # monotone on this problem
    det = ref.det_deformation_gradient(v, 4)
    assert det.min() >= 0.9 and det.max() <= 1 / 0.9
    # m_T == m_R: the lower end
    b0, _, t0 = ref.beta_search(mT, mT, v0, m, p, sp)
    assert b0 == 1e-5 and len(t0) == 2
    # unreachable bound: error carrying the trace
    with pytest.raises(ref.RefError) as e:
        ref.beta_search(mR, mT, v0, m, p, L.BetaSearchParams(0.9999999, 1e-5, 1.0, 10, 0.25))
    assert len(e.value.trials) == 1


def test_exact_reg_operator_is_exact_on_pure_modes():
    # tests/exact.py (the long-double beta A the GPU and the reference are measured against):
    # on a pure mode cos(k.x) every mode of the symbol is known in closed form
    import numpy as np
    from exact import exact_reg
    n = 32
    x = np.arange(n, dtype=np.longdouble) * (2 * np.arccos(np.longdouble(-1)) / n)
    X1, X2, X3 = np.meshgrid(x, x, x, indexing="ij")  # long double: no fp64 input round-off
    for k, kind, p in (((3, -5, 7), "h2", 2), ((1, 2, 2), "h3", 3), ((0, 16, 0), "h1", 1)):
        f = np.cos(k[0] * X1 + k[1] * X2 + k[2] * X3)
        k2 = float(sum(a * a for a in k))
        out = exact_reg(f, kind, 1e-2, "apply")
        # long-double round-off of f (1e-19) amplified by the largest symbol on the grid
        smax = (3 * (n // 2) ** 2) ** p
        assert np.abs(out - 1e-2 * k2 ** p * f).max() <= max(1e-15 * 1e-2 * k2 ** p, 1e-18 * 1e-2 * smax)
        inv = exact_reg(f, kind, 1e-2, "inverse")
        assert np.abs(inv - f / (1e-2 * k2 ** p)).max() <= 1e-15 / (1e-2 * k2 ** p)


def test_exact_reg_vs_reference_round_off(ref):
    # the reference's fp64 beta A v sits at the |k|^4-amplified round-off distance from the
    # exact operator (the effect the GPU parity bar is built on): small at 32^3, growing ~n^4
    import numpy as np
    from exact import exact_reg, rel_err
    from paper_1808_04487_b200 import phantom
    errs = []
    for n in (16, 32, 64):
        v = phantom.bandlimited_velocity(n, 6, 0.5)
        e = rel_err(ref.apply_reg_operator(v, ref.make_norm("h2"), 0, 1e-2), exact_reg(v, "h2", 1e-2))
        errs.append(e)
        assert 0 < e < 1e-11
    assert errs[2] > errs[0]


def test_config3_solve_fixture():
    """tests/golden/config3_solve.npz (the reference's config-3 beta continuation, generated by
    tests/golden/make_config3_solve.py from the compiled reference): three levels, converged,
    the iteration counts the bench reports for the reference CPU arm."""
    import os
    import numpy as np
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "config3_solve.npz"))
    assert int(g["n"]) == 256 and int(g["levels"]) == 3
    assert g["v_sub8"].shape == (3, 32, 32, 32) and g["m_R_sub8"].shape == (32, 32, 32)
    assert [int(x) for x in g["outer_iterations"]] == [1, 3, 3]
    assert 0.5 < float(g["final_mismatch_rel"][-1]) < 0.6 and float(g["final_grad_rel"][-1]) < 0.1
    assert np.isfinite(g["v_sub8"]).all() and float(g["v_norm"]) > 0
