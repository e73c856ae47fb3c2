"""GPU parity: Objective (evaluate / reduced gradient / GN Hessian matvec) vs the compiled reference.

Reference: proj/src/objective.cpp:35-186, tests proj/tests/test_objective.cpp.
Per-operator bar: relative L2 <= 1e-10 (fp64).
"""
import numpy as np
import pytest

from conftest import rel_l2
from exact import no_worse_than_reference, rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-10

MODELS = {
    "h2_default": dict(kind="h2", beta_v=1e-2, nt=4),
    "h1div_nearinc": dict(kind="h1", beta_v=1e-3, nt=4, div_penalty=True, beta_w=1e-4,
                          projection="near_incompressible"),
    "h1_leray": dict(kind="h1", beta_v=1e-2, nt=4, projection="incompressible"),
    "helmholtz": dict(kind="helmholtz", gamma=0.5, beta_v=5e-2, nt=2),
    "h3_nt8": dict(kind="h3", beta_v=1e-3, nt=8),
    "h2_nt1": dict(kind="h2", beta_v=1e-2, nt=1),
}


def exact_reg_of(kw):
    """beta_v A^{1,-1,-1/2} of the model in long double (tests/exact.py)."""
    from exact import exact_reg

    def f(u, mode):
        return exact_reg(u, kw.get("kind", "h2"), kw["beta_v"], mode, kw.get("gamma", 1.0))
    return f


def image_pair(ref, dims, max_mode, seed):
    # test_objective.cpp:22-33
    a = 0.5 + ref.random_smooth_scalar(dims, max_mode, seed, 0.3)
    b = 0.5 + ref.random_smooth_scalar(dims, max_mode, seed + 1, 0.3)
    return a, b


@pytest.mark.parametrize("name", list(MODELS))
@pytest.mark.parametrize("dims", [(16, 16, 16), (32, 16, 32), (8, 32, 64), (64, 8, 16)])
def test_objective_parity(vr, ref, ctx, name, dims):
    c = ctx(dims)
    kw = MODELS[name]
    model = vr.make_model(**kw)
    mR, mT = image_pair(ref, dims, 2, 91)
    v = ref.random_smooth_vector(dims, 2, 120, 0.3)
    if kw.get("projection") == "incompressible":
        v = ref.apply_projection(v, 1)
    vt = ref.random_smooth_vector(dims, 2, 142, 1.0)

    ro = ref.Objective(mR, mT, model)
    go = vr.Objective(c, mR, mT, model)
    assert abs(go.initial_mismatch() - ro.initial_mismatch()) <= 1e-12 * ro.initial_mismatch()

    rs = ro.evaluate(v)
    gs = go.evaluate(v)
    sc = rs.scalars()
    assert abs(gs.objective - sc["objective"]) <= 1e-10 * abs(sc["objective"])
    assert abs(gs.mismatch - sc["mismatch"]) <= 1e-10 * abs(sc["mismatch"])
    assert abs(gs.mismatch_rel - sc["mismatch_rel"]) <= 1e-10 * abs(sc["mismatch_rel"])
    assert rel_l2(gs.m_history, rs.get(4)) < TOL

    g_ref = ro.compute_gradient(rs)
    go.compute_gradient(gs)
    assert gs.has_gradient and gs.has_adjoint_ctx
    assert rel_l2(gs.get(3), rs.get(3)) < TOL  # continuity factor
    hv, hv_ref = go.hessian_matvec(gs, vt), ro.hessian_matvec(rs, vt)
    hd, hd_ref = go.hessian_data_matvec(gs, vt), ro.hessian_data_matvec(rs, vt)
    assert rel_l2(hd, hd_ref) < TOL
    # beta_v A terms (gradient = K b + beta_v A v, matvec = H_data vt + beta_v A vt,
    # objective.cpp:104-121) against the long-double operator: GPU error <= 1.5x the
    # reference's (tests/exact.py; the |k|^p symbol amplifies fp64 FFT round-off)
    reg_v = ref.apply_reg_operator(v, model.norm, 0, model.beta_v)
    assert rel_l2(gs.gradient - np.asarray(vr.apply_reg_operator(c, v, model.norm, "apply", model.beta_v)),
                  g_ref - reg_v) < TOL
    ex = exact_reg_of(kw)
    g_ex = (g_ref - reg_v) + ex(v, "apply")
    hv_ex = hd_ref + ex(vt, "apply")
    assert no_worse_than_reference(rel_err(gs.gradient, g_ex), rel_err(g_ref, g_ex))
    assert no_worse_than_reference(rel_err(hv, hv_ex), rel_err(hv_ref, hv_ex))
    for mode in (0, 1, 2):
        name = ("apply", "inverse", "inverse_sqrt")[mode]
        e = ex(vt, name)
        assert no_worse_than_reference(rel_err(go.apply_reg(vt, mode), e), rel_err(ro.apply_reg(vt, mode), e))
        if mode:
            assert rel_l2(go.apply_reg(vt, mode), ro.apply_reg(vt, mode)) < TOL
    assert rel_l2(go.apply_K(vt), ro.apply_K(vt)) < TOL
    assert go.counters() == ro.counters()


def test_counters_and_pure_reg_limit(vr, ref, ctx):
    # test_objective.cpp:160-184
    dims = (16, 16, 16)
    c = ctx(dims)
    m = np.full(dims, 0.5)
    model = vr.make_model("h2", beta_v=2.5e-3, nt=4)
    o = vr.Objective(c, m, m, model)
    s = o.evaluate(np.zeros((3,) + dims))
    o.compute_gradient(s)
    assert o.counters()["pde_solves"] == 2
    vt = ref.random_smooth_vector(dims, 2, 90, 1.0)
    hv = o.hessian_matvec(s, vt)
    assert o.counters()["pde_solves"] == 4
    reg = vr.apply_reg_operator(c, vt, model.norm, "apply", model.beta_v)
    assert np.abs(hv - reg).max() < 1e-14
    assert np.abs(o.hessian_matvec(s, np.zeros((3,) + dims))).max() == 0.0


def test_gn_symmetry_psd(vr, ref, ctx):
    # test_objective.cpp:186-215 on the GPU path
    dims = (16, 16, 16)
    c = ctx(dims)
    mR, mT = image_pair(ref, dims, 2, 91)
    o = vr.Objective(c, mR, mT, vr.make_model("h2", beta_v=1e-3, nt=4))
    s0 = o.evaluate(np.zeros((3,) + dims))
    o.compute_gradient(s0)
    for probe in range(3):
        u = ref.random_smooth_vector(dims, 2, 100 + 2 * probe, 1.0)
        w = ref.random_smooth_vector(dims, 2, 101 + 2 * probe, 1.0)
        Hu, Hw = o.hessian_matvec(s0, u), o.hessian_matvec(s0, w)
        a, b = vr.inner_product(c, Hu, w), vr.inner_product(c, u, Hw)
        assert abs(a - b) / max(abs(a), abs(b)) < 1e-6
        q = vr.inner_product(c, Hu, u)
        assert q >= -1e-10 * max(1.0, abs(q))


def test_objective_errors(vr, ref, ctx):
    dims = (16, 16, 16)
    c = ctx(dims)
    mR, mT = image_pair(ref, dims, 2, 51)
    o = vr.Objective(c, mR, mT, vr.make_model())
    v = np.zeros((3,) + dims)
    v[1, 0, 0, 7] = np.nan
    with pytest.raises(vr.NumericError):
        o.evaluate(v)
    s = o.evaluate(np.zeros((3,) + dims))
    with pytest.raises(vr.LogicError):
        o.hessian_matvec(s, np.ones((3,) + dims))
    o.compute_gradient(s)
    bad = np.ones((3,) + dims)
    bad[2, 1, 1, 1] = np.inf
    with pytest.raises(vr.NumericError):
        o.hessian_matvec(s, bad)
    with pytest.raises(vr.ArgumentError):
        vr.Objective(c, mR, mT, vr.make_model(beta_v=-1.0))


def test_matvec_host_entry(vr, ref, ctx):
    dims = (32, 32, 32)
    c = ctx(dims)
    mR, mT, vs = ref.generate_synthetic(dims, 4)
    model = vr.make_model()
    o = vr.Objective(c, mR, mT, model)
    s = o.evaluate(vs)
    o.compute_gradient(s)
    vt = ref.random_smooth_vector(dims, 2, 142, 1.0)
    out = np.empty_like(vt)
    o.hessian_matvec_host(s, vt, out)
    ro = ref.Objective(mR, mT, model)
    rs = ro.evaluate(vs)
    ro.compute_gradient(rs)
    assert rel_l2(out, ro.hessian_matvec(rs, vt)) < TOL


def test_matvec_host_async_pipeline(vr, ref, ctx):
    # vr_hessian_matvec_host_async: a stream of independent directions through two
    # device slots equals the synchronous call for each of them, bit for bit
    dims = (32, 32, 32)
    c = ctx(dims)
    mR, mT, vs = ref.generate_synthetic(dims, 4)
    o = vr.Objective(c, mR, mT, vr.make_model())
    s = o.evaluate(0.5 * vs)
    o.compute_gradient(s)
    dirs = [ref.random_smooth_vector(dims, 2, 300 + k, 1.0) for k in range(5)]
    outs = [np.empty_like(d) for d in dirs]
    for d, out in zip(dirs, outs):
        o.hessian_matvec_host_async(s, d, out)
    o.wait()
    for d, out in zip(dirs, outs):
        assert np.array_equal(out, o.hessian_matvec(s, d))
    bad = dirs[0].copy()
    bad[0, 1, 2, 3] = np.nan
    o.hessian_matvec_host_async(s, dirs[1], outs[1])
    o.hessian_matvec_host_async(s, bad, outs[0])
    with pytest.raises(vr.NumericError):
        o.wait()
    o.wait()  # nothing in flight: no error


def test_binding_rejects_wrong_shapes(vr, ref, ctx):
    """The C ABI takes bare pointers: the Python mirror checks dtype, contiguity and field
    counts before any call, raising DimensionError instead of letting the
    library read or write past a short buffer."""
    dims = (16, 16, 16)
    c = ctx(dims)
    mR, mT = image_pair(ref, dims, 2, 91)
    o = vr.Objective(c, mR, mT, vr.make_model())
    v = ref.random_smooth_vector(dims, 2, 120, 0.3)
    s = o.evaluate(v)
    o.compute_gradient(s)
    good = np.zeros((3,) + dims)
    for bad in (np.zeros((3,) + dims, dtype=np.float32), np.zeros((2,) + dims),
                np.asfortranarray(np.zeros((3,) + dims))[..., ::-1]):
        with pytest.raises(vr.DimensionError):
            o.hessian_matvec_host(s, bad, good)
        with pytest.raises(vr.DimensionError):
            o.hessian_matvec_host_async(s, bad, good)
    ro_out = np.zeros((3,) + dims)
    ro_out.setflags(write=False)
    with pytest.raises(vr.DimensionError):
        o.hessian_matvec_host(s, good, ro_out)
    with pytest.raises(vr.DimensionError):
        o.hessian_matvec(s, c.empty(1))
    with pytest.raises(vr.DimensionError):
        o.hessian_matvec(s, v, out=c.empty(1))
    with pytest.raises(vr.DimensionError):
        o.evaluate(np.zeros((2,) + dims))
    with pytest.raises(vr.DimensionError):
        vr.Objective(c, np.zeros((2,) + dims), mT, vr.make_model())
    # the well-formed call still works after the rejected ones
    out = np.zeros((3,) + dims)
    o.hessian_matvec_host(s, np.ascontiguousarray(v), out)
    assert np.isfinite(out).all() and np.abs(out).max() > 0
