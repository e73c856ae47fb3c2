"""GPU: spectral grid transfer, split matvec and the two-level preconditioner vs the
compiled reference.

Reference: proj/src/spectral.cpp:228-385 (spectrum_restrict / spectrum_prolong,
spectral_resample, frequency_filter), proj/src/objective.cpp:158-176 (split_matvec),
proj/src/precond.cpp (lanczos_bounds, cheb_solve, TwoLevelContext), the split branch of
proj/src/solver.cpp:208-221; tests modelled on proj/tests/test_precond.cpp.
"""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _field(shape, seed, ncomp=1):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(((ncomp,) if ncomp > 1 else ()) + tuple(shape))
    return a


@pytest.mark.parametrize("src,dst", [((16, 16, 16), (8, 8, 8)), ((8, 8, 8), (16, 16, 16)),
                                     ((8, 16, 32), (4, 8, 16)), ((16, 8, 16), (8, 8, 8)),
                                     ((4, 8, 8), (8, 16, 16))])
@pytest.mark.parametrize("ncomp", [1, 3])
def test_spectral_resample(vr, ref, ctx, src, dst, ncomp):
    f = _field(src, 3, ncomp)
    got = vr.spectral_resample(ctx(src), f, ctx(dst))
    want = ref.spectral_resample(f, dst)
    assert rel_l2(got, want) < TOL


def test_resample_round_trip_and_band_limited_identity(vr, ctx):
    # restrict(prolong(f)) == f (spectral.hpp:144-146)
    f = _field((8, 8, 8), 5)
    up = vr.spectral_resample(ctx((8, 8, 8)), f, ctx((16, 16, 16)))
    back = vr.spectral_resample(ctx((16, 16, 16)), up, ctx((8, 8, 8)))
    assert rel_l2(back, f) < 1e-13


@pytest.mark.parametrize("shape,cut", [((16, 16, 16), (8, 8, 8)), ((16, 16, 16), (16, 8, 4)),
                                       ((8, 16, 32), (4, 8, 16))])
@pytest.mark.parametrize("band", ["low", "high"])
def test_frequency_filter(vr, ref, ctx, shape, cut, band):
    f = _field(shape, 7, 3)
    got = vr.frequency_filter(ctx(shape), f, band, cut)
    want = ref.frequency_filter(f, band, cut)
    assert rel_l2(got, want) < TOL
    if band == "low":
        hi = vr.frequency_filter(ctx(shape), f, "high", cut)
        assert np.abs(got + hi - f).max() < 1e-12  # F_L + F_H = id


def _objective_pair(vr, ref, c, shape, model, scale=0.5):
    mR, mT, vs = ref.generate_synthetic(shape, model.nt)
    v = scale * vs
    og = vr.Objective(c, mR, mT, model)
    sg = og.evaluate(v)
    og.compute_gradient(sg)
    orf = ref.Objective(mR, mT, model)
    sr = orf.evaluate(v)
    orf.compute_gradient(sr)
    return og, sg, orf, sr


MODELS = {
    "h2": dict(kind="h2", beta_v=1e-2, nt=4),
    "h1div_nearinc": dict(kind="h1", beta_v=1e-3, nt=4, div_penalty=True, beta_w=1e-4,
                          projection="near_incompressible"),
    "helmholtz": dict(kind="helmholtz", beta_v=1e-2, nt=2),
}


@pytest.mark.parametrize("name", list(MODELS))
def test_split_matvec(vr, ref, ctx, name):
    shape = (16, 16, 16)
    model = vr.make_model(**MODELS[name])
    og, sg, orf, sr = _objective_pair(vr, ref, ctx(shape), shape, model)
    w = _field(shape, 11, 3)
    got = og.split_matvec(sg, w)
    want = orf.split_matvec(sr, w)
    assert rel_l2(got, want) < TOL


@pytest.mark.parametrize("inner", ["pcg", "cheb"])
def test_twolevel_apply_matches_reference(vr, ref, ctx, inner):
    shape = (16, 16, 16)
    model = vr.make_model("h2", beta_v=1e-2, nt=4)
    og, sg, orf, sr = _objective_pair(vr, ref, ctx(shape), shape, model)
    opts = vr.make_twolevel_options(inner=inner)
    tg = vr.TwoLevelPreconditioner(opts)
    tr = ref.TwoLevelPreconditioner(opts)
    eps_H = 0.3
    tg.rebuild(og, sg, eps_H)
    tr.rebuild(orf, sr, eps_H)
    ig, ir = tg.info(), tr.info()
    assert ig["coarse_dims"] == ir["coarse_dims"] == (8, 8, 8)
    assert ig["lanczos_runs"] == ir["lanczos_runs"] == (1 if inner == "cheb" else 0)
    if inner == "cheb":
        assert abs(ig["bounds"][0] - ir["bounds"][0]) <= 1e-9 * abs(ir["bounds"][0])
        assert abs(ig["bounds"][1] - ir["bounds"][1]) <= 1e-9 * abs(ir["bounds"][1])
    r = _field(shape, 21, 3)
    fine_before = og.counters()
    zg = tg.apply(r)
    zr = tr.apply(r)
    assert rel_l2(zg, zr) < 1e-9
    assert og.counters() == fine_before  # coarse work only
    ig, ir = tg.info(), tr.info()
    assert ig["coarse"] == ir["coarse"]
    assert ig["coarse"]["pde_solves"] == 2 * ig["coarse"]["hessian_matvecs"] > 0
    # the coarse split operator itself
    u = _field((8, 8, 8), 22, 3)
    assert rel_l2(tg.coarse_matvec(u), tr.coarse_matvec(u)) < TOL
    tg.close()


def test_twolevel_high_band_passes_through(vr, ref, ctx):
    # a purely high-frequency residual skips the coarse solve: z = F_H r = r
    shape = (16, 16, 16)
    model = vr.make_model("h2", beta_v=1e-2, nt=4)
    og, sg, _, _ = _objective_pair(vr, ref, ctx(shape), shape, model)
    tg = vr.TwoLevelPreconditioner()
    tg.rebuild(og, sg, 0.5)
    r = _field(shape, 31, 3)
    high = vr.frequency_filter(ctx(shape), r, "high", (8, 8, 8))
    z = tg.apply(high)
    assert np.abs(z - high).max() < 1e-12
    assert tg.info()["coarse"]["hessian_matvecs"] == 0
    tg.close()


def test_twolevel_errors(vr, ref, ctx):
    from paper_1808_04487_b200._lib import DimensionError, LogicError
    tg = vr.TwoLevelPreconditioner()
    tg.fine = ctx((16, 16, 16))
    with pytest.raises(LogicError):
        tg.apply(np.zeros((3, 16, 16, 16)))
    shape = (4, 8, 8)  # x1 would halve to 2 < 4
    model = vr.make_model("h2", beta_v=1e-2, nt=2)
    og, sg, _, _ = _objective_pair(vr, ref, ctx(shape), shape, model)
    with pytest.raises(DimensionError):
        tg.rebuild(og, sg, 0.5)
    tg.close()


@pytest.mark.parametrize("n,inner", [(16, "pcg"), (32, "pcg"), (16, "cheb"), (32, "cheb")])
def test_gauss_newton_two_level_solve(vr, ref, ctx, n, inner):
    # test_precond.cpp:305-324 configuration on the synthetic problem
    dims = (n, n, n)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model = vr.make_model("h2", beta_v=1e-2, nt=4)
    params = vr.make_params(eps_opt=1e-2)
    opts = vr.make_twolevel_options(inner=inner)
    v0 = np.zeros((3,) + dims)
    res = vr.gauss_newton_solve(c, mR, mT, v0, model, params, precond="two_level", twolevel=opts)
    v_r, rep_r, recs_r = ref.gauss_newton_solve_two_level(mR, mT, v0, model, params, opts)
    g = res.report
    assert g["stop"] == rep_r["stop"] and g["success"]
    assert abs(g["outer_iterations"] - rep_r["outer_iterations"]) <= 1
    assert abs(g["final_mismatch_rel"] - rep_r["final_mismatch_rel"]) <= 1e-2 * rep_r["final_mismatch_rel"]
    assert abs(g["final_grad_rel"] - rep_r["final_grad_rel"]) <= 1e-2 * rep_r["final_grad_rel"]
    f = g["fine"]
    assert f["pde_solves"] == f["objective_evals"] + f["gradient_evals"] + 2 * f["hessian_matvecs"]
    assert g["coarse"]["pde_solves"] == 2 * g["coarse"]["hessian_matvecs"] > 0
    if g["outer_iterations"] == rep_r["outer_iterations"]:
        assert rel_l2(res.v, v_r) < 1e-6
        for a, b in zip(res.records, recs_r):
            assert a["inner_iterations"] == b["inner_iterations"]
            assert a["coarse_matvecs"] == b["coarse_matvecs"]


@pytest.mark.parametrize("n,P,inner", [(32, 2, "pcg"), (32, 2, "cheb"), (64, 4, "pcg")])
def test_two_level_solve_on_slabs_matches_single_gpu(vr, ref, ctx, n, P, inner):
    """The two-level preconditioner on x1 slabs (P virtual ranks on one GPU): the coarse grid
    on a sibling slab context, the coarse band exchanged between the ranks' k2 slabs
    (restriction: per-destination partial alias sums + all-to-all; prolongation: all-gathered
    coarse spectra), the Lanczos start vector cut from the global seeded sequence -- against
    the single-GPU two-level solve, itself pinned to the reference (precond.cpp:153-249)."""
    dims = (n, n, n)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model = vr.make_model("h2", beta_v=1e-2, nt=4)
    params = vr.make_params(eps_opt=1e-2)
    opts = vr.make_twolevel_options(inner=inner)
    v0 = np.zeros((3,) + dims)
    one = vr.gauss_newton_solve(ctx(dims), mR, mT, v0, model, params, precond="two_level", twolevel=opts)
    vsol, rep = vr.dist_selftest_solve(P, mR, mT, v0, model, params, halo=8, precond="two_level",
                                       two_level=opts)
    g = one.report
    assert rep["stop"] == g["stop"] and rep["success"]
    assert rep["outer_iterations"] == g["outer_iterations"]
    assert rep["fine"]["hessian_matvecs"] == g["fine"]["hessian_matvecs"]
    assert rep["coarse"]["hessian_matvecs"] == g["coarse"]["hessian_matvecs"] > 0
    assert abs(rep["final_mismatch_rel"] - g["final_mismatch_rel"]) <= 1e-9
    assert rel_l2(vsol, one.v) < 1e-8


def test_two_level_solve_on_one_rank_nccl_slab(vr, ref, ctx, monkeypatch):
    """The same through the real NCCL transport at one rank (VR_DIST_SINGLE_RANK)."""
    dims = (32, 32, 32)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model, params = vr.make_model("h2", beta_v=1e-2, nt=4), vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3,) + dims)
    one = vr.gauss_newton_solve(ctx(dims), mR, mT, v0, model, params, precond="two_level")
    monkeypatch.setenv("VR_DIST_SINGLE_RANK", "1")
    try:
        d = vr.DistContext(dims, 0, 1, vr.nccl_unique_id(), device=0, halo=8)
    except vr.ResourceError as exc:
        pytest.skip(f"NCCL communicator unavailable: {exc}")
    res = vr.gauss_newton_solve(d, mR, mT, v0, model, params, precond="two_level")
    assert res.report["outer_iterations"] == one.report["outer_iterations"]
    assert res.report["coarse"]["hessian_matvecs"] == one.report["coarse"]["hessian_matvecs"]
    assert rel_l2(np.asarray(res.v), one.v) < 1e-8
