"""GPU: the x1-slab decomposition on ONE B200 via P virtual ranks.

Each virtual rank owns n1/P planes, exchanges halo planes before every gather,
and runs the x1 FFT pass on its k2 slab after an all-to-all transpose; the
assembled slab results must equal the single-GPU path (which is itself pinned
to the reference). The NCCL transport uses the same call sequence.
"""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _single(vr, ctx, mR, mT, v, vt, model):
    o = vr.Objective(ctx, mR, mT, model)
    s = o.evaluate(v)
    o.compute_gradient(s)
    hv = o.hessian_matvec(s, vt)
    reg = o.apply_reg(vt, "apply")
    return s, s.gradient, hv, reg


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("name,kw", [("h2", dict()),
                                     ("h1div", dict(kind="h1", beta_v=1e-3, div_penalty=True,
                                                    projection="near_incompressible")),
                                     ("h2_full_newton", dict(gauss_newton=False))])
def test_slab_objective_matches_single_gpu(vr, ref, ctx, P, name, kw):
    dims = (32, 32, 32)
    mR, mT, vs = ref.generate_synthetic(dims, 4)
    v = 0.8 * vs + 0.05 * ref.random_smooth_vector(dims, 2, 11, 1.0)
    vt = ref.random_smooth_vector(dims, 2, 142, 1.0)
    model = vr.make_model(**kw)
    s, g1, hv1, reg1 = _single(vr, ctx(dims), mR, mT, v, vt, model)
    g, hv, reg, sc = vr.dist_selftest_objective(P, mR, mT, v, vt, model, halo=8)
    assert abs(sc["objective"] - s.objective) <= 1e-12 * abs(s.objective)
    assert abs(sc["mismatch"] - s.mismatch) <= 1e-12 * abs(s.mismatch)
    assert rel_l2(reg, reg1) < 1e-13
    assert rel_l2(g, g1) < 1e-12
    assert rel_l2(hv, hv1) < 1e-12
    assert abs(sc["grad_norm"] - np.linalg.norm(g1)) <= 1e-12 * np.linalg.norm(g1)


@pytest.mark.parametrize("dims,P", [((16, 1024, 8), 2), ((32, 512, 4), 4), ((64, 8, 16), 8)])
def test_slab_transposes_long_and_short_k2_blocks(vr, ref, ctx, dims, P):
    """The fused all-to-all layouts at their limits: n2/P = 512 rows per peer block (two
    256-row groups per block in the tensor map of the inverse x2 pass), 128 rows on four
    ranks, and one row per rank; the regularisation operator and the objective's spectral
    terms against the single-GPU path."""
    mR, mT, vs = ref.generate_synthetic(dims, 4)
    v = 0.5 * vs
    vt = ref.random_smooth_vector(dims, 2, 142, 1.0)
    model = vr.make_model()
    s, g1, hv1, reg1 = _single(vr, ctx(dims), mR, mT, v, vt, model)
    g, hv, reg, sc = vr.dist_selftest_objective(P, mR, mT, v, vt, model, halo=8)
    assert rel_l2(reg, reg1) < 1e-13
    assert rel_l2(g, g1) < 1e-12
    assert rel_l2(hv, hv1) < 1e-12


def test_slab_objective_config3_like(vr, ctx):
    from paper_1808_04487_b200 import phantom
    n = 64
    mT = phantom.ellipsoid_phantom(n, count=12)
    v = phantom.bandlimited_velocity(n, 6, 0.08 * 2 * np.pi)
    vt = phantom.bandlimited_direction(n)
    c = ctx(n)
    mR = vr.solve_state(c, mT, v, 4)[-1]
    model = vr.make_model()
    s, g1, hv1, _ = _single(vr, c, mR, mT, v, vt, model)
    g, hv, _, sc = vr.dist_selftest_objective(4, mR, mT, v, vt, model, halo=8)
    assert rel_l2(g, g1) < 1e-12 and rel_l2(hv, hv1) < 1e-12


def test_slab_gn_solve_matches_single_gpu(vr, ref, ctx):
    dims = (32, 32, 32)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model, params = vr.make_model(), vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3,) + dims)
    single = vr.gauss_newton_solve(ctx(dims), mR, mT, v0, model, params)
    vsol, rep = vr.dist_selftest_solve(2, mR, mT, v0, model, params, halo=8)
    assert rep["outer_iterations"] == single.report["outer_iterations"]
    assert rep["fine"]["hessian_matvecs"] == single.report["fine"]["hessian_matvecs"]
    assert abs(rep["final_mismatch_rel"] - single.report["final_mismatch_rel"]) <= 1e-9
    assert rel_l2(vsol, single.v) < 1e-9


def test_slab_halo_too_narrow_raises(vr, ref):
    dims = (32, 32, 32)
    mR, mT, vs = ref.generate_synthetic(dims, 4)
    big = 12.0 * vs  # per-step x1 displacement of several planes
    with pytest.raises(vr.ResourceError):
        vr.dist_selftest_objective(4, mR, mT, big, vs, vr.make_model(), halo=4)


def test_slab_rejects_bad_decomposition(vr, ref):
    dims = (16, 16, 16)
    mR, mT, vs = ref.generate_synthetic(dims, 4)
    with pytest.raises(vr.ArgumentError):
        vr.dist_selftest_objective(8, mR, mT, vs, vs, vr.make_model(), halo=4)  # 2 planes per rank


@pytest.mark.parametrize("P", [2, 4])
def test_slab_interior_halo_overlap(vr, ctx, P):
    """Slabs thick enough (L > 2 halo) that every semi-Lagrangian step runs its interior
    planes while the halo exchange is in flight on the side stream, and the reg term's
    transposes run on the side stream under the sweeps (SURVEY 8(e) "Overlap"): the
    assembled results must still equal the single-GPU path."""
    from paper_1808_04487_b200 import phantom
    n = 64 if P == 2 else 128
    mT = phantom.ellipsoid_phantom(n, count=12)
    v = phantom.bandlimited_velocity(n, 6, 0.08 * 2 * np.pi)
    vt = phantom.bandlimited_direction(n)
    c = ctx(n)
    mR = vr.solve_state(c, mT, v, 4)[-1]
    model = vr.make_model()
    s, g1, hv1, reg1 = _single(vr, c, mR, mT, v, vt, model)
    halo = vr.slab_halo_required(float(np.abs(v[0]).max()), 4, n)
    assert n // P > 2 * halo
    g, hv, reg, sc = vr.dist_selftest_objective(P, mR, mT, v, vt, model, halo=halo)
    assert abs(sc["objective"] - s.objective) <= 1e-12 * abs(s.objective)
    assert rel_l2(g, g1) < 1e-12 and rel_l2(hv, hv1) < 1e-12 and rel_l2(reg, reg1) < 1e-13
