"""GPU postprocess and continuation vs the compiled reference.

Reference: proj/src/postprocess.cpp:13-167 (det grad y, deformation map,
det_stats, label transport, overlap scores; tests proj/tests/test_postprocess.cpp)
and SPEC.md:494-520 (grid / scale continuation and the beta search, which the
reference code does not implement: the oracle restates them in
oracle/ref_capi.cpp as loops over the reference's own solver and postprocess
functions). Bars: fields 1e-10 relative L2 (fp64); labels and overlap scores
exact; solves as in test_gpu_solver.py (Newton iterations +-1, final mismatch
within 1%).
"""
import numpy as np
import pytest

from conftest import periodic_diff, rel_l2

pytestmark = pytest.mark.gpu


def _compressible(ref, dims, amp=1.0):
    # seeded band-limited field of the reference test support (test_support.hpp:90-97)
    return ref.random_smooth_vector(dims, 2, 4487, amp)


@pytest.mark.parametrize("n", [16, 32])
def test_det_deformation_gradient(vr, ref, ctx, n):
    dims = (n, n, n)
    c = ctx(dims)
    for v in (_compressible(ref, dims, 0.8), ref.generate_synthetic(dims, 4)[2], np.zeros((3,) + dims)):
        g = vr.det_deformation_gradient(c, v, 4)
        r = ref.det_deformation_gradient(v, 4)
        assert rel_l2(g, r) <= 1e-10
    assert np.all(vr.det_deformation_gradient(c, np.zeros((3,) + dims), 4) == 1.0)


@pytest.mark.parametrize("absolute", [False, True])
def test_deformation_map(vr, ref, ctx, absolute):
    dims = (32, 32, 32)
    c = ctx(dims)
    v = _compressible(ref, dims, 0.6)
    g = vr.deformation_map(c, v, 4, absolute=absolute)
    r = ref.deformation_map(v, 4, absolute=absolute)
    if absolute:
        assert periodic_diff(g, r).max() <= 1e-12
    else:
        assert rel_l2(g, r) <= 1e-10


def test_det_stats(vr, ref, ctx):
    dims = (16, 16, 16)
    c = ctx(dims)
    mR, _, _ = ref.generate_synthetic(dims, 4)
    det = ref.det_deformation_gradient(_compressible(ref, dims, 0.8), 4)
    for fg in (None, mR):
        g = vr.det_stats(c, det, fg, 0.05)
        r = ref.det_stats(det, fg, 0.05)
        assert g["min"] == r["min"] and g["max"] == r["max"]
        assert abs(g["mean"] - r["mean"]) <= 1e-14 * abs(r["mean"])
    # test_postprocess.cpp:70-88 masked extremes; nothing counted -> zeros
    d = np.ones((8, 8, 8))
    d.flat[0], d.flat[1] = 0.5, 2.0
    fg = np.ones_like(d)
    fg.flat[0] = fg.flat[1] = 0.0
    c8 = ctx((8, 8, 8))
    assert vr.det_stats(c8, d)["min"] == 0.5 and vr.det_stats(c8, d)["max"] == 2.0
    m = vr.det_stats(c8, d, fg, 0.05)
    assert m["min"] == 1.0 and m["max"] == 1.0
    assert vr.det_stats(c8, d, np.zeros_like(d), 0.05) == {"min": 0.0, "mean": 0.0, "max": 0.0}


def _labels(ref, dims):
    mR, mT, vs = ref.generate_synthetic(dims, 4)
    lab = np.round(mT * 4.0)  # codes 0..4 in nested shells
    lab[lab == 2] = 7         # non-contiguous code
    lab[0, 0, :4] = -3        # negative code
    return lab, vs


@pytest.mark.parametrize("n", [16, 32])
def test_transport_labels(vr, ref, ctx, n):
    dims = (n, n, n)
    c = ctx(dims)
    lab, vs = _labels(ref, dims)
    for v in (vs, _compressible(ref, dims, 0.8), np.zeros((3,) + dims)):
        g = vr.transport_labels(c, lab, v, 4)
        r = ref.transport_labels(lab, v, 4)
        assert np.array_equal(g, r)


def test_transport_labels_limit(vr, ctx):
    dims = (16, 16, 16)
    lab = np.arange(16 ** 3, dtype=np.float64).reshape(dims) % 65 + 1  # 65 codes
    with pytest.raises(vr.ResourceError):
        vr.transport_labels(ctx(dims), lab, np.zeros((3,) + dims), 4)


def test_overlap_scores(vr, ref, ctx):
    dims = (32, 32, 32)
    c = ctx(dims)
    lab, vs = _labels(ref, dims)
    moved = ref.transport_labels(lab, vs, 4)
    mR, _, _ = ref.generate_synthetic(dims, 4)
    mask = (mR > 0.3).astype(np.float64)
    for m in (None, mask):
        g = vr.overlap_scores(c, lab, moved, m)
        r = ref.overlap_scores(lab, moved, m)
        assert g["n_labels"] == r["n_labels"]
        assert list(g["per_label"]) == list(r["per_label"])
        for k in r["per_label"]:
            assert g["per_label"][k] == pytest.approx(r["per_label"][k], rel=0, abs=0)
        assert g["union"] == pytest.approx(r["union"], rel=0, abs=0)
    # empty on both sides: dice 1, rates 0 (postprocess.hpp:52-53)
    z = np.zeros(dims)
    e = vr.overlap_scores(c, z, z)
    assert e["n_labels"] == 0 and e["union"] == {"dice": 1.0, "false_positive_rate": 0.0,
                                                  "false_negative_rate": 0.0}


def _cmp_levels(rg, rr):
    assert len(rg) == len(rr)
    for a, b in zip(rg, rr):
        assert a["stop"] == b["stop"]
        assert abs(a["outer_iterations"] - b["outer_iterations"]) <= 1
        assert abs(a["final_mismatch_rel"] - b["final_mismatch_rel"]) <= 1e-2 * b["final_mismatch_rel"]


def test_grid_continuation(vr, ref, ctx):
    dims = (32, 32, 32)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model, params = vr.make_model(), vr.make_params()
    v0 = np.zeros((3,) + dims)
    vg, rg, _ = vr.grid_continuation(c, mR, mT, v0, 2, model, params)
    vref, rr, _ = ref.grid_continuation(mR, mT, v0, 2, model, params)
    _cmp_levels(rg, rr)
    assert rel_l2(vg, vref) < 1e-6
    # one level == the plain solve
    v1, r1, _ = vr.grid_continuation(c, mR, mT, v0, 1, model, params)
    plain = vr.gauss_newton_solve(c, mR, mT, v0, model, params)
    assert np.array_equal(v1, plain.v) and r1[0]["outer_iterations"] == plain.report["outer_iterations"]
    with pytest.raises(vr.ArgumentError):
        vr.grid_continuation(c, mR, mT, v0, 3, model, params)  # coarsest would be 8^3


def test_scale_continuation(vr, ref, ctx):
    dims = (32, 32, 32)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model, params = vr.make_model(), vr.make_params()
    v0 = np.zeros((3,) + dims)
    vg, rg, _ = vr.scale_continuation(c, mR, mT, v0, [4.0, 2.0, 1.0], model, params)
    vref, rr, _ = ref.scale_continuation(mR, mT, v0, [4.0, 2.0, 1.0], model, params)
    _cmp_levels(rg, rr)
    assert rel_l2(vg, vref) < 1e-6
    with pytest.raises(vr.ArgumentError):
        vr.scale_continuation(c, mR, mT, v0, [1.0, 2.0], model, params)


def test_beta_search(vr, ref, ctx):
    dims = (16, 16, 16)
    c = ctx(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model, params = vr.make_model(), vr.make_params()
    v0 = np.zeros((3,) + dims)
    sp = vr.beta_search_params(eps_J=0.9)
    bg, vg, tg = vr.beta_search(c, mR, mT, v0, model, params, search=sp)
    br, vref, tr = ref.beta_search(mR, mT, v0, model, params, sp)
    assert [t["beta"] for t in tg] == pytest.approx([t["beta"] for t in tr], rel=1e-15)
    assert [t["feasible"] for t in tg] == [t["feasible"] for t in tr]
    assert len(tg) > 2 and bg == br
    for a, b in zip(tg, tr):
        assert abs(a["report"]["outer_iterations"] - b["report"]["outer_iterations"]) <= 1
        assert a["det_min"] == pytest.approx(b["det_min"], rel=1e-6)
        assert a["det_max"] == pytest.approx(b["det_max"], rel=1e-6)
    assert rel_l2(vg, vref) < 1e-6
    # the returned beta satisfies the bounds, a 10x smaller one does not
    det = vr.det_deformation_gradient(c, vg, 4)
    assert det.min() >= 0.9 and det.max() <= 1 / 0.9
    # m_T == m_R: every beta feasible -> the bracket's lower end
    b0, _, t0 = vr.beta_search(c, mT, mT, v0, model, params, search=sp)
    assert b0 == sp.beta_lo and len(t0) == 2
    # bound unreachable -> NumericError carrying the trials
    with pytest.raises(vr.NumericError) as e:
        vr.beta_search(c, mR, mT, v0, model, params, search=vr.beta_search_params(eps_J=0.9999999))
    assert len(e.value.trials) == 1 and not e.value.trials[0]["feasible"]


def _compressible_velocity(x, y, z):
    # proj/tests/test_postprocess.cpp:18-25 over synthetic_velocity (synthetic.cpp:10-14)
    a = 0.3
    return (np.sin(z) * np.cos(y) * np.sin(y) + a * np.cos(x) * np.sin(y) * np.sin(z),
            np.sin(x) * np.cos(z) * np.sin(z) + a * np.sin(x) * np.cos(y) * np.sin(z),
            np.sin(y) * np.cos(x) * np.sin(x) + a * np.sin(x) * np.sin(y) * np.cos(z))


def _fd_det_grad(n, eps=1e-4, substeps=100):
    """fd_det_grad (proj/tests/oracles.hpp:70-91) at every grid point, vectorised: central
    differences of RK4 backward trajectories (rk4_flow, oracles.hpp:17-35), det3."""
    h = 2 * np.pi / n
    g = np.arange(n) * h
    X = np.stack(np.meshgrid(g, g, g, indexing="ij")).reshape(3, -1)

    def flow(p):
        dt = 1.0 / substeps
        p = p.copy()
        for _ in range(substeps):
            f = lambda q: -np.array(_compressible_velocity(q[0], q[1], q[2]))  # noqa: E731
            k1 = f(p)
            k2 = f(p + 0.5 * dt * k1)
            k3 = f(p + 0.5 * dt * k2)
            k4 = f(p + dt * k3)
            p = p + (dt / 6.0) * (k1 + 2 * k2 + 2 * k3 + k4)
        return p

    J = np.empty((3, 3, X.shape[1]))
    for a in range(3):
        xp, xm = X.copy(), X.copy()
        xp[a] += eps
        xm[a] -= eps
        yp, ym = flow(xp), flow(xm)
        for c in range(3):
            J[c, a] = ((yp[c] - xp[c]) - (ym[c] - xm[c])) / (2 * eps) + (1.0 if c == a else 0.0)
    det = (J[0, 0] * (J[1, 1] * J[2, 2] - J[1, 2] * J[2, 1]) - J[0, 1] * (J[1, 0] * J[2, 2] - J[1, 2] * J[2, 0])
           + J[0, 2] * (J[1, 0] * J[2, 1] - J[1, 1] * J[2, 0]))
    return det.reshape(n, n, n)


def test_reference_postprocess_failures_are_not_the_fft_shim(vr, ref, ctx):
    """The compiled reference fails 2 of its own 7 postprocess checks under the oracle build
    (test_postprocess.cpp:66 and :142). Both failures reproduce identically on the GPU path,
    whose FFT is independent of the oracle's FFTW shim, so they are properties of the
    reference's algorithm at the test's sizes, not of the shim:
    * :66 -- det grad y by continuity transport vs the RK4/FD trajectory oracle exceeds 1e-2
      at 16^3, n_t = 4; the gap is discretisation error (it shrinks with the grid);
    * :142 -- smoothing + arg-max of two small balls at v = 0 flips more boundary voxels than
      the test's ball/20 bound; the GPU flips exactly the same voxels."""
    errs = {}
    for n in (16, 32):
        h = 2 * np.pi / n
        g = np.arange(n) * h
        X1, X2, X3 = np.meshgrid(g, g, g, indexing="ij")
        v = np.stack(_compressible_velocity(X1, X2, X3))
        fd = _fd_det_grad(n)
        d_ref = ref.det_deformation_gradient(v, 4)
        d_gpu = np.asarray(vr.det_deformation_gradient(ctx(n), v, 4))
        errs[n] = (float(np.abs(d_ref - fd).max()), float(np.abs(d_gpu - fd).max()))
    print("det grad y vs FD oracle (reference, gpu):", errs)
    assert errs[16][0] > 1e-2  # the reference's own check (<= 1e-2) fails
    assert abs(errs[16][1] - errs[16][0]) <= 1e-8  # ... identically with an independent FFT
    assert errs[32][0] < 0.5 * errs[16][0]  # discretisation error: shrinks with resolution
    labels = ref.make_ball_labels((32, 32, 32), 2)
    z = np.zeros((3, 32, 32, 32))
    same_ref = ref.transport_labels(labels, z, 4)
    same_gpu = np.asarray(vr.transport_labels(ctx(32), labels, z, 4))
    ball = int((labels != 0).sum())
    flips_ref, flips_gpu = int((same_ref != labels).sum()), int((same_gpu != labels).sum())
    print("label flips at v = 0 (reference, gpu, ball/20):", flips_ref, flips_gpu, ball // 20)
    assert flips_ref > ball // 20 and np.array_equal(same_gpu, same_ref)


# ---- x1 slabs (round 2b): deformation measures, beta search and grid continuation -----------
def _pp_velocity(ref, dims):
    _, _, vs = ref.generate_synthetic(dims, 4)
    return 0.7 * vs + 0.1 * ref.random_smooth_vector(dims, 2, 7, 1.0)


@pytest.mark.parametrize("P", [2, 4])
def test_slab_deformation_measures_match_single_gpu(vr, ref, ctx, P):
    """det grad y, the absolute deformation map (global x1 coordinates on every rank) and
    det_stats (min / max / mean over ranks) on P virtual slab ranks vs one GPU
    (postprocess.cpp:13-81)."""
    dims = (32, 32, 32)
    v = _pp_velocity(ref, dims)
    c = ctx(dims)
    det1 = np.asarray(vr.det_deformation_gradient(c, v, 4))
    map1 = np.asarray(vr.deformation_map(c, v, 4, absolute=True))
    st1 = vr.det_stats(c, det1)
    det, ymap, st = vr.dist_selftest_postprocess(P, v, 4, halo=8)
    assert rel_l2(det, det1) < 1e-13
    assert np.abs(np.angle(np.exp(1j * (ymap - map1)))).max() < 1e-12  # equal modulo 2 pi
    for k in ("min", "max", "mean"):  # the slab divergence takes the 3D transform path: ~1e-16
        assert abs(st[k] - st1[k]) <= 1e-12 * abs(st1[k])


def _one_rank_slab(vr, dims, monkeypatch, halo=8):
    monkeypatch.setenv("VR_DIST_SINGLE_RANK", "1")
    try:
        return vr.DistContext(dims, 0, 1, vr.nccl_unique_id(), device=0, halo=halo)
    except vr.ResourceError as exc:
        pytest.skip(f"NCCL communicator unavailable: {exc}")


def test_slab_beta_search_and_grid_continuation_one_rank_nccl(vr, ref, ctx, monkeypatch):
    """The outer loops on a slab context over the real NCCL transport at one rank: beta search
    (solves + det grad y + det_stats on slabs) and grid continuation (sibling slab contexts per
    level, slab resampling) reproduce the plain context's trials / levels."""
    dims = (32, 32, 32)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model, params = vr.make_model(), vr.make_params()
    v0 = np.zeros((3,) + dims)
    c = ctx(dims)
    d = _one_rank_slab(vr, dims, monkeypatch)
    sp = vr.beta_search_params(eps_J=0.9)
    b1, v1, t1 = vr.beta_search(c, mR, mT, v0, model, params, search=sp)
    bd, vd, td = vr.beta_search(d, mR, mT, v0, model, params, search=sp)
    assert bd == b1 and [t["feasible"] for t in td] == [t["feasible"] for t in t1]
    for a, b in zip(td, t1):
        assert a["report"]["outer_iterations"] == b["report"]["outer_iterations"]
        assert a["det_min"] == pytest.approx(b["det_min"], rel=1e-9)
    assert rel_l2(np.asarray(vd), np.asarray(v1)) < 1e-8
    vg1, rg1, _ = vr.grid_continuation(c, mR, mT, v0, 2, model, params)
    vgd, rgd, _ = vr.grid_continuation(d, mR, mT, v0, 2, model, params)
    assert [r["outer_iterations"] for r in rgd] == [r["outer_iterations"] for r in rg1]
    assert rel_l2(np.asarray(vgd), np.asarray(vg1)) < 1e-8


@pytest.mark.parametrize("P", [2, 4])
def test_slab_label_transport_and_overlap_match_single_gpu(vr, ref, ctx, P):
    """transport_labels (code table and per-code advection with halo exchanges) and
    overlap_scores (voxel counts summed over ranks) on P virtual slab ranks vs one GPU:
    labels equal voxel for voxel, scores equal (postprocess.cpp:83-165)."""
    dims = (32, 32, 32)
    lab, vs = _labels(ref, dims)
    c = ctx(dims)
    w1 = np.asarray(vr.transport_labels(c, lab, vs, 4))
    s1 = vr.overlap_scores(c, lab, w1)
    w, s = vr.dist_selftest_labels(P, lab, vs, 4, halo=8)
    assert np.array_equal(w, w1)
    assert s["n_labels"] == s1["n_labels"] and s["union"] == s1["union"]
    assert s["per_label"] == s1["per_label"]
