"""x1-slab decomposition on CPU: world_size 2 and 4 over torch.distributed gloo.

Each rank holds its slab (geometry from the library's own vr_slab_layout) and
runs the slab protocol of tests/slab_np.py -- halo exchange, all-to-all FFT
transposes, slab-relative tricubic gathers, rank-ordered reductions -- through
a full Gauss-Newton Hessian matvec; every intermediate is compared with the
global numpy oracle restricted to that slab. The CUDA slab path itself runs on
the GPU in tests/test_gpu_dist.py.
"""
from __future__ import annotations

import json
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

NT = 4
BETA = 1e-2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(shape):
    from oracle import veloreg_np as O
    _, m_T, v = O.generate_synthetic(shape, NT)
    rng = np.random.default_rng(7)
    spec = np.zeros((3, shape[0], shape[1], shape[2] // 2 + 1), dtype=np.complex128)
    for c in range(3):  # smooth random direction (|k|_inf <= 2)
        for k1 in (-2, -1, 0, 1, 2):
            for k2 in (-2, -1, 0, 1, 2):
                for k3 in (0, 1, 2):
                    spec[c, k1, k2, k3] = rng.standard_normal() + 1j * rng.standard_normal()
    vt = np.stack([np.fft.irfftn(spec[c], s=shape, axes=(0, 1, 2)) for c in range(3)])
    return m_T, v, vt / np.abs(vt).max()


def _rel(a, b):
    nb = float(np.linalg.norm(np.ravel(b)))
    return float(np.linalg.norm(np.ravel(a - b))) / (nb if nb > 0 else 1.0)


def _worker(rank, P, shape, halo, port, out):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    from oracle import veloreg_np as O
    import paper_1808_04487_b200.veloreg as V
    from slab_np import Slab

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        S = Slab(shape, rank, P, halo)
        lo, hi = S.off1, S.off1 + S.L
        sl = (slice(None), slice(lo, hi))
        m_T, v, vt = _inputs(shape)
        res = {}

        def put(name, err):
            res[name] = S.allmax(err)

        # geometry: the slabs tile x1, the spectrum rows tile x2
        res["cover_x1"] = S.allsum(S.L) == shape[0]
        res["cover_x2"] = S.allsum(S.n2s) == shape[1]
        # halo exchange = periodic wrap of the global field
        idx = np.arange(lo - S.H, hi + S.H) % shape[0]
        put("halo", float(np.abs(S.halo_pad(m_T[lo:hi]) - m_T[idx]).max()))
        # distributed r2c / c2r
        spec = S.rfft(m_T[lo:hi])
        gspec = np.fft.rfftn(m_T)[:, S.k2_off:S.k2_off + S.n2s]
        put("rfft", _rel(spec, gspec))
        put("irfft", _rel(S.irfft(spec), m_T[lo:hi]))
        # spectral operators
        put("gradient", _rel(S.gradient(m_T[lo:hi]), O.gradient(m_T)[sl]))
        put("divergence", _rel(S.divergence(v[sl]), O.divergence(v)[lo:hi]))
        put("reg", _rel(S.reg(vt[sl], BETA), O.apply_reg_operator(vt, O.H2, O.APPLY, BETA)[sl]))
        ip = S.inner_product(v[sl], vt[sl])
        put("inner_product", abs(ip - O.inner_product(v, vt)) / abs(O.inner_product(v, vt)))
        # semi-Lagrangian: characteristics, gathers through the halo, state solve
        bwd = S.trace(v[sl], NT, "backward")
        gbwd = O.trace_characteristics(v, NT, "backward")
        put("trace", float(np.abs(np.mod(bwd - gbwd[sl] + np.pi, 2 * np.pi) - np.pi).max()))
        _, reach = S.tricubic(S.halo_pad(m_T[lo:hi]), bwd)
        vmax1 = S.allmax(np.abs(v[0][lo:hi]).max())
        res["halo_required"] = V.slab_halo_required(vmax1, NT, shape[0])
        res["reach"] = S.allmax(reach)
        hist = S.solve_state(m_T[lo:hi], bwd, NT)
        put("state", _rel(hist, O.solve_state(m_T, v, NT)[:, lo:hi]))
        # the full GN Hessian matvec
        obj = O.Objective(m_T, m_T, O.H2, BETA, NT)
        s = obj.evaluate(v)
        obj.compute_gradient(s)
        hv, _ = S.hessian_matvec(None, m_T[lo:hi], v[sl], vt[sl], NT, BETA)
        ghv = obj.hessian_matvec(s, vt)
        put("matvec", _rel(hv, ghv[sl]))
        hvt = S.inner_product(hv, vt[sl])
        put("matvec_quad", abs(hvt - O.inner_product(ghv, vt)) / abs(O.inner_product(ghv, vt)))
        # two-level grid transfer: restriction / prolongation of a field below the coarse
        # Nyquist frequency is exact sub-sampling / the identity
        cshape = tuple(d // 2 for d in shape)
        if cshape[0] % P == 0 and cshape[1] % P == 0 and cshape[0] // P >= 4 and min(cshape) >= 4:
            C = Slab(cshape, rank, P, 4)
            x1, x2, x3 = O.coords(shape)
            X1, X2, X3 = np.meshgrid(x1, x2, x3, indexing="ij")
            band = np.sin(X1) * np.cos(X2) + 0.5 * np.cos(X3 + X1) - 0.25 * np.sin(X2 - X3) + 0.1
            coarse_spec = S.restrict_to(S.rfft(band[lo:hi]), C)
            clo, chi = C.off1, C.off1 + C.L
            put("restrict", _rel(C.irfft(coarse_spec), band[::2, ::2, ::2][clo:chi]))
            put("prolong", _rel(S.irfft(C.prolong_to(coarse_spec, S)), band[lo:hi]))
        if rank == 0:
            with open(out, "w") as f:
                json.dump(res, f)
    finally:
        dist.destroy_process_group()


CASES = [(2, (16, 16, 16), 6), (4, (32, 16, 16), 5)]


@pytest.fixture(scope="module", params=CASES, ids=lambda c: f"P{c[0]}-{'x'.join(map(str, c[1]))}")
def slab_run(request, tmp_path_factory):
    import torch.multiprocessing as mp
    P, shape, halo = request.param
    out = str(tmp_path_factory.mktemp("slab") / "res.json")
    mp.spawn(_worker, args=(P, shape, halo, _free_port(), out), nprocs=P, join=True)
    with open(out) as f:
        return P, shape, halo, json.load(f)


def test_slab_geometry_tiles_grid(slab_run):
    _, _, _, r = slab_run
    assert r["cover_x1"] and r["cover_x2"]


def test_slab_halo_exchange(slab_run):
    assert slab_run[3]["halo"] == 0.0


@pytest.mark.parametrize("key", ["rfft", "irfft", "gradient", "divergence", "reg"])
def test_slab_spectral_matches_global(slab_run, key):
    assert slab_run[3][key] <= 1e-12, (key, slab_run[3][key])


def test_slab_rank_ordered_inner_product(slab_run):
    assert slab_run[3]["inner_product"] <= 1e-13


def test_slab_semi_lagrangian_matches_global(slab_run):
    r = slab_run[3]
    assert r["trace"] <= 1e-12
    assert r["state"] <= 1e-12


def test_slab_halo_requirement_covers_stencil_reach(slab_run):
    _, _, halo, r = slab_run
    # planes b .. b+3 of a point on either slab edge stay inside the halo
    assert r["reach"] + 3 <= r["halo_required"] <= halo


def test_slab_gn_matvec_matches_global(slab_run):
    r = slab_run[3]
    assert r["matvec"] <= 1e-11, r["matvec"]
    assert r["matvec_quad"] <= 1e-11


def test_slab_two_level_band_exchange(slab_run):
    """The coarse-band exchange of the slab two-level preconditioner: fine k2 rows travel to
    the rank owning the coarse row they alias onto (restriction) and the all-gathered coarse
    slabs fill every rank's fine rows (prolongation)."""
    r = slab_run[3]
    if "restrict" not in r:
        pytest.skip("coarse grid too small for this rank count")
    assert r["restrict"] < 1e-12 and r["prolong"] < 1e-12


def test_slab_layout_validation():
    import paper_1808_04487_b200.veloreg as V
    from paper_1808_04487_b200._lib import ArgumentError
    with pytest.raises(ArgumentError):
        V.slab_layout(16, 0, 3, 4)           # n1 not divisible by P
    with pytest.raises(ArgumentError):
        V.slab_layout((16, 6, 16), 0, 2, 4)  # not a power of two -> dimension error
    with pytest.raises(ArgumentError):
        V.slab_layout(16, 0, 2, 9)           # halo > planes per rank
    with pytest.raises(ArgumentError):
        V.slab_layout(16, 2, 2, 4)           # rank out of range
    lay = V.slab_layout((32, 16, 8), 3, 4, 8)
    assert (lay["planes"], lay["first_plane"], lay["n2s"], lay["k2_off"]) == (8, 24, 4, 12)
    assert lay["padded_stride"] == (8 + 16) * 16 * 8 and lay["global_points"] == 32 * 16 * 8
