"""Generate tests/golden/golden_*.npz from the compiled reference (oracle/_ref).

Run in the build container (where /root/reference exists):
    make -C oracle lib && python tests/golden/make_golden.py
The fixtures let CPU tests pin the numpy oracle and GPU tests check the product
even on a box where the reference sources are absent. Inputs are the reference
test-suite generators (proj/tests/test_support.hpp) and generate_synthetic
(proj/src/synthetic.cpp), outputs the reference operators at the same inputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref  # noqa: E402
import paper_1808_04487_b200._lib as L  # noqa: E402  (POD layouts only)


def model(kind=1, beta_v=1e-2, nt=4, projection=0, div_penalty=0, beta_w=1e-4, gamma=1.0, hsq=1):
    m = L.Model()
    m.norm = L.RegNorm(kind, gamma, hsq, div_penalty, beta_w)
    m.projection, m.beta_v, m.nt, m.gauss_newton = projection, beta_v, nt, 1
    return m


def make(shape, tag):
    out = {}
    f = ref.random_smooth_scalar(shape, 3, 5, 1.0) + 0.1 * ref.random_rough_scalar(shape, 6)
    v = ref.random_smooth_vector(shape, 3, 7, 1.0)
    out["f"], out["v"] = f, v
    out["fft_r2c"] = ref.fft_forward(f)
    out["gradient"] = ref.gradient(f)
    out["divergence"] = ref.divergence(v)
    out["laplacian"] = ref.laplacian(f)
    out["gaussian_1_2_1p5"] = ref.gaussian_smooth(f, (1.0, 2.0, 1.5))
    for kind, nm in ((0, "h1"), (1, "h2"), (2, "h3"), (3, "helmholtz")):
        n = L.RegNorm(kind, 0.7, 1, 0, 1e-4)
        for mode, mn in ((0, "apply"), (1, "inverse"), (2, "inverse_sqrt")):
            out[f"reg_{nm}_{mn}"] = ref.apply_reg_operator(v, n, mode, 3e-2)
    out["leray"] = ref.apply_projection(v, 1)
    out["nearinc"] = ref.apply_projection(v, 2, 1e-3, 1e-4)
    rng = np.random.default_rng(3)
    pts = rng.uniform(-3.0, 10.0, size=(3,) + tuple(shape))
    out["pts"] = pts
    out["tricubic"] = ref.tricubic_interpolate(f, pts)
    mR, mT, vs = ref.generate_synthetic(shape, 4)
    out["syn_mR"], out["syn_mT"], out["syn_v"] = mR, mT, vs
    out["trace_bwd"] = ref.trace_characteristics(vs, 4, "backward")
    out["trace_fwd"] = ref.trace_characteristics(vs, 4, "forward")
    out["state"] = ref.solve_state(mT, vs, 4)
    vt = ref.random_smooth_vector(shape, 2, 142, 1.0)
    out["vt"] = vt
    for name, m in (("h2", model()), ("h1div", model(kind=0, beta_v=1e-3, projection=2, div_penalty=1))):
        o = ref.Objective(mR, mT, m)
        s = o.evaluate(0.5 * vs)
        sc = s.scalars()
        out[f"obj_{name}_J"] = np.array([sc["objective"], sc["mismatch"], sc["mismatch_rel"]])
        out[f"obj_{name}_grad"] = o.compute_gradient(s)
        out[f"obj_{name}_factor"] = s.get(3)
        out[f"obj_{name}_matvec"] = o.hessian_matvec(s, vt)
    p = L.SolverParams(1e-2, 1e-6, 50, 100, 1e-4, 0.5, 20, 1)
    vsol, rep, recs = ref.gauss_newton_solve(mR, mT, np.zeros((3,) + tuple(shape)), model(), p)
    out["gn_v"] = vsol
    out["gn_report"] = np.array([rep["outer_iterations"], rep["final_mismatch_rel"], rep["final_grad_rel"],
                                 rep["fine"]["hessian_matvecs"], rep["fine"]["pde_solves"]])
    out["gn_inner"] = np.array([r["inner_iterations"] for r in recs])
    np.savez_compressed(os.path.join(HERE, f"golden_{tag}.npz"), **out)


if __name__ == "__main__":
    ref.set_workers(4)
    make((16, 16, 16), "16")
    make((8, 16, 32), "8x16x32")
    for fn in sorted(os.listdir(HERE)):
        if fn.endswith(".npz"):
            print(fn, os.path.getsize(os.path.join(HERE, fn)))
