"""diag_fullsize.py -- per-stage GPU vs reference differences at config 3 (diagnostic)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_04487_b200 as vr  # noqa: E402
from oracle import ref  # noqa: E402
from paper_1808_04487_b200 import phantom  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


n = int(os.environ.get("N", "256"))
ref.set_workers(os.cpu_count())
m_T, v = phantom.make_config_inputs(3, n)
c = vr.Context(n)
m_R = np.asarray(vr.solve_state(c, m_T, v, 4))[4]
model = vr.make_model()
for scale in (0.5, 0.0):
    ve = scale * v
    o = vr.Objective(c, m_R, m_T, model)
    s = o.evaluate(ve)
    o.compute_gradient(s)
    ro = ref.Objective(m_R, m_T, model)
    rs = ro.evaluate(ve)
    g_ref = ro.compute_gradient(rs)
    g = s.gradient
    print("scale", scale, "mismatch_rel", s.mismatch_rel, rs.scalars()["mismatch_rel"])
    for w, name in ((1, "X_bwd"), (4, "m_hist"), (2, "X_fwd"), (3, "factor")):
        a, b = s.get(w), rs.get(w)
        if w in (1, 2):
            d = np.mod(a - b + np.pi, 2 * np.pi) - np.pi
            print(f"  {name}: max periodic diff {np.abs(d).max():.3e}")
        else:
            print(f"  {name}: rel {rel(a, b):.3e}")
    print("  gradient rel", rel(g, g_ref), "per comp", [rel(g[i], g_ref[i]) for i in range(3)])
    reg = np.asarray(vr.apply_reg_operator(c, ve, model.norm, "apply", model.beta_v))
    print("  |g| =", np.linalg.norm(g_ref), " |beta A v| =", np.linalg.norm(reg), " |data| =", np.linalg.norm(g_ref - reg))
    dg = g - g_ref
    idx = np.unravel_index(np.argmax(np.abs(dg)), dg.shape)
    print("  worst", idx, dg[idx], g_ref[idx])
