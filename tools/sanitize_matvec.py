"""One 32^3 evaluate + gradient + GN Hessian matvec + PCG step through the C ABI; the
driver of the compute-sanitizer test (tests/test_gpu_sanitizer.py)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_04487_b200 as vr  # noqa: E402
from paper_1808_04487_b200 import phantom  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
c = vr.Context(n)
mT = phantom.ellipsoid_phantom(n, count=8)
v = phantom.bandlimited_velocity(n, 4, 0.3)
vt = phantom.bandlimited_direction(n)
mR = np.asarray(vr.solve_state(c, mT, v, 4))[4]
o = vr.Objective(c, mR, mT, vr.make_model())
s = o.evaluate(0.5 * v)
o.compute_gradient(s)
hv = np.asarray(o.hessian_matvec(s, vt))
x, st = vr.pcg_solve(o, s, -np.asarray(s.gradient), 0.1, 3)
c.synchronize()
print("ok", float(np.linalg.norm(hv)), st["iterations"])
# release every device object before the context (memcheck --leak-check full)
s.close()
o.close()
c.close()
