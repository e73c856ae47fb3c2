"""Write the gather_lab inputs: config-3 (256^3) backward departure points of the
seeded band-limited velocity (vr_trace_characteristics, RK2, n_t = 4) and the
ellipsoid phantom, as raw fp64 files."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_04487_b200 as vr  # noqa: E402
from paper_1808_04487_b200 import phantom  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
direction = sys.argv[2] if len(sys.argv) > 2 else "backward"
cfg = phantom.CONFIGS[3]
v = phantom.bandlimited_velocity(n, cfg["kmax"], cfg["disp"])
m = phantom.ellipsoid_phantom(n)
c = vr.Context(n)
X = np.asarray(vr.trace_characteristics(c, v, 4, direction))
X.astype(np.float64).tofile("/tmp/lab_X.bin")
m.astype(np.float64).tofile("/tmp/lab_f.bin")
print("wrote", X.shape, m.shape)
