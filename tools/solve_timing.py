"""Config-3 beta-continuation solve with VR_TIMING phase times (host wall per phase,
stream drained at each boundary) and plain wall-clock runs; prints JSON lines."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_04487_b200 as vr  # noqa: E402
from paper_1808_04487_b200 import phantom  # noqa: E402

n = int(os.environ.get("N", "256"))
cfg = phantom.CONFIGS[3]
m_T = phantom.ellipsoid_phantom(n)
v = phantom.bandlimited_velocity(n, cfg["kmax"], cfg["disp"])
c = vr.Context(n)
dT, dv = c.to_device(m_T), c.to_device(v)
hist = vr.solve_state(c, dT, dv, 4)
dR = c.empty(1)
vr._lib.call("vr_memcpy_d2d", c.handle, dR.ptr, hist.field(4), 8 * c.N)
model, params = vr.make_model(), vr.make_params(eps_opt=1e-2)
d0 = c.to_device(np.zeros((3, n, n, n)))
runs = []
for i in range(int(os.environ.get("RUNS", "6"))):
    c.synchronize()
    t0 = time.perf_counter()
    vs, reps, _ = vr.parameter_continuation(c, dR, dT, d0, model, params)
    c.synchronize()
    runs.append(time.perf_counter() - t0)
    vs.free()
print(json.dumps({"n": n, "runs_s": runs, "median_steady_s": float(np.median(runs[1:])),
                  "newton": [r["outer_iterations"] for r in reps],
                  "matvecs": sum(r["fine"]["hessian_matvecs"] for r in reps),
                  "evals": sum(r["fine"]["objective_evals"] for r in reps),
                  "grads": sum(r["fine"]["gradient_evals"] for r in reps)}), flush=True)
c.set_profiling(True)
vs, reps, _ = vr.parameter_continuation(c, dR, dT, d0, model, params)
c.synchronize()
prof = c.profile_read()
c.set_profiling(False)
tot = sum(t for _, t in prof.values())
print(json.dumps({"kernel_ms_total": tot, "by_cat_ms": {k: round(t, 2) for k, (cnt, t) in
                                                         sorted(prof.items(), key=lambda kv: -kv[1][1])}}),
      flush=True)
