"""variant_bench.py -- time the config-3 matvec and its per-kernel profile for
the library selected by VR_LIB (tuning experiments; prints one JSON line)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_04487_b200 as vr  # noqa: E402
import paper_1808_04487_b200.veloreg as V  # noqa: E402
from paper_1808_04487_b200 import phantom  # noqa: E402


def main():
    n, nt, steps = int(os.environ.get("N", "256")), 4, int(os.environ.get("STEPS", "30"))
    cache = f"/tmp/vb_inputs_{n}.npz"
    if os.path.exists(cache):
        z = np.load(cache)
        m_T, v, vt = z["m_T"], z["v"], z["vt"]
    else:
        cfg = phantom.CONFIGS[3]
        m_T = phantom.ellipsoid_phantom(n)
        v = phantom.bandlimited_velocity(n, cfg["kmax"], cfg["disp"])
        vt = phantom.bandlimited_direction(n)
        np.savez(cache, m_T=m_T, v=v, vt=vt)
    ctx = vr.Context(n)
    model = V.make_model("h2", beta_v=1e-2, nt=nt)
    d_mT, d_v, d_vt = ctx.to_device(m_T), ctx.to_device(v), ctx.to_device(vt)
    obj = V.Objective(ctx, d_mT, d_mT, model)
    st = obj.evaluate(d_v)
    obj.compute_gradient(st)
    out = ctx.empty(3)
    stream = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(3):
        obj.hessian_matvec(st, d_vt, out=out)
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        obj.hessian_matvec(st, d_vt, out=out)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ctx.set_profiling(True)
    for _ in range(10):
        obj.hessian_matvec(st, d_vt, out=out)
    ctx.synchronize()
    prof = ctx.profile_read()
    ctx.set_profiling(False)
    import hashlib
    o = out.numpy()
    res = {"lib": os.environ.get("VR_LIB", "default"),
           "ms_per_matvec": ms, "out_sha1": hashlib.sha1(o.tobytes()).hexdigest()[:12],
           "out_norm": float(np.linalg.norm(o)),
           "kernels_us": {k: round(1e3 * t / c, 1) for k, (c, t) in sorted(prof.items(), key=lambda kv: -kv[1][1])},
           "serial_ms_per_matvec": sum(t for c, t in prof.values()) / 10}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
