"""solve_profile.py -- config-3 beta continuation with the spectral and the two-level
preconditioner: wall time, per-iteration records and per-category kernel time
(CUDA events per launch; the gap to wall time is host/launch overhead)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_04487_b200 as vr  # noqa: E402
import paper_1808_04487_b200.veloreg as V  # noqa: E402
from paper_1808_04487_b200 import phantom  # noqa: E402


def _pool_reserved():
    try:
        from cuda.bindings import runtime as rt
    except ImportError:
        try:
            from cuda import cudart as rt
        except ImportError:
            return None
    err, pool = rt.cudaDeviceGetDefaultMemPool(0)
    err, v = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    return int(v) / 1e9


def main():
    if os.environ.get("TORCH_FIRST"):  # the bench's order: torch owns the primary context
        import torch
        torch.cuda.set_device(0)
        torch.zeros(1, device="cuda")
    n = int(os.environ.get("N", "256"))
    cfg = phantom.CONFIGS[3]
    m_T = phantom.ellipsoid_phantom(n)
    v = phantom.bandlimited_velocity(n, cfg["kmax"], cfg["disp"])
    ctx = vr.Context(n)
    d_mT = ctx.to_device(m_T)
    d_mR = ctx.to_device(np.asarray(V.solve_state(ctx, m_T, v, 4))[4])
    model = V.make_model("h2", beta_v=1e-2, nt=4)
    params = V.make_params(eps_opt=1e-2)
    d_v0 = ctx.to_device(np.zeros((3, n, n, n)))
    if os.environ.get("HOT"):  # the bench's preamble: 100 matvecs at the generating velocity
        o = V.Objective(ctx, d_mR, d_mT, V.make_model("h2", beta_v=1e-2, nt=4))
        st = o.evaluate(ctx.to_device(v))
        o.compute_gradient(st)
        vt = ctx.to_device(phantom.bandlimited_direction(n))
        out = ctx.empty(3)
        for _ in range(100):
            o.hessian_matvec(st, vt, out=out)
        ctx.synchronize()
    plan = [(pc, prof) for pc in ("spectral", "two_level", "spectral", "two_level") for prof in (False, True)]
    if os.environ.get("REPEAT"):
        plan = [("spectral", False)] * int(os.environ["REPEAT"])
    for pc, prof in plan:
        if True:
            ctx.synchronize()
            ctx.set_profiling(prof)
            t0 = time.perf_counter()
            _, reps, recs = V.parameter_continuation(ctx, d_mR, d_mT, d_v0, model, params, precond=pc)
            ctx.synchronize()
            wall = time.perf_counter() - t0
            out = {"precond": pc, "profiling": prof, "wall_s": wall, "pool_reserved_GB": _pool_reserved(),
                   "newton": [r["outer_iterations"] for r in reps],
                   "fine_mv": sum(r["fine"]["hessian_matvecs"] for r in reps),
                   "coarse_mv": sum(r["coarse"]["hessian_matvecs"] for r in reps),
                   "records": [{k: rr[k] for k in ("k", "inner_iterations", "fine_matvecs", "coarse_matvecs",
                                                   "wall_time_s")} for rr in recs]}
            if prof:
                p = ctx.profile_read()
                out["kernel_ms"] = {k: round(t, 2) for k, (c, t) in sorted(p.items(), key=lambda kv: -kv[1][1])}
                out["kernel_total_ms"] = sum(t for c, t in p.values())
                ctx.set_profiling(False)
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
