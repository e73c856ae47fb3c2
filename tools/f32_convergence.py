import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1808_04487_b200 as vr
from oracle import ref
ref.set_workers(16)
for n in (32, 64, 128):
    dims = (n, n, n)
    c = vr.Context(dims)
    mR, mT, _ = ref.generate_synthetic(dims, 4)
    model, params = vr.make_model(), vr.make_params(eps_opt=1e-2)
    v0 = np.zeros((3,) + dims)
    g = vr.gauss_newton_solve_f32(c, mR, mT, v0, model, params).report
    d = vr.gauss_newton_solve(c, mR, mT, v0, model, params).report
    line = {"n": n, "gpu_f32": (g["outer_iterations"], g["stop_name"], round(g["final_grad_rel"], 4)),
            "gpu_f64": (d["outer_iterations"], d["stop_name"], round(d["final_grad_rel"], 4))}
    if n <= 64:
        t = time.time()
        _, r, _ = ref.gauss_newton_solve_f32(mR, mT, v0, model, params)
        line["ref_f32"] = (r["outer_iterations"], r["stop"], round(r["final_grad_rel"], 4), round(time.time() - t, 1))
    print(line, flush=True)
