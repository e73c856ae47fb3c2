"""Generate tests/golden/config3_solve.npz: the reference's own config-3 solve.

Run in the build container (where /root/reference exists):
    make -C oracle lib && python tests/golden/make_config3_solve.py
BASELINE config 3 (256^3 ellipsoid phantom, band-limited velocity, n_t = 4): the reference's
beta continuation 1 -> 1e-1 -> 1e-2 (gauss_newton_solve per level, proj/src/solver.cpp:154-269)
on the host cores (about 6.5 min on 16 cores). Stored: per level Newton / Krylov iterations,
mismatch, gradient norm and stop reason, and the final velocity on every 8th grid point per
axis plus its norms. tests/test_gpu_fullsize.py compares the GPU solve of the same arrays with
it on every run, so the default GPU suite does not depend on the speed of the box's host cores;
VR_LIVE_CONFIG3=1 re-runs the reference live next to it.
Imports only the oracle and the numpy-only generators (never the GPU library).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref  # noqa: E402
from paper_1808_04487_b200 import phantom  # noqa: E402  (numpy only)

KEYS = ("outer_iterations", "krylov_iterations", "final_mismatch_rel", "final_grad_rel", "final_objective", "stop")


def main():
    n = phantom.CONFIGS[3]["n"]
    m_T, v = phantom.make_config_inputs(3)
    m_R = np.asarray(ref.solve_state(m_T, v, 4))[4]
    model = ref.make_model("h2", beta_v=1e-2, nt=4)
    p = ref.SolverParams()
    p.eps_opt, p.abs_grad_tol, p.max_newton, p.max_krylov = 1e-2, 1e-6, 50, 100
    p.armijo_c1, p.armijo_backtrack, p.armijo_max_trials, p.squared_norm_stop = 1e-4, 0.5, 20, 1
    t0 = time.perf_counter()
    vref, reps, _ = ref.parameter_continuation(m_R, m_T, np.zeros((3, n, n, n)), model, p)
    secs = time.perf_counter() - t0
    out = {"n": n, "seconds": secs, "levels": len(reps), "v_sub8": vref[:, ::8, ::8, ::8].copy(),
           "v_norm": np.linalg.norm(vref.ravel()), "v_absmax": np.abs(vref).max(),
           "m_R_sub8": m_R[::8, ::8, ::8].copy()}
    for k in KEYS:
        if k in reps[0]:
            out[k] = np.array([r[k] for r in reps], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "config3_solve.npz"), **out)
    print("wrote config3_solve.npz in", secs, "s:", [(r["outer_iterations"], r["final_mismatch_rel"], r["final_grad_rel"]) for r in reps])


if __name__ == "__main__":
    main()
