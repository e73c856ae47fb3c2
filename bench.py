#!/usr/bin/env python
"""bench.py -- Gauss-Newton Hessian matvec throughput on B200 (BASELINE config 3).

Workload (BASELINE.json configs[2], the 1-GPU config the metric is quoted on):
256^3 seeded ellipsoid phantom, band-limited random stationary velocity
(|k| <= 6, max displacement 0.08*2pi), H2 regularization, beta_v = 1e-2,
n_t = 4, Gauss-Newton, K = identity. A "step" is one reduced-space GN Hessian
matvec H vt (objective.cpp:114-156) at the generating velocity, with the
EvalState (state, adjoint context, grad m cache) frozen as in a PCG solve.

Arms:
  default           our sm_100a path through the C ABI (libveloreg_gpu.so)
  --impl reference  the reference C++ code (oracle/_ref, compiled unmodified
                    from /root/reference/proj/src) on the host cores, rank 0 only

Multi-GPU (torchrun, N > 1): BASELINE config 4 (512^3, |k| <= 10) at N = 2..7
and config 5 (1024^3, |k| <= 16, max displacement 0.05*2pi) at N = 8, split
into x1 slabs, one per rank (NCCL all-to-all FFT transposes, P2P halo exchange
for the semi-Lagrangian gathers, halo sized from the actual velocity); every
rank generates only its own slab of the inputs. "scaling": "strong", value =
global matvecs / max-over-ranks time. There is no fallback: if the slab path
cannot start, the rank raises and torchrun tears the job down.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Hessian matvecs/s"
UNIT = "matvec/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--grid", dest="n", type=int, default=None,
                    help="grid size (default: the config's own: 256^3 on one GPU, 512^3 on 2-7, 1024^3 on 8); "
                         "under torchrun spell it --grid (its parser rejects the abbreviation-like --n)")
    ap.add_argument("--config", type=int, default=None, choices=[3, 4, 5],
                    help="BASELINE config whose phantom / velocity parameters to use (default: by world size)")
    ap.add_argument("--nt", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=60.0,
                    help="wall budget for the reference arm's timed matvecs")
    ap.add_argument("--no-ref-detail", action="store_true",
                    help="reference arm: skip the FFT split, 1-worker timing and the CPU GN solves")
    ap.add_argument("--ref-solve3", action="store_true",
                    help="reference arm: also run the reference's config-3 beta-continuation solve "
                         "(~6.5 min on 16 cores; its record is profiles/r02_bench_reference.json and "
                         "the fixture tests/golden/config3_solve.npz)")
    ap.add_argument("--ref-sample-n", type=int, default=256,
                    help="reference arm: largest grid the CPU reference is timed on; a larger config is "
                         "timed on this sub-grid of the same workload and scaled by the point ratio")
    ap.add_argument("--no-solve", action="store_true", help="skip the GN solve timings")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32-lane gather micro-benchmark")
    ap.add_argument("--no-config2", action="store_true",
                    help="skip the 128^3 (config 2) per-operator micro-benchmarks and solve")
    ap.add_argument("--no-config4", action="store_true",
                    help="skip the 512^3 (config 4, one GPU) matvec throughput")
    ap.add_argument("--slab-two-level", action="store_true",
                    help="x1 slabs: also time the continuation with the two-level preconditioner (one GPU "
                         "does it by default; on slabs it is opt-in so that a first multi-GPU run times "
                         "the spectral-preconditioner solve only)")
    ap.add_argument("--force-slabs", action="store_true",
                    help="run the multi-GPU code path (x1 slabs over the NCCL transport, per-slab input "
                         "generation, exchange timing) with whatever world size this is, including 1: a "
                         "one-rank check of the path a torchrun launch takes, not a benchmark")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def config_for(world, n_arg, cid_arg=None):
    """BASELINE config id and grid: config 3 (256^3) on one GPU, config 4 (512^3) on 2-7
    GPUs, config 5 (1024^3) on 8; --n overrides the grid, --config the parameters."""
    cid = cid_arg or (3 if world == 1 else (5 if world >= 8 else 4))
    from paper_1808_04487_b200 import phantom  # numpy only; does not load the product library
    return cid, (n_arg or phantom.CONFIGS[cid]["n"])


def workload_desc(cid, n, nt):
    from paper_1808_04487_b200 import phantom
    c = phantom.CONFIGS[cid]
    return (f"config{cid}: {n}^3 ellipsoid phantom (40, seed 1808, sigma 2 vox), band-limited v "
            f"(|k|<={c['kmax']}, max disp {c['disp'] / (2 * np.pi):.2f}*2pi, seed 4487), GN Hessian matvec at v, "
            f"H2 beta_v=1e-2, n_t={nt}, K=identity, spectral-precond solve setting")


def workload(cid, n, nt):
    """Global host arrays (one process: the single-GPU arm and the reference arm)."""
    from paper_1808_04487_b200 import phantom
    c = phantom.CONFIGS[cid]
    m_T = phantom.ellipsoid_phantom(n)
    v = phantom.bandlimited_velocity(n, c["kmax"], c["disp"])
    vt = phantom.bandlimited_direction(n)
    return m_T, v, vt, workload_desc(cid, n, nt)


def bench_config(cid, n, nt, world):
    """The `config` dict of the JSON line -- identical in both arms."""
    return {"workload": workload_desc(cid, n, nt), "grid": n, "nt": nt,
            "l2": f"inputs larger than L2 (each fp64 field {8 * n ** 3 / 2 ** 20:.0f} MiB of the global grid; "
                  f"~{int(bytes_model(n, nt)[0] / 8 / n ** 3)} fields touched per step)",
            "parallelism": "single" if world == 1 else f"x1-slabs-{world}"}


def bytes_model(n, nt):
    """Algorithmic bytes with F = 8N and F_c = 16 n^2 (n/2+1)."""
    N = n ** 3
    F = 8.0 * N
    Fc = 16.0 * n * n * (n // 2 + 1)
    per_matvec = 8.0 * N * (9 + 8 * (nt + 1) + 12 * nt) + 6 * Fc
    per_launch = {
        # our kernels' compulsory traffic per launch
        "sl_incstate_step": 11 * F,   # X 3F + gather src 1F + grad m 3F + vt 3F + write 1F
        "sl_adjoint_step": 6 * F,     # X 3F + gather src 1F + factor 1F + write 1F
        "sl_accumulate": (4 * (nt + 1) + 3) * F,
        "sl_pointwise": 7 * F,
        "fft_x3_r2c": F + Fc,
        "fft_axis": 2 * Fc,
        "fft_x1_mult": 2 * Fc,
        "fft_x3_c2r": Fc + 2 * F,     # spectrum in, add-field in, real out
    }
    return per_matvec, per_launch


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        # nvidia-smi needs ~0.2 s before its first line: wait for it here, outside the timed
        # region, so that even a short region (K x 6 ms) is covered by the 25 ms samples that
        # follow; the pre-roll line itself is only reported when no later sample exists
        self.pre = None
        if self.proc is not None:
            try:
                self.pre = self.proc.stdout.readline()
            except Exception:
                self.pre = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            p = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except (ValueError, IndexError):
                continue
            for nm, val in zip(names, p[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        out = {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
               "samples": len(sm), "reasons": sorted(reasons)}
        if not sm and getattr(self, "pre", None):  # region shorter than one sampling interval
            p = [x.strip() for x in self.pre.split(",")]
            try:
                out.update(sm_mhz=float(p[0]), sm_max_mhz=float(p[1]), pre_roll_sample=True,
                           reasons=sorted(nm for nm, val in zip(names, p[3:7]) if val.lower() == "active"))
            except (ValueError, IndexError):
                pass
        return out


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
def run_reference_matvecs(m_R, m_T, v, vt, nt, steps, warmup, budget_s):
    """Reference CPU arm: the compiled reference (oracle/_ref) on the host cores."""
    from oracle import ref  # the reference only: never maps libveloreg_gpu.so
    cores = os.cpu_count() or 1
    ref.set_workers(cores)
    model = ref.make_model("h2", beta_v=1e-2, nt=nt)
    t0 = time.perf_counter()
    obj = ref.Objective(m_R, m_T, model)
    s = obj.evaluate(v)
    obj.compute_gradient(s)
    setup = time.perf_counter() - t0
    for _ in range(warmup):
        obj.hessian_matvec(s, vt)
    times = []
    t_start = time.perf_counter()
    for _ in range(max(1, steps)):
        t = time.perf_counter()
        obj.hessian_matvec(s, vt)
        times.append(time.perf_counter() - t)
        if time.perf_counter() - t_start > budget_s:
            break
    total = sum(times)
    return {"value": len(times) / total, "steps": len(times), "seconds": total, "cores": cores,
            "setup_s": setup}


def reference_detail(m_T, v, vt, m_R, nt, n, with_solves=True, with_config3=False):
    """BASELINE.md section 3 for the reference CPU arm (same box, same run): the shim-FFT
    time split at the bench grid, 1-worker vs all-worker matvec at 128^3 (a bounded sample),
    and the reference's full GN solves at configs 1-3 (config 3: beta continuation)."""
    from oracle import ref  # the reference only: never maps libveloreg_gpu.so
    cores = os.cpu_count() or 1
    out = {"cores": cores}
    ref.set_workers(cores)
    t0 = time.perf_counter()
    spec = ref.fft_forward(m_T)
    t1 = time.perf_counter()
    ref.fft_inverse(spec, m_T.shape)
    t2 = time.perf_counter()
    # a production single-threaded FFT for comparison: numpy's pocketfft (FFTW's layout and
    # normalisation), the same r2c / c2r pair on the same field
    t3 = time.perf_counter()
    sp2 = np.fft.rfftn(m_T)
    t4 = time.perf_counter()
    np.fft.irfftn(sp2, s=m_T.shape, axes=(0, 1, 2))
    t5 = time.perf_counter()
    shim_pair, pocket_pair = (t1 - t0) + (t2 - t1), (t4 - t3) + (t5 - t4)
    out["fft"] = {"grid": n, "r2c_s": t1 - t0, "c2r_s": t2 - t1,
                  "per_matvec_transforms": 46, "per_matvec_fft_s_estimate": 23 * shim_pair,
                  "pocketfft_r2c_s": t4 - t3, "pocketfft_c2r_s": t5 - t4,
                  "per_matvec_fft_s_pocketfft_estimate": 23 * pocket_pair,
                  "note": "oracle FFT = the from-scratch FFTW3-API shim (radix-2, long-double twiddles), "
                          "single-threaded as the reference's plan cache is (fft.cpp:56-83); pocketfft "
                          "(numpy, one thread) times the same transforms as a stand-in for FFTW, which is "
                          "absent here"}
    del spec, sp2
    # 1 worker vs all workers on the 128^3 config-2 problem (one matvec each)
    n2 = 128
    mR2, mT2, vs2 = ref.generate_synthetic((n2, n2, n2), nt)
    model = ref.make_model("h2", beta_v=1e-2, nt=nt)
    vt2 = ref.random_smooth_vector((n2, n2, n2), 2, 142, 1.0)
    res = {}
    for w in (cores, 1):
        ref.set_workers(w)
        obj = ref.Objective(mR2, mT2, model)
        st = obj.evaluate(vs2)
        obj.compute_gradient(st)
        t0 = time.perf_counter()
        obj.hessian_matvec(st, vt2)
        res[w] = time.perf_counter() - t0
    ref.set_workers(cores)
    out["matvec_128"] = {"workers_all_s": res[cores], "workers_1_s": res[1], "speedup": res[1] / res[cores]}
    if with_solves:
        solves = {}
        for name, (a, b) in (("config1_64", ref.generate_synthetic((64,) * 3, nt)[:2]),
                             ("config2_128", (mR2, mT2))):
            p = _ref_params(ref)
            t0 = time.perf_counter()
            _, rep, _ = ref.gauss_newton_solve(a, b, np.zeros((3,) + a.shape), model, p)
            solves[name] = {"seconds": time.perf_counter() - t0, "newton_iterations": rep["outer_iterations"],
                            "final_mismatch_rel": rep["final_mismatch_rel"]}
        if with_config3:
            p = _ref_params(ref)
            t0 = time.perf_counter()
            _, reps, _ = ref.parameter_continuation(m_R, m_T, np.zeros_like(v), model, p)
            solves[f"config3_{n}_beta_continuation"] = {
                "seconds": time.perf_counter() - t0, "newton_iterations": [r["outer_iterations"] for r in reps],
                "final_mismatch_rel": reps[-1]["final_mismatch_rel"], "final_grad_rel": reps[-1]["final_grad_rel"]}
        else:
            solves[f"config3_{n}_beta_continuation"] = {
                "seconds": None, "note": "run with --ref-solve3 (393 s on this pool's 16 host cores: "
                                         "profiles/r02_bench_reference.json; results pinned in "
                                         "tests/golden/config3_solve.npz)"}
        out["gn_solves"] = solves
    return out


def _ref_params(ref):
    """SolverParams (solver.hpp:13-33) with the configs' eps_opt = 1e-2."""
    p = ref.SolverParams()
    p.eps_opt, p.abs_grad_tol, p.max_newton, p.max_krylov = 1e-2, 1e-6, 50, 100
    p.armijo_c1, p.armijo_backtrack, p.armijo_max_trials, p.squared_norm_stop = 1e-4, 0.5, 20, 1
    return p


def fp32_block(ctx, V, d_v, d_mT, nt, dev, torch):
    """fp32 lane micro-benchmark at the bench grid: one tricubic gather of a scalar (a state
    step) and of the 3 velocity components at the backward departure points, fp32 vs fp64."""
    L = V._lib
    N = ctx.N
    x = ctx.empty(3)
    L.call("vr_trace_characteristics", ctx.handle, d_v.ptr, nt, 0, x.ptr)
    xf = V.DeviceBufferF32.from_host(ctx, x.numpy())
    mf = V.DeviceBufferF32.from_host(ctx, d_mT.numpy())
    vf = V.DeviceBufferF32.from_host(ctx, d_v.numpy())
    o1, o3 = ctx.empty(1), ctx.empty(3)
    of1, of3 = V.DeviceBufferF32(ctx, N), V.DeviceBufferF32(ctx, 3 * N)
    ops = {
        "state_step_f64": lambda: L.call("vr_tricubic_interpolate", ctx.handle, d_mT.ptr, x.ptr, o1.ptr, 1),
        "state_step_f32": lambda: L.call("vr_tricubic_interpolate_f32", ctx.handle, mf.ptr, xf.ptr, of1.ptr, 1),
        "velocity_3_fields_f64": lambda: L.call("vr_tricubic_interpolate", ctx.handle, d_v.ptr, x.ptr, o3.ptr, 3),
        "velocity_3_fields_f32": lambda: L.call("vr_tricubic_interpolate_f32", ctx.handle, vf.ptr, xf.ptr,
                                                of3.ptr, 3),
    }
    st = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", dev))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    for name, fn in ops.items():
        for _ in range(3):
            fn()
        ctx.synchronize()
        e0.record(st)
        for _ in range(20):
            fn()
        e1.record(st)
        e1.synchronize()
        res[name + "_us"] = e0.elapsed_time(e1) / 20 * 1e3
    # the fp32 objective's GN Hessian matvec at the same state (composed, not yet fused)
    try:
        of = V.ObjectiveF32(ctx, d_mT.numpy(), d_mT.numpy(), V.make_model("h2", beta_v=1e-2, nt=nt))
        sf = of.evaluate(d_v.numpy())
        of.compute_gradient(sf)
        vt = V.DeviceBufferF32.from_host(ctx, d_v.numpy())
        out = V.DeviceBufferF32(ctx, 3 * N)
        mv = lambda: L.call("vr_hessian_matvec_f32", of._h, sf._h, vt.ptr, out.ptr)  # noqa: E731
        for _ in range(2):
            mv()
        ctx.synchronize()
        e0.record(st)
        for _ in range(10):
            mv()
        e1.record(st)
        e1.synchronize()
        res["matvec_f32_ms"] = e0.elapsed_time(e1) / 10
        res["matvec_f32_note"] = ("Objective<float> GN Hessian matvec at the generating velocity: fused fp32 sweep "
                                  "steps, beta_v A vt through fp64 scratch views")
        vt.free()
        out.free()
        sf.close()
        of.close()
    except Exception as exc:  # report, do not lose the line
        res["matvec_f32_ms"] = f"unavailable: {exc}"
    # the config-3 beta continuation in fp32 (device-resident fp32 images and initial guess)
    try:
        mR32 = V.DeviceBufferF32.from_host(ctx, V.solve_state(ctx, d_mT, d_v, nt).numpy()[nt])
        mT32 = V.DeviceBufferF32.from_host(ctx, d_mT.numpy())
        z32 = V.DeviceBufferF32.from_host(ctx, np.zeros((3,) + ctx.local_dims))
        runs, reps = [], None
        for _ in range(3):
            ctx.synchronize()
            t0 = time.perf_counter()
            vsol, reps, _ = V.parameter_continuation_f32(ctx, mR32, mT32, z32, V.make_model("h2", beta_v=1e-2, nt=nt),
                                                         V.make_params(eps_opt=1e-2))
            ctx.synchronize()
            runs.append(time.perf_counter() - t0)
            vsol.free()
        res["config3_solve_f32"] = {"seconds": float(np.median(runs[1:])), "seconds_runs": runs,
                                    "newton_iterations": [r["outer_iterations"] for r in reps],
                                    "hessian_matvecs": sum(r["fine"]["hessian_matvecs"] for r in reps),
                                    "final_mismatch_rel": reps[-1]["final_mismatch_rel"],
                                    "final_grad_rel": reps[-1]["final_grad_rel"],
                                    "stop": reps[-1]["stop_name"],
                                    "note": "the reference's float semantics at 256^3: fp32 round-off of v, amplified "
                                            "by the H2 symbol |k|^4 (up to 2.4e9), floors the gradient near the "
                                            "tolerance, so the beta = 1 level may stall (DESIGN.md section 9)"}
        for b in (mR32, mT32, z32):
            b.free()
    except Exception as exc:
        res["config3_solve_f32"] = f"unavailable: {exc}"
    res["speedup_state_step"] = res["state_step_f64_us"] / res["state_step_f32_us"]
    res["speedup_3_fields"] = res["velocity_3_fields_f64_us"] / res["velocity_3_fields_f32_us"]
    res["note"] = "fp32 fields and departure points, fp64 weights and sums (the reference's float lane)"
    for b in (xf, mf, vf, of1, of3):
        b.free()
    return res


def config2_block(vr, V, dev, nt, model, torch, with_cpu=True):
    """BASELINE config 2: 128^3 section-4.2 problem. Per-operator GPU times (20 launches after
    3 warm-ups, CUDA events on the library stream, outputs preallocated) with algorithmic
    bytes, the reference's time for the same operator on the host cores, and the GN solve."""
    n = 128
    N = n ** 3
    F, Fc = 8.0 * N, 16.0 * n * n * (n // 2 + 1)
    c = vr.Context(n, device=dev)
    mR, mT, vs = V.generate_synthetic(c, nt)
    d_v, d_mT = c.to_device(vs), c.to_device(mT)
    d_f = c.to_device(mT)
    spec = c.empty(1, complex_spectrum=True)
    o1, o3, x = c.empty(1), c.empty(3), c.empty(3)
    L = V._lib
    L.call("vr_trace_characteristics", c.handle, d_v.ptr, nt, 0, x.ptr)  # RK2 departure points of v*
    ops = {
        "fft_r2c": (lambda: L.call("vr_fft_r2c", c.handle, d_f.ptr, spec.ptr), F + Fc),
        "fft_c2r": (lambda: L.call("vr_fft_c2r", c.handle, spec.ptr, o1.ptr), Fc + F),
        "gradient": (lambda: L.call("vr_gradient", c.handle, d_f.ptr, o3.ptr), 4 * F),
        "divergence": (lambda: L.call("vr_divergence", c.handle, d_v.ptr, o1.ptr), 4 * F),
        "leray": (lambda: L.call("vr_apply_projection", c.handle, d_v.ptr, o3.ptr, 1, 0.0, 0.0), 6 * F),
        "tricubic_3_fields": (lambda: L.call("vr_tricubic_interpolate", c.handle, d_v.ptr, x.ptr, o3.ptr, 3),
                              9 * F),
        "tricubic_1_field": (lambda: L.call("vr_tricubic_interpolate", c.handle, d_mT.ptr, x.ptr, o1.ptr, 1),
                             5 * F),
    }
    st = torch.cuda.ExternalStream(c.stream, device=torch.device("cuda", dev))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    for name, (fn, nbytes) in ops.items():
        for _ in range(3):
            fn()
        c.synchronize()
        e0.record(st)
        for _ in range(20):
            fn()
        e1.record(st)
        e1.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        res[name] = {"gpu_us": us, "bytes": nbytes, "gpu_GBps": nbytes / (us * 1e-6) / 1e9}
    params = V.make_params(eps_opt=1e-2)
    d_mR = c.to_device(mR)
    d_v0 = c.to_device(np.zeros((3, n, n, n)))
    t_runs = []
    for _ in range(2):
        c.synchronize()
        t0 = time.perf_counter()
        r = V.gauss_newton_solve(c, d_mR, d_mT, d_v0, model, params)
        c.synchronize()
        t_runs.append(time.perf_counter() - t0)
    solve = {"gpu_seconds": t_runs[-1], "gpu_seconds_first_run": t_runs[0],
             "newton_iterations": r.report["outer_iterations"],
             "hessian_matvecs": r.report["fine"]["hessian_matvecs"],
             "final_mismatch_rel": r.report["final_mismatch_rel"], "final_grad_rel": r.report["final_grad_rel"]}
    if with_cpu:
        try:
            from oracle import ref
            ref.set_workers(os.cpu_count() or 1)
            xh = x.numpy()
            sp = ref.fft_forward(mT)
            cpu_ops = {
                "fft_r2c": lambda: ref.fft_forward(mT),
                "fft_c2r": lambda: ref.fft_inverse(sp, (n, n, n)),
                "gradient": lambda: ref.gradient(mT),
                "divergence": lambda: ref.divergence(vs),
                "leray": lambda: ref.apply_projection(vs, 1),
                "tricubic_3_fields": lambda: ref.tricubic_interpolate(vs, xh),
                "tricubic_1_field": lambda: ref.tricubic_interpolate(mT, xh),
            }
            for name, fn in cpu_ops.items():
                fn()
                t0 = time.perf_counter()
                for _ in range(3):
                    fn()
                ms = (time.perf_counter() - t0) / 3 * 1e3
                res[name]["cpu_ms"] = ms
                res[name]["speedup"] = ms * 1e3 / res[name]["gpu_us"]
            t0 = time.perf_counter()
            _, rep_c, _ = ref.gauss_newton_solve(mR, mT, np.zeros((3, n, n, n)), model, params)
            solve.update({"cpu_reference_seconds": time.perf_counter() - t0,
                          "cpu_newton_iterations": rep_c["outer_iterations"],
                          "cpu_final_mismatch_rel": rep_c["final_mismatch_rel"], "cpu_cores": os.cpu_count()})
        except Exception as exc:
            solve["cpu_reference"] = f"unavailable: {exc}"
    c.close()
    return {"grid": n, "workload": "config2: 128^3 synthetic problem (synthetic.cpp:16-34), H2 beta_v=1e-2, "
            "n_t=4; operators on device-resident fields (tricubic at the RK2 departure points of v*)",
            "operators": res, "solve": solve}


def ref_memory_ok(n):
    """The reference keeps ~70 fp64 fields of the global grid (SURVEY 8(d) CPU baseline)."""
    need = 70 * 8 * n ** 3
    try:
        import psutil
        have = psutil.virtual_memory().available
    except Exception:
        have = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_AVPHYS_PAGES")
    return have >= need, need, have


def main():
    args = parse()
    rank, world, local = dist_env()
    nt = args.nt
    cid, n = config_for(world, args.n, args.config)

    if args.impl == "reference":
        if rank != 0:
            return 0
        # bounded sample: configs larger than --ref-sample-n (config 4 / 5 under torchrun) are
        # timed on the same workload at that grid and scaled by the point ratio (the reference's
        # cost is linear in N up to the FFT's log factor, so this favours the reference)
        n_full, n = n, min(n, args.ref_sample_n)
        scale = (n / n_full) ** 3
        ok, need, have = ref_memory_ok(n)
        if not ok:
            print(json.dumps({"impl": "reference", "unavailable": f"the reference needs ~{need / 2 ** 30:.0f} GiB of "
                              f"host RAM at {n}^3 (70 fp64 fields), {have / 2 ** 30:.0f} GiB available"}), flush=True)
            return 0
        m_T, v, vt, desc = workload(cid, n, nt)
        from oracle import ref  # the reference only: never maps libveloreg_gpu.so
        ref.set_workers(os.cpu_count() or 1)
        m_R = ref.solve_state(m_T, v, nt)[-1]
        r = run_reference_matvecs(m_R, m_T, v, vt, nt, args.steps, 0, args.ref_budget_s)
        sample = (f"{r['steps']} GN Hessian matvec(s) at {n}^3 after an untimed evaluate+gradient "
                  f"({r['setup_s']:.1f}s); capped at {args.ref_budget_s:.0f}s")
        if n != n_full:
            sample += (f"; the {n_full}^3 workload sampled at {n}^3 (same phantom / velocity parameters), "
                       f"matvec/s scaled by ({n}/{n_full})^3 = {scale:.4g}")
            r["value"] *= scale
            r["seconds"] /= scale
        detail = None
        if not args.no_ref_detail:
            detail = reference_detail(m_T, v, vt, m_R, nt, n, with_solves=(world == 1),
                                      with_config3=args.ref_solve3)
            f = detail["fft"]
            s_mv = r["seconds"] / r["steps"]
            detail["matvec_s_measured"] = s_mv
            detail["matvec_s_with_pocketfft_estimate"] = (s_mv - f["per_matvec_fft_s_estimate"]
                                                          + f["per_matvec_fft_s_pocketfft_estimate"])
        line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world, "steps": r["steps"],
                "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * r["seconds"] / r["steps"],
                "higher_is_better": True, "scaling": "weak" if world == 1 else "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": bench_config(cid, n_full, nt, world),
                "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "reference_detail": detail}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import paper_1808_04487_b200 as vr
    import paper_1808_04487_b200.veloreg as V

    dist = None
    slabs = world > 1 or args.force_slabs
    single = not slabs
    if slabs:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if "MASTER_ADDR" not in os.environ:  # --force-slabs outside torchrun: a one-rank group
            import socket
            with socket.socket() as sk:  # any free port
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = local

    model = V.make_model("h2", beta_v=1e-2, nt=nt)
    desc = workload_desc(cid, n, nt)
    scaling, comm_info = "weak", None
    if slabs:
        # x1 slabs over the ranks (NCCL all-to-all FFT transposes, P2P halos): one global
        # problem split across the GPUs, i.e. strong scaling. No fallback: any failure
        # raises on this rank and torchrun tears the job down.
        from paper_1808_04487_b200 import phantom

        def _red(x, op):
            t = torch.tensor([float(x)], dtype=torch.float64, device=f"cuda:{dev}")
            dist.all_reduce(t, op=op)
            return float(t.item())
        planes = n // world
        first = rank * planes
        m_T, v, vt, vmax1 = phantom.make_config_inputs_slab(
            cid, first, planes, n=n, allreduce_max=lambda x: _red(x, dist.ReduceOp.MAX),
            allreduce_min=lambda x: _red(x, dist.ReduceOp.MIN))
        # the halo covers the generating velocity with 30 % headroom: the solve's Armijo trials may
        # overshoot it, and a trial that needs more planes raises ResourceError (never clamps)
        halo = min(planes, max(V.slab_halo_required(vmax1, nt, n), V.slab_halo_required(1.3 * vmax1, nt, n)))
        uid = [V.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = V.DistContext(n, rank, world, uid[0], device=dev, halo=halo)
        assert (ctx.first_plane, ctx.planes) == (first, planes), "slab geometry mismatch"
        d_mT, d_v, d_vt = (ctx.to_device(a) for a in (m_T, v, vt))
        del m_T, v
        # m_R = m_T transported by v: the state history of an objective at v
        tmp = V.Objective(ctx, d_mT, d_mT, model)
        s0 = tmp.evaluate(d_v)
        d_mR = ctx.to_device(s0.m_history[nt])
        s0.close()
        tmp.close()
        scaling = "strong"
        comm_info = {"halo_planes": halo, "vmax_x1": vmax1, "planes_per_rank": planes}
    else:
        m_T, v, vt, desc = workload(cid, n, nt)
        ctx = vr.Context(n, device=dev)
        d_mT = ctx.to_device(m_T)
        d_v = ctx.to_device(v)
        d_vt = ctx.to_device(vt)
        hist = V.solve_state(ctx, d_mT, d_v, nt)                   # m_R = m_T transported by v
        d_mR = ctx.empty(1)
        _ = V._lib.call("vr_memcpy_d2d", ctx.handle, d_mR.ptr, hist.field(nt), 8 * ctx.N)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", dev))
    obj = V.Objective(ctx, d_mR, d_mT, model)
    mem0 = ctx.memory()
    st = obj.evaluate(d_v)
    obj.compute_gradient(st)
    out = ctx.empty(3)
    mem1 = ctx.memory()
    F_bytes = 8.0 * ctx.N
    memory = {"context_live_GiB": mem1["live_bytes"] / 2 ** 30,
              "eval_state_fields": (mem1["live_bytes"] - mem0["live_bytes"] - 3 * F_bytes) / F_bytes,
              "peak_GiB": mem1["peak_bytes"] / 2 ** 30,
              "pool_reserved_high_GiB": mem1["pool_reserved_high_bytes"] / 2 ** 30,
              "note": "library device allocations of this rank (vr_ctx_memory): images, objective workspace, "
                      "EvalState (v, X_bwd, m history, X_fwd, factor, grad m cache, gradient) and scratch"}

    for _ in range(max(3, args.warmup)):
        obj.hessian_matvec(st, d_vt, out=out)
    ctx.synchronize()

    # ---- timed region: device-resident inputs ------------------------------
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = ctx.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            obj.hessian_matvec(st, d_vt, out=out)
        e1.record(stream)
        e1.synchronize()
    launches = ctx.kernel_launches() - l0
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- per-kernel CUDA-event profile: a second pass of the same steps with
    # every kernel bracketed by events on its launch stream (side-stream work
    # serialised, so each interval is one kernel running alone) ------------------
    k_prof = max(3, min(args.steps, 20))
    ctx.set_profiling(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(k_prof):
        obj.hessian_matvec(st, d_vt, out=out)
    p1.record(stream)
    p1.synchronize()
    prof = ctx.profile_read()
    ctx.set_profiling(False)
    ms_prof = p0.elapsed_time(p1)
    ms_per_step = ms / args.steps
    per_step_units = 1  # one global matvec per step (slabs split it; one GPU does all of it)
    value = per_step_units * args.steps / (ms / 1e3)

    # ---- end to end through the public C ABI with host buffers -------------
    e2e = None
    if not args.no_e2e:
        nbytes = 3 * ctx.N * 8  # this rank's vt in / H vt out
        hp_in, hp_out = V.C.c_void_p(), V.C.c_void_p()
        V._lib.call("vr_host_alloc_pinned", nbytes, V.C.byref(hp_in))
        V._lib.call("vr_host_alloc_pinned", nbytes, V.C.byref(hp_out))
        h_in = np.ctypeslib.as_array((V.C.c_double * (3 * ctx.N)).from_address(hp_in.value))
        h_out = np.ctypeslib.as_array((V.C.c_double * (3 * ctx.N)).from_address(hp_out.value))
        h_in[:] = vt.ravel()  # this rank's slab (or the whole grid on one GPU)
        obj.hessian_matvec_host(st, h_in, h_out)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        k_e2e = max(3, min(args.steps, 50))  # enough steps for a stable pipelined rate
        # (1) synchronous calls: upload, matvec, download, one after the other
        e0.record(stream)
        for _ in range(k_e2e):
            obj.hessian_matvec_host(st, h_in, h_out)
        e1.record(stream)
        e1.synchronize()
        ms_sync = e0.elapsed_time(e1)
        # (2) pipelined calls (one GPU): step k+1's upload and step k's download overlap
        # the matvecs; wall clock from the first call to the wait that drains the last download
        ms_e2e, path = ms_sync, "vr_hessian_matvec_host (pinned host vt in, H vt out)"
        if scaling != "strong":
            obj.hessian_matvec_host_async(st, h_in, h_out)
            obj.wait()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for _ in range(k_e2e):
                obj.hessian_matvec_host_async(st, h_in, h_out)
            obj.wait()
            ms_e2e = (time.perf_counter() - t0) * 1e3
            path = ("vr_hessian_matvec_host_async x steps + vr_objective_wait (pinned host vt in, H vt "
                    "out; uploads / matvecs / downloads of consecutive steps overlap)")
        if dist is not None:
            t = torch.tensor([ms_e2e, ms_sync], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_e2e, ms_sync = float(t[0].item()), float(t[1].item())
        e2e = {"value": per_step_units * k_e2e / (ms_e2e / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": nbytes * world, "d2h_bytes_per_step": nbytes * world, "steps": k_e2e,
               "path": path, "value_synchronous_calls": per_step_units * k_e2e / (ms_sync / 1e3)}
        V._lib.call("vr_host_free_pinned", hp_in)
        V._lib.call("vr_host_free_pinned", hp_out)

    # ---- x1 slabs: 10 PCG iterations of the first Newton step ----
    pcg10 = None
    if slabs and not args.no_solve:
        d_zero = ctx.to_device(np.zeros((3,) + ctx.local_dims))
        s_zero = obj.evaluate(d_zero)
        obj.compute_gradient(s_zero)
        rhs = s_zero.get(V._lib.STATE_GRADIENT, host=False)
        V._lib.call("vr_scale", ctx.handle, rhs.ptr, 3, -1.0)
        V.pcg_solve(obj, s_zero, rhs, 1e-30, 2)  # warm-up
        ctx.synchronize()
        if dist is not None:
            dist.barrier()
        e0.record(stream)
        _, pst = V.pcg_solve(obj, s_zero, rhs, 1e-30, 10)
        e1.record(stream)
        e1.synchronize()
        ms_pcg = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms_pcg], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_pcg = float(t.item())
        b_pcg = 148.0 * 8 * n ** 3  # B_mv + 39 F + 6 F_c ~ 148 F per PCG iteration
        its = max(1, pst["iterations"])
        peak_pcg, _ = measured_peak()
        pcg10 = {"ms": ms_pcg, "iterations": pst["iterations"], "ms_per_iteration": ms_pcg / its,
                 "bytes_per_iteration": b_pcg,
                 "frac_of_aggregate_hbm": b_pcg / (ms_pcg / its / 1e3) / 1e9 / (peak_pcg * world),
                 "note": "first Newton step (v = 0), spectral preconditioner; device events, max over ranks"}
        s_zero.close()

    # ---- roofline of the dominant kernel ------------------------------------
    peak, peak_kind = measured_peak()
    per_matvec_bytes, per_launch = bytes_model(n, nt)
    share = ctx.N / float(n ** 3)  # this rank's fraction of the grid (1 unless slabs)
    per_launch = {k: b * share for k, b in per_launch.items()}
    kernels = {k: {"launches": c, "total_ms": t, "avg_ms": t / c if c else None,
                   "share": t / ms_prof if ms_prof else None} for k, (c, t) in prof.items()}
    dom = max((k for k in prof if k in per_launch), key=lambda k: prof[k][1], default=None)
    roof = None
    if dom is not None:
        c, t = prof[dom]
        avg_s = t / c / 1e3
        ach = per_launch[dom] / avg_s / 1e9
        traffic = None
        try:  # ncu-measured DRAM bytes per launch of this kernel (profiles/ncu_traffic.json)
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic = json.load(f).get(dom)
            if traffic is not None:
                traffic = traffic * share
        except Exception:
            traffic = None
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": traffic, "peak_source": peak_kind,
                "limiter": "L1 return path of the 64-node fp64 gathers: 64 B/clk/SM, 512 B per point = 0.46 ms "
                           "floor per gather at 256^3 (ncu: data-pipe wavefronts 79-85 %, DRAM 29 %)"
                           if dom.startswith("sl_") and "step" in dom else None,
                "bytes_per_launch": per_launch[dom], "avg_launch_ms": t / c}
    # x1 slabs: NCCL exchange time per matvec (all-to-all transposes + halos run on the
    # compute stream, so this is also the exposed communication time)
    comm = None
    if scaling == "strong":
        cats = {k: v for k, v in prof.items() if k.startswith("comm_")}
        comm_ms = sum(t for c, t in cats.values()) / k_prof
        compute_ms = sum(t for k, (c, t) in prof.items() if not k.startswith("comm_")) / k_prof
        comm = {"total_ms_per_matvec": comm_ms,
                "by_kind_ms_per_matvec": {k: t / k_prof for k, (c, t) in cats.items()},
                "compute_ms_per_matvec": compute_ms,
                "exposed_ms_per_matvec": max(0.0, ms_per_step - compute_ms),
                "note": "total / by kind from the serialised profile pass (every kernel and exchange "
                        "bracketed alone); exposed = timed ms per matvec (reg-term transposes and halos "
                        "overlapped with the sweeps) minus the serialised compute time", **(comm_info or {})}
    # per-matvec HBM bytes over the aggregate HBM bandwidth, plus (slabs) the
    # all-to-all and halo bytes over NVLink (900 GB/s per direction per GPU)
    nvl_bytes = 0.0
    if world > 1:
        Fc = 16.0 * n * n * (n // 2 + 1)
        nvl_bytes = 6 * Fc * (world - 1) / world ** 2 + 2 * nt * 2 * comm_info["halo_planes"] * n * n * 8
    t_roof = per_matvec_bytes / world / (peak * 1e9) + nvl_bytes / 900e9
    matvec_roof = {"bytes_per_matvec": per_matvec_bytes,
                   "achieved_GBps": per_matvec_bytes / (ms_per_step / 1e3) / 1e9,
                   "frac_of_peak": per_matvec_bytes / (ms_per_step / 1e3) / 1e9 / (peak * world),
                   "nvlink_bytes_per_gpu": nvl_bytes, "roofline_ms": t_roof * 1e3,
                   "frac_of_roofline": t_roof * 1e3 / ms_per_step}

    # ---- GN solve time (the metric's second half) ----------------------------
    solve = None
    if not args.no_solve:
        solve = {}
        # config 3: beta continuation 1 -> 1e-1 -> 1e-2, warm starts, eps_opt 1e-2; images,
        # initial guess and result device resident (host I/O is not solver time)
        params = V.make_params(eps_opt=1e-2)
        d_v0 = ctx.to_device(np.zeros((3,) + ctx.local_dims))  # device-resident initial guess
        t_runs, reps, solve_error = [], None, None
        try:
            for _ in range(6):  # the first run also grows the stream-ordered memory pool
                ctx.synchronize()
                t0 = time.perf_counter()
                vsol, reps, _ = V.parameter_continuation(ctx, d_mR, d_mT, d_v0, model, params)
                ctx.synchronize()
                t_runs.append(time.perf_counter() - t0)
        except vr.VelouregError as exc:
            # library errors are raised from rank-consistent data (all-reduced flags and norms), so
            # every rank lands here together; the matvec line above is still reported
            if single:
                raise
            solve_error = f"{type(exc).__name__}: {exc}"
        if solve_error is not None or reps is None:
            solve[f"config{cid}"] = {"grid": n, "error": solve_error, "seconds_runs": t_runs}
            reps = None
        t_solve = float(np.median(t_runs[1:])) if len(t_runs) > 1 else None  # median of the steady runs
        if reps is not None:
            solve[f"config{cid}"] = {
                "grid": n, "seconds": t_solve, "seconds_runs": t_runs, "levels": len(reps),
                "newton_iterations": [r["outer_iterations"] for r in reps],
                "hessian_matvecs": sum(r["fine"]["hessian_matvecs"] for r in reps),
                "pde_solves": sum(r["fine"]["pde_solves"] for r in reps),
                "final_mismatch_rel": reps[-1]["final_mismatch_rel"], "final_grad_rel": reps[-1]["final_grad_rel"],
                "stop": reps[-1]["stop_name"], "precond": "spectral", "continuation": "beta_v 1, 1e-1, 1e-2"}
        # the same continuation with the two-level preconditioner; one GPU only
        if (single or args.slab_two_level) and reps is not None:
            t2 = []
            for _ in range(6):  # first run: coarse context, plans and pool growth
                ctx.synchronize()
                t0 = time.perf_counter()
                _, reps2, _ = V.parameter_continuation(ctx, d_mR, d_mT, d_v0, model, params,
                                                       precond="two_level")
                ctx.synchronize()
                t2.append(time.perf_counter() - t0)
            solve[f"config{cid}_two_level"] = {
                "grid": n, "seconds": float(np.median(t2[1:])), "seconds_runs": t2, "levels": len(reps2),
                "newton_iterations": [r["outer_iterations"] for r in reps2],
                "fine_hessian_matvecs": sum(r["fine"]["hessian_matvecs"] for r in reps2),
                "coarse_hessian_matvecs": sum(r["coarse"]["hessian_matvecs"] for r in reps2),
                "final_mismatch_rel": reps2[-1]["final_mismatch_rel"],
                "final_grad_rel": reps2[-1]["final_grad_rel"], "stop": reps2[-1]["stop_name"],
                "precond": f"two-level, PCG(0.1) inner on the {n // 2}^3 coarse grid"}
    if not args.no_solve and single:
        # config 1: 64^3 analytic problem, GPU vs the reference on the host cores
        ctx1 = vr.Context(64, device=dev)
        mR1, mT1, _ = V.generate_synthetic(ctx1, nt)
        p1 = V.make_params(eps_opt=1e-2)
        t0 = time.perf_counter()
        r1 = V.gauss_newton_solve(ctx1, mR1, mT1, np.zeros((3, 64, 64, 64)), model, p1)
        t_gpu1 = time.perf_counter() - t0
        solve["config1"] = {"grid": 64, "gpu_seconds": t_gpu1,
                            "newton_iterations": r1.report["outer_iterations"],
                            "hessian_matvecs": r1.report["fine"]["hessian_matvecs"],
                            "final_mismatch_rel": r1.report["final_mismatch_rel"],
                            "final_grad_rel": r1.report["final_grad_rel"]}
        if rank == 0 and single and not args.no_cpu_baseline:
            try:
                from oracle import ref
                ref.set_workers(os.cpu_count() or 1)
                t0 = time.perf_counter()
                _, rep_c, _ = ref.gauss_newton_solve(mR1, mT1, np.zeros((3, 64, 64, 64)), model, p1)
                solve["config1"].update({"cpu_reference_seconds": time.perf_counter() - t0,
                                         "cpu_newton_iterations": rep_c["outer_iterations"],
                                         "cpu_final_mismatch_rel": rep_c["final_mismatch_rel"],
                                         "cpu_cores": os.cpu_count()})
            except Exception as exc:
                solve["config1"]["cpu_reference"] = f"unavailable: {exc}"
        ctx1.close()

    # ---- config 4 on one GPU: 512^3 phantom (|k| <= 10), the P = 1 point of the
    # strong-scaling curve; device-resident matvecs timed like the main line -----
    cfg4 = None
    if single and not args.no_config4 and n == 256:
        from paper_1808_04487_b200 import phantom
        n4 = phantom.CONFIGS[4]["n"]
        m_T4, v4 = phantom.make_config_inputs(4)
        vt4 = phantom.bandlimited_direction(n4)
        c4 = vr.Context(n4, device=dev)
        dT4, dv4, dvt4 = c4.to_device(m_T4), c4.to_device(v4), c4.to_device(vt4)
        del m_T4, v4, vt4
        h4 = V.solve_state(c4, dT4, dv4, nt)
        dR4 = c4.empty(1)
        V._lib.call("vr_memcpy_d2d", c4.handle, dR4.ptr, h4.field(nt), 8 * c4.N)
        h4.free()
        o4 = V.Objective(c4, dR4, dT4, model)
        s4 = o4.evaluate(dv4)
        o4.compute_gradient(s4)
        out4 = c4.empty(3)
        for _ in range(3):
            o4.hessian_matvec(s4, dvt4, out=out4)
        st4 = torch.cuda.ExternalStream(c4.stream, device=torch.device("cuda", dev))
        k4 = max(3, min(args.steps, 20))
        c4.synchronize()
        e0.record(st4)
        for _ in range(k4):
            o4.hessian_matvec(s4, dvt4, out=out4)
        e1.record(st4)
        e1.synchronize()
        ms4 = e0.elapsed_time(e1) / k4
        b4, _ = bytes_model(n4, nt)
        cfg4 = {"workload": f"config4 on one GPU: {n4}^3 ellipsoid phantom, band-limited v (|k|<=10, "
                            "max disp 0.08*2pi), GN Hessian matvec at v", "grid": n4, "steps": k4,
                "value": 1e3 / ms4, "unit": UNIT, "ms_per_step": ms4, "bytes_per_matvec": b4,
                "achieved_GBps": b4 / (ms4 / 1e3) / 1e9, "frac_of_peak": b4 / (ms4 / 1e3) / 1e9 / peak}
        s4.close()
        # 10 PCG iterations of the first Newton step (v = 0, beta_v 1e-2, spectral
        # preconditioner; SURVEY 8(d) row C5's unit, here on one GPU at 512^3)
        dv0 = c4.to_device(np.zeros((3, n4, n4, n4)))
        s0 = o4.evaluate(dv0)
        o4.compute_gradient(s0)
        rhs = s0.get(V._lib.STATE_GRADIENT, host=False)
        V._lib.call("vr_scale", c4.handle, rhs.ptr, 3, -1.0)
        V.pcg_solve(o4, s0, rhs, 1e-30, 2)  # warm-up
        c4.synchronize()
        e0.record(st4)
        _, pst = V.pcg_solve(o4, s0, rhs, 1e-30, 10)
        e1.record(st4)
        e1.synchronize()
        ms_pcg = e0.elapsed_time(e1)
        b_pcg = 148.0 * 8 * n4 ** 3  # B_mv + 39 F + 6 F_c ~ 148 F per PCG iteration
        cfg4["pcg_10_iterations"] = {"ms": ms_pcg, "iterations": pst["iterations"],
                                     "ms_per_iteration": ms_pcg / max(1, pst["iterations"]),
                                     "bytes_per_iteration": b_pcg,
                                     "frac_of_peak": b_pcg / (ms_pcg / max(1, pst["iterations"]) / 1e3) / 1e9 / peak,
                                     "note": "first Newton step (v = 0); PCG carries beta_v A s, so an iteration "
                                             "is a data matvec + the spectral preconditioner"}
        s0.close()
        o4.close()
        # the config-4 solve on one GPU (beta continuation, spectral preconditioner)
        c4.synchronize()
        t0 = time.perf_counter()
        _, reps4, _ = V.parameter_continuation(c4, dR4, dT4, dv0, model, V.make_params(eps_opt=1e-2))
        c4.synchronize()
        cfg4["gn_solve"] = {"seconds": time.perf_counter() - t0, "levels": len(reps4),
                            "newton_iterations": [r["outer_iterations"] for r in reps4],
                            "hessian_matvecs": sum(r["fine"]["hessian_matvecs"] for r in reps4),
                            "final_mismatch_rel": reps4[-1]["final_mismatch_rel"],
                            "final_grad_rel": reps4[-1]["final_grad_rel"], "stop": reps4[-1]["stop_name"],
                            "note": "single run (includes memory-pool growth)"}
        c4.close()

    # ---- fp32 lane: the same tricubic gathers at the config-3 departure
    # points with fp32 fields / points (fp64 stencil arithmetic), next to the fp64 kernel --
    f32 = None
    if single and not args.no_fp32:
        f32 = fp32_block(ctx, V, d_v, d_mT, nt, dev, torch)

    # ---- config 2 (128^3 analytic problem): per-operator micro-benchmarks and the full
    # GN solve, GPU (device-resident, CUDA events) next to the reference on the host cores --
    cfg2 = None
    if single and not args.no_config2:
        cfg2 = config2_block(vr, V, dev, nt, model, torch, with_cpu=not args.no_cpu_baseline)

    cpu = None
    if rank == 0 and single and not args.no_cpu_baseline:
        try:
            m_R_host = d_mR.numpy()
            r = run_reference_matvecs(m_R_host, m_T, v, vt, nt, 1, 0, 60.0)
            cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "reference",
                   "sample": f"1 GN Hessian matvec at {n}^3 by the compiled reference (oracle/_ref) after "
                             f"an untimed evaluate+gradient ({r['setup_s']:.1f}s)"}
        except Exception as exc:  # the oracle must be built; report instead of dying
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": bench_config(cid, n, nt, world),
                "e2e": e2e, "gpu_launches": launches, "roofline": roof, "matvec_roofline": matvec_roof,
                "kernels": kernels, "kernel_profile": {"steps": k_prof, "ms_per_step": ms_prof / k_prof,
                                                        "note": "separate serialised pass, events per kernel"},
                "cpu_baseline": cpu, "clocks": clk.summary(), "gn_solve": solve,
                "config4_single_gpu": cfg4, "config2": cfg2, "fp32_lane": f32, "comm": comm,
                "memory": memory, "forced_slabs": bool(args.force_slabs), "pcg_10_iterations": pcg10}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
