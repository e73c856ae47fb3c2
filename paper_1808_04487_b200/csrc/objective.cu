// objective.cu -- Objective<double> on the device (proj/src/objective.cpp:35-186)
// and the C++ host driver: PCG, Armijo, Gauss-Newton (proj/src/solver.cpp:23-269).
//
// The host driver keeps the reference's algorithm and constants verbatim
// (forcing min(0.5, sqrt(|g|/|g0|)), unweighted dots in PCG and the stop test,
// weighted inner product for the Armijo slope, squared-norm relative stop);
// every vector it touches stays in HBM and only scalars cross to the host.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <string>

#include <memory>

#include "objective.cuh"
#include "twolevel.cuh"

vr_state::~vr_state() {
    vr_ctx* ctx = obj ? obj->ctx : nullptr;
    if (!ctx) return;
    for (double* p : {v, xb, mhist, xf, factor, gradm, grad, vpad, lamhist}) vr::dev_free(ctx, p);
}

vr_objective::~vr_objective() {
    if (!ctx) return;
    for (double* p : {ws_lam, ws_tmp, ws_div, ws_b, host_vt, host_out}) vr::dev_free(ctx, p);
    if (pipe.h2d) {
        cudaStreamSynchronize(pipe.h2d);
        cudaStreamSynchronize(pipe.d2h);
        for (int q = 0; q < 2; ++q) {
            vr::dev_free(ctx, pipe.vt[q]);
            vr::dev_free(ctx, pipe.out[q]);
            cudaEventDestroy(pipe.up[q]);
            cudaEventDestroy(pipe.done[q]);
            cudaEventDestroy(pipe.down[q]);
        }
        cudaStreamDestroy(pipe.h2d);
        cudaStreamDestroy(pipe.d2h);
    }
}

namespace vr {

bool timing_enabled() {
    static const bool on = std::getenv("VR_TIMING") != nullptr;
    return on;
}
void slow_op(const char* what, double ms) {
    static const double thr = std::getenv("VR_SLOW_MS") ? std::atof(std::getenv("VR_SLOW_MS")) : 20.0;
    if (ms > thr) std::fprintf(stderr, "VR_TIMING slow %s: %.1f ms\n", what, ms);
}

double* dev_alloc(vr_ctx* ctx, long long n) {
    auto range = ctx->free_cache.equal_range(n);
    for (auto it = range.first; it != range.second; ++it) {
        if (it->second.second != ctx->stream) continue;
        double* p = it->second.first;
        ctx->free_cache.erase(it);
        mem_track_alloc(ctx, p, static_cast<long long>(sizeof(double)) * n);
        return p;
    }
    void* p = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaMallocAsync(&p, sizeof(double) * static_cast<size_t>(n), ctx->stream);
    if (timing_enabled())
        slow_op("cudaMallocAsync", std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    if (e != cudaSuccess) {
        cudaGetLastError();
        release_cache(ctx);  // give the cached buffers back and retry once
        e = cudaMallocAsync(&p, sizeof(double) * static_cast<size_t>(n), ctx->stream);
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw_resource("device allocation of " + std::to_string(sizeof(double) * n) +
                           " bytes failed: " + cudaGetErrorString(e));
        }
    }
    mem_track_alloc(ctx, p, static_cast<long long>(sizeof(double)) * n);
    return static_cast<double*>(p);
}
void dev_free(vr_ctx* ctx, double* p) {
    if (!p) return;
    auto it = ctx->mem_sizes.find(p);
    if (it != ctx->mem_sizes.end()) {
        const long long n = it->second / static_cast<long long>(sizeof(double));
        mem_track_free(ctx, p);
        ctx->free_cache.emplace(n, std::make_pair(p, ctx->stream));
        return;
    }
    cudaFreeAsync(p, ctx->stream);
}
void release_cache(vr_ctx* ctx) {
    for (auto& kv : ctx->free_cache) cudaFreeAsync(kv.second.first, kv.second.second);
    ctx->free_cache.clear();
}

void validate_model(const vr_model& m) {
    // RegNorm::validate (spectral.hpp:82-87), RegModel::validate (objective.hpp:18-22)
    if (m.norm.kind < VR_REG_H1 || m.norm.kind > VR_REG_HELMHOLTZ)
        throw_argument("RegNorm: unknown regularization kind");
    if (m.norm.kind == VR_REG_HELMHOLTZ && m.norm.gamma <= 0.0)
        throw_argument("RegNorm: helmholtz gamma must be > 0");
    if (m.norm.div_penalty && m.norm.beta_w <= 0.0)
        throw_argument("RegNorm: beta_w must be > 0 when the divergence penalty is on");
    if (m.beta_v <= 0.0) throw_argument("RegModel: beta_v must be > 0");
    if (m.nt < 1) throw_argument("RegModel: n_t must be >= 1");
    if (m.projection < VR_PROJ_IDENTITY || m.projection > VR_PROJ_NEAR_INCOMPRESSIBLE)
        throw_argument("RegModel: unknown projection kind");
}

void validate_params(const vr_solver_params& p) {
    // SolverParams::validate (solver.hpp:24-32)
    if (p.eps_opt <= 0 || p.abs_grad_tol <= 0 || p.armijo_c1 <= 0)
        throw_argument("SolverParams: tolerances must be > 0");
    if (p.max_newton < 1 || p.max_krylov < 1 || p.armijo_max_trials < 1)
        throw_argument("SolverParams: iteration limits must be >= 1");
    if (p.armijo_backtrack <= 0 || p.armijo_backtrack >= 1)
        throw_argument("SolverParams: backtracking factor must be in (0,1)");
}

// ---------------------------------------------------------------------------
// reductions with the reference's component order (field_ops.hpp:51-64,
// spectral.cpp:47-62)
// ---------------------------------------------------------------------------
static double cell_volume(const GridDims& g) { return g.h1 * g.h2 * g.h3; }

double dot_l2_vec(vr_ctx* ctx, const double* a, const double* b) {
    double r[3];
    dot_components(ctx, a, b, ctx->g.N, 3, r);
    double s = 0.0;
    for (int c = 0; c < 3; ++c) s += r[c];
    return s;
}
double norm_l2_vec(vr_ctx* ctx, const double* a) { return std::sqrt(dot_l2_vec(ctx, a, a)); }
double inner_product_vec(vr_ctx* ctx, const double* a, const double* b) {
    double r[3];
    dot_components(ctx, a, b, ctx->g.N, 3, r);
    const double vol = cell_volume(ctx->g);
    double s = 0.0;
    for (int c = 0; c < 3; ++c) s += r[c] * vol;
    return s;
}
double inner_product_scalar(vr_ctx* ctx, const double* a, const double* b) {
    double r;
    dot_components(ctx, a, b, ctx->g.N, 1, &r);
    return r * cell_volume(ctx->g);
}

// ---------------------------------------------------------------------------
// Objective
// ---------------------------------------------------------------------------
vr_objective* objective_create(vr_ctx* ctx, const double* mR, const double* mT,
                               const vr_model& model) {
    validate_model(model);
    auto* o = new vr_objective();
    o->ctx = ctx;
    o->mR = mR;
    o->mT = mT;
    o->model = model;
    const long long N = ctx->g.N;
    try {
        o->ws_lam = dev_alloc(ctx, (model.nt + 1) * ctx->hstride);
        o->ws_tmp = dev_alloc(ctx, 2 * ctx->hstride);
        o->ws_div = dev_alloc(ctx, ctx->hstride);
        o->ws_b = dev_alloc(ctx, 3 * N);
        // initial_mismatch_ = <m_T - m_R, m_T - m_R>_h (objective.cpp:40-44)
        o->initial_mismatch = sum_sq_diff(ctx, mT, mR, N) * cell_volume(ctx->g);
    } catch (...) {
        delete o;
        throw;
    }
    return o;
}

// ---- halo-padded fields (x1 slabs) -------------------
// A field that is a gather source is stored with `halo` planes on each side:
// slice j of a padded series starts at base + j*hstride, its interior at +hoff.
// On one GPU hstride = N and hoff = 0, i.e. the plain layout.
long long hoff(const vr_ctx* ctx) {
    return static_cast<long long>(ctx->g.halo) * ctx->g.n2 * ctx->g.n3;
}
double* pslice(const vr_ctx* ctx, double* base, int j) {
    return base + j * ctx->hstride + hoff(ctx);
}
void exchange(vr_ctx* ctx, double* interior) {
    if (ctx->dist)
        ctx->dist->halo(ctx, interior, static_cast<size_t>(ctx->g.n2) * ctx->g.n3, ctx->g.L,
                        ctx->g.halo);
}

// One semi-Lagrangian step whose gather source `src` needs its halo (SURVEY 8(e)
// "Overlap"): on x1 slabs with a concurrent-capable transport the halo exchange runs on
// the side stream while the step runs on the interior planes [H, L - H) -- whose stencils
// stay inside the slab, since H >= the x1 displacement + 4 -- and the two boundary bands
// run once the halo has arrived. `launch` issues the step on ctx->stream over the plane
// window in ctx->g (z0, zn). Elsewhere: exchange, then one launch over all planes.
template <class Launch>
void step_with_halo(vr_ctx* ctx, double* src, Launch&& launch) {
    GridDims& g = ctx->g;
    const int L = g.L, H = g.halo;
    // VR_OVERLAP_HALO=0/1 overrides the context's overlap switch for this mechanism alone
    static const int halo_env = [] {
        const char* e = std::getenv("VR_OVERLAP_HALO");
        return e ? std::atoi(e) : -1;
    }();
    const bool overlap = halo_env < 0 ? ctx->overlap : halo_env != 0;
    if (!ctx->dist || !overlap || !ctx->dist->side_stream_ok() || ctx->profiling || L <= 2 * H) {
        exchange(ctx, src);
        launch();
        return;
    }
    VR_CUDA(cudaEventRecord(ctx->ev_halo_fork, ctx->stream));
    VR_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_halo_fork, 0));
    cudaStream_t main = ctx->stream;
    ctx->stream = ctx->side;
    try {
        exchange(ctx, src);
    } catch (...) {
        ctx->stream = main;
        throw;
    }
    ctx->stream = main;
    VR_CUDA(cudaEventRecord(ctx->ev_halo, ctx->side));
    struct Window {  // restores the full plane range on exit
        GridDims& g;
        ~Window() { g.z0 = 0, g.zn = g.L; }
    } restore{g};
    g.z0 = H, g.zn = L - 2 * H;
    launch();
    VR_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
    g.z0 = 0, g.zn = H;
    launch();
    g.z0 = L - H, g.zn = H;
    launch();
}
// The per-call device flags: [0] non-finite direction, [1] departure beyond halo. They
// are sticky and reset whenever they are read. A matvec inside the solver does not
// synchronise for them: it marks them pending (defer_flags) and the next reduction
// (PCG's s.Hs) copies them back together with its result, raising the same error one
// reduction later; public entry points drain them before returning.
namespace {
void raise_flags(vr_ctx* ctx, const char* what) {
    double f[2] = {static_cast<double>(ctx->flag_host[0]), static_cast<double>(ctx->flag_host[1])};
    if (ctx->dist) ctx->dist->allreduce(ctx, f, 2, true);
    if (f[0] != 0.0 || f[1] != 0.0)
        VR_CUDA(cudaMemsetAsync(ctx->flag_dev, 0, 2 * sizeof(int), ctx->stream));
    if (f[1] != 0.0)
        throw_resource(std::string(what) + ": departure points beyond the x1 halo of " +
                       std::to_string(ctx->g.halo) + " planes (use a wider halo or fewer ranks)");
    if (f[0] != 0.0) throw_numeric(std::string(what) + ": non-finite direction");
}
}  // namespace

void check_flags(vr_ctx* ctx, const char* what) {
    ctx->flags_pending = nullptr;
    VR_CUDA(cudaMemcpyAsync(ctx->flag_host, ctx->flag_dev, 2 * sizeof(int), cudaMemcpyDeviceToHost,
                            ctx->stream));
    VR_CUDA(cudaStreamSynchronize(ctx->stream));
    raise_flags(ctx, what);
}
void defer_flags(vr_ctx* ctx, const char* what) {
    if (!ctx->flags_pending) ctx->flags_pending = what;
}
void drain_flags(vr_ctx* ctx) {
    if (ctx->flags_pending) check_flags(ctx, ctx->flags_pending);
}
void flags_enqueue_copy(vr_ctx* ctx) {
    if (ctx->flags_pending)
        VR_CUDA(cudaMemcpyAsync(ctx->flag_host, ctx->flag_dev, 2 * sizeof(int),
                                cudaMemcpyDeviceToHost, ctx->stream));
}
void flags_after_sync(vr_ctx* ctx) {
    if (!ctx->flags_pending) return;
    const char* what = ctx->flags_pending;
    ctx->flags_pending = nullptr;
    raise_flags(ctx, what);
}

vr_state* objective_evaluate(vr_objective* o, const double* v3) {
    Range nvtx("evaluate");
    vr_ctx* ctx = o->ctx;
    const GridDims& g = ctx->g;
    const long long N = g.N;
    const int nt = o->model.nt;
    if (!all_finite(ctx, v3, 3 * N)) throw_numeric("evaluate_objective: non-finite velocity");

    auto* s = new vr_state();
    s->obj = o;
    s->nt = nt;
    try {
        drain_flags(ctx);
        VR_CUDA(cudaMemsetAsync(ctx->flag_dev, 0, 2 * sizeof(int), ctx->stream));
        s->v = dev_alloc(ctx, 3 * N);
        s->xb = dev_alloc(ctx, 3 * N);
        s->mhist = dev_alloc(ctx, (nt + 1) * ctx->hstride);
        VR_CUDA(cudaMemcpyAsync(s->v, v3, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice,
                                ctx->stream));
        const double* vg = s->v;  // gather source of the RK2 midpoint step
        long long vstride = N;
        if (ctx->dist) {
            // the departure points of this velocity must stay within the halo
            const double vmax = max_abs(ctx, v3, N);  // |v_1|, all ranks
            const int need = halo_required(vmax, nt, g.n1);
            if (need > g.halo)
                throw_resource("evaluate: x1 displacement needs a halo of " +
                               std::to_string(need) + " planes, ctx has " +
                               std::to_string(g.halo));
            s->vpad = dev_alloc(ctx, 3 * ctx->hstride);
            for (int c = 0; c < 3; ++c) {
                VR_CUDA(cudaMemcpyAsync(pslice(ctx, s->vpad, c), v3 + c * N, sizeof(double) * N,
                                        cudaMemcpyDeviceToDevice, ctx->stream));
                exchange(ctx, pslice(ctx, s->vpad, c));
            }
            vg = pslice(ctx, s->vpad, 0);
            vstride = ctx->hstride;
        }
        sl_trace(ctx, vg, vstride, nt, VR_TRACE_BACKWARD, s->xb);
        // solve_state (transport.cpp:72-79)
        VR_CUDA(cudaMemcpyAsync(pslice(ctx, s->mhist, 0), o->mT, sizeof(double) * N,
                                cudaMemcpyDeviceToDevice, ctx->stream));
        for (int j = 0; j < nt; ++j)
            step_with_halo(ctx, pslice(ctx, s->mhist, j), [&] {
                sl_advect(ctx, pslice(ctx, s->mhist, j), s->xb, pslice(ctx, s->mhist, j + 1));
            });
        o->counters.pde_solves += 1;

        s->mismatch = sum_sq_diff(ctx, pslice(ctx, s->mhist, nt), o->mR, N) * cell_volume(g);
        s->mismatch_rel = o->initial_mismatch > 0.0 ? s->mismatch / o->initial_mismatch : 0.0;

        // reg = 1/2 beta_v <A v, v>_h with A applied at beta = 1 (objective.cpp:63-64);
        // on one GPU by Parseval on the forward spectra (no inverse transforms)
        double reg;
        if (!ctx->dist) {
            reg = 0.5 * o->model.beta_v * reg_energy(ctx, v3, o->model.norm);
        } else {
            double* Av = o->ws_b;
            op_reg(ctx, v3, Av, o->model.norm, VR_REGOP_APPLY, 1.0);
            reg = 0.5 * o->model.beta_v * inner_product_vec(ctx, Av, v3);
        }
        double penalty = 0.0;
        if (o->model.norm.div_penalty) {
            double* w = pslice(ctx, o->ws_tmp, 0);
            double* hw = pslice(ctx, o->ws_tmp, 1);
            op_divergence(ctx, v3, w);
            MultParams mp;
            mp.kind = Mult::helmholtz1;
            spectral_scalar_op(ctx, w, hw, mp);
            penalty = 0.5 * o->model.norm.beta_w * inner_product_scalar(ctx, hw, w);
        }
        s->objective = 0.5 * s->mismatch + reg + penalty;
        if (!std::isfinite(s->objective))
            throw_numeric("evaluate_objective: objective is not finite");
        if (ctx->dist) check_flags(ctx, "evaluate_objective");
    } catch (...) {
        delete s;
        throw;
    }
    o->counters.objective_evals += 1;
    return s;
}

// prepare_adjoint_ctx (objective.cpp:77-84) + the grad m_j cache
static void prepare_adjoint_ctx(vr_objective* o, vr_state* s) {
    if (s->has_adjoint_ctx) return;
    Range nvtx("prepare_adjoint_ctx");
    vr_ctx* ctx = o->ctx;
    const long long N = ctx->g.N;
    const int nt = s->nt;
    const double dt = 1.0 / nt;
    if (!s->xf) s->xf = dev_alloc(ctx, 3 * N);
    if (!s->factor) s->factor = dev_alloc(ctx, N);
    if (!s->gradm) s->gradm = dev_alloc(ctx, 3LL * (nt + 1) * N);
    drain_flags(ctx);
    VR_CUDA(cudaMemsetAsync(ctx->flag_dev, 0, 2 * sizeof(int), ctx->stream));
    if (ctx->dist)
        sl_trace(ctx, pslice(ctx, s->vpad, 0), ctx->hstride, nt, VR_TRACE_FORWARD, s->xf);
    else
        sl_trace(ctx, s->v, N, nt, VR_TRACE_FORWARD, s->xf);
    double* div_v = pslice(ctx, o->ws_div, 0);
    op_divergence(ctx, s->v, div_v);
    exchange(ctx, div_v);
    sl_factor(ctx, div_v, s->xf, 0.5 * dt, s->factor);
    for (int j = 0; j <= nt; ++j)
        op_gradient(ctx, pslice(ctx, s->mhist, j), s->gradm + 3LL * j * N);
    s->has_adjoint_ctx = true;
}

// An evaluation context assembled from given v and m history (the coarse
// state of TwoLevelContext::rebuild, precond.cpp:177-196): backward
// characteristics traced here, the adjoint context (X_fwd, factor, grad m
// cache) built as for a gradient. One GPU.
vr_state* state_from_history(vr_objective* o, const double* v3, const double* mhist, int nt,
                             const double* lamhist) {
    vr_ctx* ctx = o->ctx;
    const long long N = ctx->g.N;
    auto* s = new vr_state();
    s->obj = o;
    s->nt = nt;
    try {
        drain_flags(ctx);
        VR_CUDA(cudaMemsetAsync(ctx->flag_dev, 0, 2 * sizeof(int), ctx->stream));
        s->v = dev_alloc(ctx, 3 * N);
        s->xb = dev_alloc(ctx, 3 * N);
        s->mhist = dev_alloc(ctx, (nt + 1) * ctx->hstride);
        VR_CUDA(cudaMemcpyAsync(s->v, v3, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice,
                                ctx->stream));
        for (int j = 0; j <= nt; ++j)
            VR_CUDA(cudaMemcpyAsync(pslice(ctx, s->mhist, j), mhist + j * N, sizeof(double) * N,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
        if (ctx->dist) {  // as objective_evaluate: halo check, halo-padded gather copy of v
            const double vmax = max_abs(ctx, v3, N);
            const int need = halo_required(vmax, nt, ctx->g.n1);
            if (need > ctx->g.halo)
                throw_resource("state_from_history: x1 displacement needs a halo of " +
                               std::to_string(need) + " planes, ctx has " + std::to_string(ctx->g.halo));
            s->vpad = dev_alloc(ctx, 3 * ctx->hstride);
            for (int c = 0; c < 3; ++c) {
                VR_CUDA(cudaMemcpyAsync(pslice(ctx, s->vpad, c), v3 + c * N, sizeof(double) * N,
                                        cudaMemcpyDeviceToDevice, ctx->stream));
                exchange(ctx, pslice(ctx, s->vpad, c));
            }
            sl_trace(ctx, pslice(ctx, s->vpad, 0), ctx->hstride, nt, VR_TRACE_BACKWARD, s->xb);
        } else {
            sl_trace(ctx, s->v, N, nt, VR_TRACE_BACKWARD, s->xb);
        }
        prepare_adjoint_ctx(o, s);
        if (lamhist) {
            s->lamhist = dev_alloc(ctx, (nt + 1) * ctx->hstride);
            for (int j = 0; j <= nt; ++j)
                VR_CUDA(cudaMemcpyAsync(pslice(ctx, s->lamhist, j), lamhist + j * N,
                                        sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
        }
        if (ctx->dist) check_flags(ctx, "state_from_history");
    } catch (...) {
        delete s;
        throw;
    }
    return s;
}

void objective_gradient(vr_objective* o, vr_state* s) {
    Range nvtx("compute_gradient");
    vr_ctx* ctx = o->ctx;
    const long long N = ctx->g.N;
    prepare_adjoint_ctx(o, s);
    const int nt = s->nt;
    const double dt = 1.0 / nt;
    if (!s->grad) s->grad = dev_alloc(ctx, 3 * N);
    on_side_stream(ctx, [&] {  // beta_v A v overlaps the adjoint sweep
        op_reg_begin(ctx, s->v, o->model.norm, VR_REGOP_APPLY, o->model.beta_v);
    });

    // terminal lambda = m_R - m_nt and the observer at j = nt (objective.cpp:91-99); the
    // full-Newton Hessian needs every lambda_j (keep_hist, objective.cpp:100-102)
    // The sweep keeps every lambda_j (the objective's workspace, or the state's history
    // for full Newton) and one pass then accumulates b = sum_{j = nt..0} (w_j lambda_j)
    // grad m_j in the observer order -- cheaper than accumulating inside each gather
    // step (0.80 vs 0.60 ms per step at 256^3 for a 0.43 ms pass).
    const bool keep_hist = !o->model.gauss_newton;
    if (keep_hist && !s->lamhist) s->lamhist = dev_alloc(ctx, (nt + 1) * ctx->hstride);
    double* hist = keep_hist ? s->lamhist : o->ws_lam;
    double* b = o->ws_b;
    sl_grad_terminal(ctx, o->mR, pslice(ctx, s->mhist, nt), s->gradm + 3LL * nt * N, 0.5 * dt,
                     pslice(ctx, hist, nt), nullptr);
    for (int j = nt - 1; j >= 0; --j)
        step_with_halo(ctx, pslice(ctx, hist, j + 1), [&] {
            sl_adjoint_step(ctx, pslice(ctx, hist, j + 1), s->xf, s->factor, pslice(ctx, hist, j),
                            nullptr, 0.0, nullptr);
        });
    sl_accumulate(ctx, pslice(ctx, hist, 0), s->gradm, nt, dt, b);
    o->counters.pde_solves += 1;
    if (ctx->dist) check_flags(ctx, "compute_gradient");
    if (o->model.projection != VR_PROJ_IDENTITY)
        op_projection(ctx, b, b, o->model.projection, o->model.beta_v, o->model.norm.beta_w);
    // g = b + beta_v A v (objective.cpp:106-110), the add fused into the c2r epilogue
    join_side(ctx);
    op_reg_finish(ctx, s->grad, b);
    s->has_gradient = true;
    o->counters.gradient_evals += 1;
}

// hessian_data_matvec (objective.cpp:123-156) [+ beta_v A vt, objective.cpp:114-121]
void objective_matvec(vr_objective* o, const vr_state* s, const double* vt3, double* out3,
                      bool add_reg, const double* reg_given, bool check) {
    Range nvtx(add_reg || reg_given ? "hessian_matvec" : "hessian_data_matvec");
    vr_ctx* ctx = o->ctx;
    const long long N = ctx->g.N;
    if (!s->has_adjoint_ctx)
        throw_logic("hessian_matvec: evaluation context is missing the adjoint sweep data "
                    "(compute the gradient first)");
    const int nt = s->nt;
    const double dt = 1.0 / nt;
    const double hdt = 0.5 / nt;
    if (check && !ctx->flags_pending)  // stale flags of an unchecked call must not surface here
        VR_CUDA(cudaMemsetAsync(ctx->flag_dev, 0, 2 * sizeof(int), ctx->stream));
    // beta_v A vt depends only on vt: its FFT passes (HBM-bound) run on the side
    // stream under the L1-bound transport sweeps; only the c2r + add waits for b
    if (add_reg)
        on_side_stream(ctx, [&] {
            op_reg_begin(ctx, vt3, o->model.norm, VR_REGOP_APPLY, o->model.beta_v);
        });

    // incremental state (transport.cpp:150-173), terminal = -mt_nt into lam[nt]
    double* tmp[2] = {pslice(ctx, o->ws_tmp, 0), pslice(ctx, o->ws_tmp, 1)};
    double* lam0 = pslice(ctx, o->ws_lam, 0);
    auto lam = [&](int j) { return pslice(ctx, o->ws_lam, j); };
    double* b = o->ws_b;
    const bool identity_K = o->model.projection == VR_PROJ_IDENTITY;
    // full Newton (transport.cpp:192-226, objective.cpp:146-147): mt history and its
    // gradients, sources r_j = div(lambda_j vt), two-field inc-adjoint steps
    const bool full = !o->model.gauss_newton;
    if (full && !s->lamhist)
        throw_logic("hessian_matvec: full Newton mode needs the adjoint history");
    struct Scratch {
        vr_ctx* c;
        double *mt = nullptr, *gmt = nullptr, *rh = nullptr, *lv = nullptr;
        ~Scratch() {
            for (double* p : {mt, gmt, rh, lv}) dev_free(c, p);
        }
    } fn{ctx};
    if (full) {
        fn.mt = dev_alloc(ctx, (nt + 1) * N);
        fn.gmt = dev_alloc(ctx, 3LL * (nt + 1) * N);
        fn.rh = dev_alloc(ctx, (nt + 1) * ctx->hstride);
        fn.lv = dev_alloc(ctx, 3 * N);
        VR_CUDA(cudaMemsetAsync(fn.mt, 0, sizeof(double) * N, ctx->stream));  // mt_0 = 0
    }
    // fused: b accumulates inside the sweep (observer order j = nt..0), lam_j ping-pongs
    const bool fused = ctx->fuse_acc && !full;
    sl_incstate_first(ctx, s->gradm, vt3, hdt, tmp[0]);
    int cur = 0;
    for (int j = 0; j < nt; ++j) {
        const bool last = (j + 1 == nt);
        step_with_halo(ctx, tmp[cur], [&] {
            if (last && fused)
                sl_incstate_step(ctx, tmp[cur], s->xb, s->gradm + 3LL * nt * N, vt3, hdt, lam(1), 2, b,
                                 0.5 * dt);
            else
                sl_incstate_step(ctx, tmp[cur], s->xb, s->gradm + 3LL * (j + 1) * N, vt3, hdt,
                                 last ? lam(nt) : tmp[cur ^ 1], last ? 1 : 0, nullptr, 0.0,
                                 full ? fn.mt + (j + 1) * N : nullptr);
        });
        cur ^= 1;
    }
    o->counters.pde_solves += 1;
    if (full) {
        for (int j = 0; j <= nt; ++j) {
            op_gradient(ctx, fn.mt + j * N, fn.gmt + 3LL * j * N);
            sl_scale_vec(ctx, pslice(ctx, s->lamhist, j), vt3, fn.lv);
            op_divergence(ctx, fn.lv, pslice(ctx, fn.rh, j));
        }
    }
    // incremental adjoint, Gauss-Newton branch = plain continuity sweep (transport.cpp:188-190)
    bool out_done = false;
    if (full) {
        for (int j = nt - 1; j >= 0; --j) {
            exchange(ctx, lam(j + 1));
            exchange(ctx, pslice(ctx, fn.rh, j + 1));
            sl_adjoint_fn_step(ctx, lam(j + 1), pslice(ctx, fn.rh, j + 1), s->xf, s->factor,
                               pslice(ctx, fn.rh, j), hdt, lam(j));
        }
        const double* lam2 = pslice(ctx, s->lamhist, 0);
        if (reg_given && identity_K) {
            sl_accumulate(ctx, lam0, s->gradm, nt, dt, out3, reg_given, lam2, fn.gmt);
            out_done = true;
        } else {
            sl_accumulate(ctx, lam0, s->gradm, nt, dt, b, nullptr, lam2, fn.gmt);
        }
    } else if (fused) {
        int lc = 1;  // lam_j alternates between lam(1) and lam(0)
        for (int j = nt - 1; j >= 0; --j) {
            const double w = (j == 0) ? 0.5 * dt : dt;
            // the last step also adds u = beta_v A vt when it is given (out = b + u)
            const bool fin = (j == 0) && reg_given && identity_K;
            step_with_halo(ctx, lam(lc), [&] {
                sl_adjoint_step(ctx, lam(lc), s->xf, s->factor, lam(lc ^ 1), s->gradm + 3LL * j * N, w,
                                b, fin ? reg_given : nullptr, fin ? out3 : b);
            });
            lc ^= 1;
            out_done = fin;
        }
    } else {
        for (int j = nt - 1; j >= 0; --j)
            step_with_halo(ctx, lam(j + 1), [&] {
                sl_adjoint_step(ctx, lam(j + 1), s->xf, s->factor, lam(j), nullptr, 0.0, nullptr);
            });
        if (reg_given && identity_K) {
            sl_accumulate(ctx, lam0, s->gradm, nt, dt, out3, reg_given);  // out = b + u, one pass
            out_done = true;
        } else {
            sl_accumulate(ctx, lam0, s->gradm, nt, dt, b);
        }
    }
    o->counters.pde_solves += 1;
    if (!out_done) {
        if (!identity_K)
            op_projection(ctx, b, b, o->model.projection, o->model.beta_v, o->model.norm.beta_w);
        if (add_reg) {
            join_side(ctx);
            op_reg_finish(ctx, out3, b);  // out = b + beta_v A vt (objective.cpp:118-120)
        } else if (reg_given) {
            lin_comb(ctx, out3, 1.0, b, 1.0, reg_given, 3 * N);
        } else {
            VR_CUDA(cudaMemcpyAsync(out3, b, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice,
                                    ctx->stream));
        }
    }
    o->counters.hessian_matvecs += 1;
    if (check) defer_flags(ctx, "hessian_matvec");  // raised by the next reduction or drain
}

void objective_matvec_host_async(vr_objective* o, const vr_state* s, const double* vt3_host,
                                 double* out3_host) {
    vr_ctx* ctx = o->ctx;
    if (ctx->dist) throw_argument("hessian_matvec_host_async: one GPU only");
    if (!s->has_adjoint_ctx)
        throw_logic("hessian_matvec: evaluation context is missing the adjoint sweep data "
                    "(compute the gradient first)");
    auto& P = o->pipe;
    const long long n3 = 3 * ctx->g.N;
    const size_t bytes = sizeof(double) * n3;
    if (!P.h2d) {
        VR_CUDA(cudaStreamCreateWithFlags(&P.h2d, cudaStreamNonBlocking));
        VR_CUDA(cudaStreamCreateWithFlags(&P.d2h, cudaStreamNonBlocking));
        for (int q = 0; q < 2; ++q) {
            P.vt[q] = dev_alloc(ctx, n3);
            P.out[q] = dev_alloc(ctx, n3);
            VR_CUDA(cudaEventCreateWithFlags(&P.up[q], cudaEventDisableTiming));
            VR_CUDA(cudaEventCreateWithFlags(&P.done[q], cudaEventDisableTiming));
            VR_CUDA(cudaEventCreateWithFlags(&P.down[q], cudaEventDisableTiming));
        }
        VR_CUDA(cudaStreamSynchronize(ctx->stream));  // slots allocated on the compute stream
    }
    if (P.issued == 0) {
        drain_flags(ctx);
        VR_CUDA(cudaMemsetAsync(ctx->flag_dev, 0, 2 * sizeof(int), ctx->stream));
    }
    const int q = static_cast<int>(P.issued & 1);
    // upload once the compute two calls back has finished reading this slot
    VR_CUDA(cudaStreamWaitEvent(P.h2d, P.done[q], 0));
    VR_CUDA(cudaMemcpyAsync(P.vt[q], vt3_host, bytes, cudaMemcpyHostToDevice, P.h2d));
    VR_CUDA(cudaEventRecord(P.up[q], P.h2d));
    // compute once uploaded and once the previous download of this slot's result is done
    VR_CUDA(cudaStreamWaitEvent(ctx->stream, P.up[q], 0));
    VR_CUDA(cudaStreamWaitEvent(ctx->stream, P.down[q], 0));
    objective_matvec(o, s, P.vt[q], P.out[q], true, nullptr, false);
    VR_CUDA(cudaEventRecord(P.done[q], ctx->stream));
    VR_CUDA(cudaStreamWaitEvent(P.d2h, P.done[q], 0));
    VR_CUDA(cudaMemcpyAsync(out3_host, P.out[q], bytes, cudaMemcpyDeviceToHost, P.d2h));
    VR_CUDA(cudaEventRecord(P.down[q], P.d2h));
    P.issued += 1;
}

void objective_pipe_wait(vr_objective* o) {
    vr_ctx* ctx = o->ctx;
    auto& P = o->pipe;
    if (P.h2d) {
        VR_CUDA(cudaStreamSynchronize(P.h2d));
        VR_CUDA(cudaStreamSynchronize(P.d2h));
    }
    const bool any = P.issued > 0;
    P.issued = 0;
    if (any) check_flags(ctx, "hessian_matvec_host_async");
}

void objective_apply_reg(vr_objective* o, const double* u3, int mode, double* out3) {
    if (mode < VR_REGOP_APPLY || mode > VR_REGOP_INVERSE_SQRT)
        throw_argument("apply_reg: unknown mode");
    op_reg(o->ctx, u3, out3, o->model.norm, mode, o->model.beta_v);
}
void objective_apply_K(vr_objective* o, const double* u3, double* out3) {
    op_projection(o->ctx, u3, out3, o->model.projection, o->model.beta_v, o->model.norm.beta_w);
}

// ---------------------------------------------------------------------------
// PCG (solver.cpp:51-100)
// ---------------------------------------------------------------------------
vr_pcg_stats pcg_solve(vr_ctx* ctx, const DevOp& apply, const double* rhs, double rel_tol,
                       int max_iter, const DevOp& precond, double* x) {
    Range nvtx("pcg_solve");
    const long long n3 = 3 * ctx->g.N;
    vr_pcg_stats st{};
    st.rel_residual = 1.0;
    VR_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n3, ctx->stream));
    const double r0 = norm_l2_vec(ctx, rhs);
    if (r0 == 0.0) {
        st.converged = 1;
        st.rel_residual = 0.0;
        return st;
    }
    const double target = rel_tol * r0;
    double* r = dev_alloc(ctx, n3);
    double* z = dev_alloc(ctx, n3);
    double* s = dev_alloc(ctx, n3);
    double* Hs = dev_alloc(ctx, n3);
    auto cleanup = [&] {
        for (double* p : {r, z, s, Hs}) dev_free(ctx, p);
    };
    try {
        VR_CUDA(cudaMemcpyAsync(r, rhs, sizeof(double) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
        precond(r, z);
        VR_CUDA(cudaMemcpyAsync(s, z, sizeof(double) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
        double rz = dot_l2_vec(ctx, r, z);
        for (int it = 0; it < max_iter; ++it) {
            apply(s, Hs);
            const double sHs = dot_l2_vec(ctx, s, Hs);
            if (sHs <= 0.0) {
                st.negative_curvature = 1;
                if (it == 0)
                    VR_CUDA(cudaMemcpyAsync(x, z, sizeof(double) * n3, cudaMemcpyDeviceToDevice,
                                            ctx->stream));
                st.iterations = it + 1;
                st.rel_residual = norm_l2_vec(ctx, r) / r0;
                cleanup();
                return st;
            }
            const double kappa = rz / sHs;
            add_scaled(ctx, x, kappa, s, n3);
            add_scaled(ctx, r, -kappa, Hs, n3);
            st.iterations = it + 1;
            const double rn = norm_l2_vec(ctx, r);
            st.rel_residual = rn / r0;
            if (rn < target) {
                st.converged = 1;
                cleanup();
                return st;
            }
            precond(r, z);
            const double rz_new = dot_l2_vec(ctx, r, z);
            const double mu = rz_new / rz;
            rz = rz_new;
            lin_comb(ctx, s, 1.0, z, mu, s, n3);
        }
        st.hit_max_iterations = 1;
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
    return st;
}

// ---------------------------------------------------------------------------
// PCG on the GN Hessian with the spectral preconditioner. Same iteration as
// pcg_solve (solver.cpp:51-100, identical stop / curvature / update formulas),
// with two exact rewrites that remove work from every iteration:
//  * u = beta_v A s is carried through the recurrence instead of recomputed by
//    FFT in each matvec: z = (beta_v A)^-1 r gives beta_v A z = r - P0 r (P0 =
//    per-component mean when A has a zero singular value, spectral.cpp:176-177,
//    else 0), so s = z + mu s implies u = (r - P0 r) + mu u, and H s = H_data s + u.
//  * x += kappa s, r -= kappa Hs and |r|^2 (plus sum r for P0) are one pass.
// The rewrites change rounding only (~1e-15 relative per iteration).
vr_pcg_stats pcg_solve_gn(vr_objective* o, const vr_state* s, const double* rhs, double rel_tol,
                          int max_iter, double* x) {
    Range nvtx("pcg_solve_gn");
    vr_ctx* ctx = o->ctx;
    const long long N = ctx->g.N;
    const long long n3 = 3 * N;
    const bool zero_mode = reg_symbol(o->model.norm, 0.0) == 0.0;
    vr_pcg_stats st{};
    st.rel_residual = 1.0;
    VR_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n3, ctx->stream));
    const double r0 = norm_l2_vec(ctx, rhs);
    if (r0 == 0.0) {
        st.converged = 1;
        st.rel_residual = 0.0;
        return st;
    }
    const double target = rel_tol * r0;
    double* r = dev_alloc(ctx, n3);
    double* z = dev_alloc(ctx, n3);
    double* sd = dev_alloc(ctx, n3);
    double* Hs = dev_alloc(ctx, n3);
    double* u = dev_alloc(ctx, n3);
    auto cleanup = [&] {
        for (double* p : {r, z, sd, Hs, u}) dev_free(ctx, p);
    };
    auto means_of = [&](const double* sums, double* m) {
        for (int c = 0; c < 3; ++c)
            m[c] = zero_mode ? sums[c] / static_cast<double>(ctx->g.Ng) : 0.0;  // global mean
    };
    try {
        VR_CUDA(cudaMemcpyAsync(r, rhs, sizeof(double) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
        objective_apply_reg(o, r, VR_REGOP_INVERSE, z);  // SpectralPreconditioner::apply
        VR_CUDA(cudaMemcpyAsync(sd, z, sizeof(double) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
        double sums[3], mean[3];
        sum_components(ctx, r, N, 3, sums);
        means_of(sums, mean);
        pcg_direction(ctx, nullptr, u, nullptr, r, 0.0, mean);  // u = beta_v A z
        double rz = dot_l2_vec(ctx, r, z);
        for (int it = 0; it < max_iter; ++it) {
            objective_matvec(o, s, sd, Hs, false, u);  // flags checked with the s.Hs reduction
            const double sHs = dot_l2_vec(ctx, sd, Hs);
            if (sHs <= 0.0) {
                st.negative_curvature = 1;
                if (it == 0)
                    VR_CUDA(cudaMemcpyAsync(x, z, sizeof(double) * n3, cudaMemcpyDeviceToDevice,
                                            ctx->stream));
                st.iterations = it + 1;
                st.rel_residual = norm_l2_vec(ctx, r) / r0;
                cleanup();
                return st;
            }
            const double kappa = rz / sHs;
            double rr[3];
            pcg_update(ctx, x, r, sd, Hs, kappa, rr, sums);
            st.iterations = it + 1;
            const double rn = std::sqrt(rr[0] + rr[1] + rr[2]);
            st.rel_residual = rn / r0;
            if (rn < target) {
                st.converged = 1;
                cleanup();
                return st;
            }
            objective_apply_reg(o, r, VR_REGOP_INVERSE, z);
            const double rz_new = dot_l2_vec(ctx, r, z);
            const double mu = rz_new / rz;
            rz = rz_new;
            means_of(sums, mean);
            pcg_direction(ctx, sd, u, z, r, mu, mean);
        }
        st.hit_max_iterations = 1;
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
    return st;
}

// ---------------------------------------------------------------------------
// Armijo (solver.cpp:104-129) and Gauss-Newton (solver.cpp:154-269)
// ---------------------------------------------------------------------------
namespace {

struct LineSearch {
    bool success = false;
    double alpha = 0.0;
    int trials = 0;
    vr_state* state = nullptr;
};

LineSearch armijo_search(vr_objective* o, const vr_state* cur, const double* dir,
                         const vr_solver_params& p) {
    Range nvtx("armijo_search");
    vr_ctx* ctx = o->ctx;
    const long long n3 = 3 * ctx->g.N;
    if (!cur->has_gradient) throw_logic("armijo_search: current state has no gradient");
    const double slope = inner_product_vec(ctx, cur->grad, dir);
    if (slope >= 0.0)
        throw_argument("armijo_search: not a descent direction (slope = " + std::to_string(slope) +
                       ")");
    LineSearch res;
    double alpha = 1.0;
    double* trial_v = dev_alloc(ctx, n3);
    try {
        for (int t = 0; t < p.armijo_max_trials; ++t) {
            lin_comb(ctx, trial_v, 1.0, cur->v, alpha, dir, n3);
            const auto t0 = std::chrono::steady_clock::now();
            vr_state* trial = objective_evaluate(o, trial_v);
            if (timing_enabled())
                slow_op("armijo trial evaluate",
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
            res.trials = t + 1;
            if (trial->objective <= cur->objective + p.armijo_c1 * alpha * slope) {
                res.success = true;
                res.alpha = alpha;
                res.state = trial;
                break;
            }
            delete trial;
            alpha *= p.armijo_backtrack;
        }
    } catch (...) {
        dev_free(ctx, trial_v);
        throw;
    }
    dev_free(ctx, trial_v);
    return res;
}

vr_iteration_record make_record(int k, const vr_state* s, double gn, double g0,
                                const vr_counters& fine, const vr_counters& coarse,
                                double elapsed) {
    vr_iteration_record r{};
    r.k = k;
    r.objective = s->objective;
    r.mismatch_rel = s->mismatch_rel;
    r.grad_norm = gn;
    r.grad_rel = g0 > 0 ? gn / g0 : 0.0;
    r.fine_matvecs = fine.hessian_matvecs;
    r.coarse_matvecs = coarse.hessian_matvecs;
    r.pde_solves = fine.pde_solves;
    r.wall_time_s = elapsed;
    return r;
}

}  // namespace

GnResult gauss_newton_solve(vr_ctx* ctx, const double* mR, const double* mT, const double* v0,
                            const vr_model& model, const vr_solver_params& params, int precond,
                            double* v_out, const vr_twolevel_options* tl_opts) {
    Range nvtx("gauss_newton_solve");
    validate_params(params);
    if (precond != VR_PRECOND_NONE && precond != VR_PRECOND_SPECTRAL &&
        precond != VR_PRECOND_TWO_LEVEL)
        throw_argument("gauss_newton_solve: unknown preconditioner");
    std::unique_ptr<TwoLevel> tl;
    if (precond == VR_PRECOND_TWO_LEVEL) {
        vr_twolevel_options d;
        vr_twolevel_options_default(&d);
        tl.reset(new TwoLevel(tl_opts ? *tl_opts : d));
    }
    auto coarse = [&] { return tl ? tl->counters() : vr_counters{}; };
    const auto t0 = std::chrono::steady_clock::now();
    // VR_TIMING=1: host wall time per phase (stream drained at each boundary) on stderr
    static const bool timing = std::getenv("VR_TIMING") != nullptr;
    double ph[5] = {0, 0, 0, 0, 0};  // setup, pcg, line search, gradient, other
    auto tp = std::chrono::steady_clock::now();
    auto mark = [&](int phase) {
        if (!timing) return;
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        const auto now = std::chrono::steady_clock::now();
        ph[phase] += std::chrono::duration<double>(now - tp).count();
        tp = now;
    };
    auto elapsed = [&] {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    const long long n3 = 3 * ctx->g.N;
    GnResult res;
    vr_solve_report& rep = res.report;
    rep.stop = VR_STOP_MAX_ITERATIONS;
    vr_objective* obj = objective_create(ctx, mR, mT, model);
    vr_state* state = nullptr;
    double* dir = nullptr;
    double* rhs = nullptr;
    auto cleanup = [&] {
        delete state;
        dev_free(ctx, dir);
        dev_free(ctx, rhs);
        delete obj;
    };
    try {
        state = objective_evaluate(obj, v0);
        objective_gradient(obj, state);
        const double g0 = norm_l2_vec(ctx, state->grad);
        mark(0);
        rep.grad0 = g0;
        res.records.push_back(make_record(0, state, g0, g0, obj->counters, coarse(), elapsed()));
        if (g0 == 0.0) {
            rep.stop = VR_STOP_ZERO_GRADIENT;
            rep.success = 1;
        } else {
            dir = dev_alloc(ctx, n3);
            rhs = dev_alloc(ctx, n3);
            double gk = g0;
            int k = 0;
            for (;;) {
                const bool rel_ok = params.squared_norm_stop ? (gk * gk <= params.eps_opt * g0 * g0)
                                                             : (gk <= params.eps_opt * g0);
                if (rel_ok) {
                    rep.stop = VR_STOP_CONVERGED_REL;
                    rep.success = 1;
                    break;
                }
                if (gk <= params.abs_grad_tol) {
                    rep.stop = VR_STOP_CONVERGED_ABS;
                    rep.success = 1;
                    break;
                }
                if (k >= params.max_newton) {
                    rep.stop = VR_STOP_MAX_ITERATIONS;
                    break;
                }
                mark(4);
                const double eps_H = std::min(0.5, std::sqrt(gk / g0));  // compute_forcing
                const vr_state* cs = state;
                DevOp op = [&](const double* u, double* out) {
                    objective_matvec(obj, cs, u, out, true);
                };
                DevOp pc = [&](const double* r, double* z) {
                    if (precond == VR_PRECOND_SPECTRAL)
                        objective_apply_reg(obj, r, VR_REGOP_INVERSE, z);
                    else
                        VR_CUDA(cudaMemcpyAsync(z, r, sizeof(double) * n3,
                                                cudaMemcpyDeviceToDevice, ctx->stream));
                };
                vr_pcg_stats pcg;
                if (tl) {
                    // split system (solver.cpp:208-221): (I + R H_data R) w = -R g, v~ = R w
                    tl->rebuild(obj, state, eps_H);
                    DevOp sop = [&](const double* w, double* out) { split_matvec(obj, cs, w, out); };
                    DevOp spc = [&](const double* r, double* z) { tl->apply(ctx, r, z); };
                    objective_apply_reg(obj, state->grad, VR_REGOP_INVERSE_SQRT, rhs);
                    scale(ctx, rhs, n3, -1.0);
                    pcg = pcg_solve(ctx, sop, rhs, eps_H, params.max_krylov, spc, dir);
                    objective_apply_reg(obj, dir, VR_REGOP_INVERSE_SQRT, dir);
                } else {
                    // rhs = -g (scale(rhs, -1.0))
                    lin_comb(ctx, rhs, -1.0, state->grad, 0.0, state->grad, n3);
                    pcg = precond == VR_PRECOND_SPECTRAL
                              ? pcg_solve_gn(obj, state, rhs, eps_H, params.max_krylov, dir)
                              : pcg_solve(ctx, op, rhs, eps_H, params.max_krylov, pc, dir);
                }

                mark(1);
                const double slope = inner_product_vec(ctx, state->grad, dir);
                if (slope >= 0.0) {
                    rep.stop = VR_STOP_LINE_SEARCH_FAILURE;
                    break;
                }
                LineSearch ls = armijo_search(obj, state, dir, params);
                if (!ls.success) {
                    rep.stop = VR_STOP_LINE_SEARCH_FAILURE;
                    break;
                }
                mark(2);
                delete state;
                state = ls.state;
                objective_gradient(obj, state);
                gk = norm_l2_vec(ctx, state->grad);
                mark(3);
                ++k;
                vr_iteration_record row =
                    make_record(k, state, gk, g0, obj->counters, coarse(), elapsed());
                row.step_length = ls.alpha;
                row.forcing = eps_H;
                row.inner_iterations = pcg.iterations;
                res.records.push_back(row);
            }
            rep.outer_iterations = k;
        }
        rep.final_objective = state->objective;
        rep.final_mismatch_rel = state->mismatch_rel;
        const double gfin = norm_l2_vec(ctx, state->grad);
        rep.final_grad_rel = g0 > 0 ? gfin / g0 : 0.0;
        rep.fine = obj->counters;
        rep.coarse = coarse();
        rep.n_records = static_cast<int>(res.records.size());
        VR_CUDA(cudaMemcpyAsync(v_out, state->v, sizeof(double) * n3, cudaMemcpyDeviceToDevice,
                                ctx->stream));
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        rep.wall_time_s = elapsed();
        if (timing)
            std::fprintf(stderr, "VR_TIMING gn_solve %.1f ms: setup %.1f pcg %.1f linesearch %.1f gradient %.1f other %.1f (%d iterations)\n",
                         1e3 * rep.wall_time_s, 1e3 * ph[0], 1e3 * ph[1], 1e3 * ph[2], 1e3 * ph[3], 1e3 * ph[4],
                         rep.outer_iterations);
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
    return res;
}

}  // namespace vr
