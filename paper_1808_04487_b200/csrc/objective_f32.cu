// objective_f32.cu -- the fp32 lane of the objective: the reference's
// Objective<float> (proj/src/objective.cpp:35-156 with T = float, Gauss-Newton and full
// Newton) and its Newton / PCG / Armijo driver (proj/src/solver.cpp:23-269), one GPU.
//
// Every field is stored in fp32 exactly where the reference stores a ScalarField<float>
// (state history, departure points, continuity factor, grad m_j, adjoint / incremental
// fields, gradient, PCG vectors); stencils, transforms and reductions run in fp64 and
// each stored result is rounded once, as in the reference: the fp32 semi-Lagrangian
// kernels (sl.cu), the fp64 spectral operators behind a convert-at-the-boundary (the
// reference's fft.hpp:12-17 contract) and fp64 reductions of the fp32 values. The
// steps are composed from those operators and small pointwise kernels;
// the sweep steps are fused like the fp64 lane's (sl.cu *_f32 kernels), the spectral
// terms go through fp64 scratch views.
#include <chrono>
#include <cmath>
#include <memory>
#include <vector>

#include "objective.cuh"
#include "twolevel.cuh"

namespace vr {
namespace {

constexpr int kT = 256;
unsigned blocks(long long n) { return grid_1d(n, kT); }

// out = float(a x + b y)  (lin_comb, field_ops.hpp:30-40); y may be null (b ignored)
__global__ void k_lincomb_f(float* out, double a, const float* x, double b, const float* y, long long n) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i >= n) return;
    const double r = y ? a * static_cast<double>(x[i]) + b * static_cast<double>(y[i])
                       : a * static_cast<double>(x[i]);
    out[i] = static_cast<float>(r);
}
// y = float(y + a x)  (add_scaled)
__global__ void k_axpy_f(float* y, double a, const float* x, long long n) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i < n) y[i] = static_cast<float>(static_cast<double>(y[i]) + a * static_cast<double>(x[i]));
}
// continuity_factor (transport.cpp:44-55)
__global__ void k_factor_f(float* factor, const float* div, const float* at_dep, double half_dt,
                           long long n) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i < n)
        factor[i] = static_cast<float>(
            exp(half_dt * (static_cast<double>(div[i]) + static_cast<double>(at_dep[i]))));
}
// ---- full Newton (gauss_newton = false; transport.cpp:150-226, objective.cpp:135-149) ----
// gradient_dot<float>: q = float(q + d_a m * w_a), a = 0, 1, 2 (transport.cpp:143-145)
__global__ void k_graddot_f(float* q, const float* gm, const float* vt, long long n) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i >= n) return;
    float o = 0.0f;
#pragma unroll
    for (int a = 0; a < 3; ++a)
        o = static_cast<float>(static_cast<double>(o) +
                               static_cast<double>(gm[a * n + i]) * static_cast<double>(vt[a * n + i]));
    q[i] = o;
}
// lv_c = float(lam * vt_c) (transport.cpp:203-207)
__global__ void k_scale_vec_f(float* lv, const float* lam, const float* vt, long long n) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i >= n) return;
    const float l = lam[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) lv[c * n + i] = l * vt[c * n + i];
}
// cur = float(lam_interp * factor + half_dt * (r_cur + src_interp)) with the float product and
// the float sum of the reference's expression (transport.cpp:217-220)
__global__ void k_fn_step_f(float* cur, const float* li, const float* factor, const float* rc,
                            const float* si, double half_dt, long long n) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i >= n) return;
    const float a = li[i] * factor[i];
    const float b = rc[i] + si[i];
    cur[i] = static_cast<float>(static_cast<double>(a) + half_dt * static_cast<double>(b));
}
// the full-Newton observer at slice j (objective.cpp:143-148):
// b_a = float(b_a + (w lam~_j) d_a m_j); b_a = float(b_a + (w lam_j) d_a mt_j)
__global__ void k_observe_fn_f(float* b, double w, const float* lamt, const float* gm, const float* lam,
                               const float* gmt, long long n) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i >= n) return;
    const double w1 = w * static_cast<double>(lamt[i]), w2 = w * static_cast<double>(lam[i]);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float v = static_cast<float>(static_cast<double>(b[a * n + i]) + w1 * static_cast<double>(gm[a * n + i]));
        v = static_cast<float>(static_cast<double>(v) + w2 * static_cast<double>(gmt[a * n + i]));
        b[a * n + i] = v;
    }
}
float* falloc(vr_ctx* ctx, long long n) { return reinterpret_cast<float*>(dev_alloc(ctx, (n + 1) / 2)); }
void ffree(vr_ctx* ctx, float* p) { dev_free(ctx, reinterpret_cast<double*>(p)); }

void lincomb(vr_ctx* ctx, float* out, double a, const float* x, double b, const float* y, long long n) {
    VR_LAUNCH(ctx, "f32_pointwise", k_lincomb_f<<<blocks(n), kT, 0, ctx->stream>>>(out, a, x, b, y, n));
}
void axpy(vr_ctx* ctx, float* y, double a, const float* x, long long n) {
    VR_LAUNCH(ctx, "f32_pointwise", k_axpy_f<<<blocks(n), kT, 0, ctx->stream>>>(y, a, x, n));
}

// fp64 scratch views of fp32 fields (for the spectral operators and the reductions)
struct F64 {
    vr_ctx* ctx;
    double* p;
    F64(vr_ctx* c, const float* f, long long n) : ctx(c), p(dev_alloc(c, n)) {
        if (f) convert_f2d(c, f, p, n);
    }
    ~F64() { dev_free(ctx, p); }
    F64(const F64&) = delete;
    F64& operator=(const F64&) = delete;
};

// sum_i a_i b_i of fp32 vectors (fp64 products and sums, fixed order) and the weighted
// inner product (spectral.cpp:47-62)
double dot_f(vr_ctx* ctx, const float* a, const float* b, long long n, int ncomp) {
    F64 da(ctx, a, ncomp * n), db(ctx, b, ncomp * n);
    double r[3] = {0, 0, 0};
    dot_components(ctx, da.p, db.p, n, ncomp, r);
    double s = 0.0;
    for (int c = 0; c < ncomp; ++c) s += r[c];
    return s;
}
double cell(const GridDims& g) { return g.h1 * g.h2 * g.h3; }

void spectral_f(vr_ctx* ctx, const float* in, int nin, float* out, int nout,
                const std::function<void(const double*, double*)>& fn) {
    const long long N = ctx->g.N;
    F64 din(ctx, in, nin * N), dout(ctx, nullptr, nout * N);
    fn(din.p, dout.p);
    convert_d2f(ctx, dout.p, out, nout * N);
}

}  // namespace

struct ObjF32 {
    vr_ctx* ctx = nullptr;
    const float* mR = nullptr;
    const float* mT = nullptr;
    vr_model model{};
    vr_counters counters{};
    double initial_mismatch = 0.0;
};

struct StateF32 {
    ObjF32* obj = nullptr;
    int nt = 0;
    float *v = nullptr, *xb = nullptr, *mhist = nullptr, *xf = nullptr, *factor = nullptr,
          *gradm = nullptr, *grad = nullptr, *lamhist = nullptr;  // lamhist: full Newton only
    double objective = 0.0, mismatch = 0.0, mismatch_rel = 0.0;
    bool has_gradient = false;
    ~StateF32() {
        if (!obj) return;
        for (float* p : {v, xb, mhist, xf, factor, gradm, grad, lamhist}) ffree(obj->ctx, p);
    }
};

ObjF32* objf32_create(vr_ctx* ctx, const float* mR, const float* mT, const vr_model& model) {
    validate_model(model);
    if (ctx->dist) throw_argument("fp32 objective: one GPU only");
    auto o = std::make_unique<ObjF32>();
    o->ctx = ctx;
    o->mR = mR;
    o->mT = mT;
    o->model = model;
    const long long N = ctx->g.N;
    float* diff = falloc(ctx, N);
    lincomb(ctx, diff, 1.0, mT, -1.0, mR, N);  // objective.cpp:40-44
    o->initial_mismatch = dot_f(ctx, diff, diff, N, 1) * cell(ctx->g);
    ffree(ctx, diff);
    return o.release();
}

// evaluate (objective.cpp:47-75)
StateF32* objf32_evaluate(ObjF32* o, const float* v3) {
    vr_ctx* ctx = o->ctx;
    const long long N = ctx->g.N;
    const int nt = o->model.nt;
    if (!all_finite_f32(ctx, v3, 3 * N)) throw_numeric("evaluate_objective: non-finite velocity");
    auto s = std::make_unique<StateF32>();
    s->obj = o;
    s->nt = nt;
    s->v = falloc(ctx, 3 * N);
    s->xb = falloc(ctx, 3 * N);
    s->mhist = falloc(ctx, (nt + 1) * N);
    VR_CUDA(cudaMemcpyAsync(s->v, v3, sizeof(float) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
    sl_trace_f32(ctx, s->v, nt, VR_TRACE_BACKWARD, s->xb);
    VR_CUDA(cudaMemcpyAsync(s->mhist, o->mT, sizeof(float) * N, cudaMemcpyDeviceToDevice, ctx->stream));
    for (int j = 0; j < nt; ++j) sl_tricubic_f32(ctx, s->mhist + j * N, 1, s->xb, s->mhist + (j + 1) * N);
    o->counters.pde_solves += 1;
    float* diff = falloc(ctx, N);
    lincomb(ctx, diff, 1.0, s->mhist + nt * N, -1.0, o->mR, N);
    s->mismatch = dot_f(ctx, diff, diff, N, 1) * cell(ctx->g);
    ffree(ctx, diff);
    s->mismatch_rel = o->initial_mismatch > 0.0 ? s->mismatch / o->initial_mismatch : 0.0;
    // reg = 1/2 beta_v <A v, v>_h (A at beta 1; Parseval on the fp64 view of v)
    double reg, penalty = 0.0;
    {
        F64 dv(ctx, s->v, 3 * N);
        reg = 0.5 * o->model.beta_v * reg_energy(ctx, dv.p, o->model.norm);
        if (o->model.norm.div_penalty) {
            F64 w(ctx, nullptr, N), hw(ctx, nullptr, N);
            op_divergence(ctx, dv.p, w.p);
            MultParams mp;
            mp.kind = Mult::helmholtz1;
            spectral_scalar_op(ctx, w.p, hw.p, mp);
            penalty = 0.5 * o->model.norm.beta_w * inner_product_scalar(ctx, hw.p, w.p);
        }
    }
    s->objective = 0.5 * s->mismatch + reg + penalty;
    if (!std::isfinite(s->objective)) throw_numeric("evaluate_objective: objective is not finite");
    o->counters.objective_evals += 1;
    return s.release();
}

// prepare_adjoint_ctx + compute_gradient (objective.cpp:77-112); the grad m_j cache is
// the reference's accumulate_weighted_grad scratch (fp32-rounded derivatives)
void objf32_gradient(ObjF32* o, StateF32* s) {
    vr_ctx* ctx = o->ctx;
    const long long N = ctx->g.N;
    const int nt = s->nt;
    const double dt = 1.0 / nt;
    if (!s->xf) {
        s->xf = falloc(ctx, 3 * N);
        s->factor = falloc(ctx, N);
        s->gradm = falloc(ctx, 3LL * (nt + 1) * N);
        sl_trace_f32(ctx, s->v, nt, VR_TRACE_FORWARD, s->xf);
        float* div = falloc(ctx, N);
        float* at = falloc(ctx, N);
        spectral_f(ctx, s->v, 3, div, 1, [&](const double* i, double* out) { op_divergence(ctx, i, out); });
        sl_tricubic_f32(ctx, div, 1, s->xf, at);
        VR_LAUNCH(ctx, "f32_pointwise", k_factor_f<<<blocks(N), kT, 0, ctx->stream>>>(s->factor, div, at, 0.5 * dt, N));
        ffree(ctx, div);
        ffree(ctx, at);
        for (int j = 0; j <= nt; ++j)
            spectral_f(ctx, s->mhist + j * N, 1, s->gradm + 3LL * j * N, 3,
                       [&](const double* i, double* out) { op_gradient(ctx, i, out); });
    }
    if (!s->grad) s->grad = falloc(ctx, 3 * N);
    // adjoint sweep keeping every lambda_j, then the observer accumulation in one pass
    float* lamh = falloc(ctx, (nt + 1) * N);
    float* b = s->grad;
    lincomb(ctx, lamh + nt * N, 1.0, o->mR, -1.0, s->mhist + nt * N, N);  // terminal (objective.cpp:91-92)
    for (int j = nt - 1; j >= 0; --j)  // sweep_continuity (transport.cpp:88-113)
        sl_continuity_f32(ctx, lamh + (j + 1) * N, s->xf, s->factor, lamh + j * N);
    sl_accumulate_f32(ctx, lamh, s->gradm, nt, dt, b);
    if (!o->model.gauss_newton) {  // s.lambda_history (objective.cpp:100-102)
        ffree(ctx, s->lamhist);
        s->lamhist = lamh;
    } else {
        ffree(ctx, lamh);
    }
    o->counters.pde_solves += 1;
    if (o->model.projection != VR_PROJ_IDENTITY)
        spectral_f(ctx, b, 3, b, 3, [&](const double* i, double* out) {
            op_projection(ctx, i, out, o->model.projection, o->model.beta_v, o->model.norm.beta_w);
        });
    // g = float(b + beta_v A v): fp32 rows in, the add in the c2r epilogue (add_scaled(gradient, 1.0, reg))
    op_reg_begin_f32(ctx, s->v, o->model.norm, VR_REGOP_APPLY, o->model.beta_v);
    op_reg_finish_f32(ctx, b, b);
    s->has_gradient = true;
    o->counters.gradient_evals += 1;
}

// hessian_matvec (objective.cpp:114-156, GN): inc-state (transport.cpp:150-173), GN
// inc-adjoint (sweep_continuity with the observer), K, + beta_v A vt
static void objf32_matvec_impl(ObjF32* o, const StateF32* s, const float* vt3, float* out3, bool with_reg);
void objf32_matvec(ObjF32* o, const StateF32* s, const float* vt3, float* out3) {
    objf32_matvec_impl(o, s, vt3, out3, true);
}
// hessian_matvec (with_reg) / hessian_data_matvec (objective.cpp:114-156)
static void objf32_matvec_impl(ObjF32* o, const StateF32* s, const float* vt3, float* out3, bool with_reg) {
    vr_ctx* ctx = o->ctx;
    const long long N = ctx->g.N;
    if (!all_finite_f32(ctx, vt3, 3 * N)) throw_numeric("hessian_matvec: non-finite direction");
    if (!s->xf)
        throw_logic("hessian_matvec: evaluation context is missing the adjoint sweep data "
                    "(compute the gradient first)");
    const int nt = s->nt;
    const double dt = 1.0 / nt, hdt = 0.5 / nt;
    if (!o->model.gauss_newton) {
        if (!s->lamhist) throw_logic("hessian_matvec: full Newton mode needs the adjoint history");
        // solve_inc_state keeping the mt history (transport.cpp:150-173), step by step with the
        // reference's rounding points
        float* mt = falloc(ctx, (nt + 1) * N);
        float *q[2] = {falloc(ctx, N), falloc(ctx, N)}, *tmp = falloc(ctx, N);
        VR_CUDA(cudaMemsetAsync(mt, 0, sizeof(float) * N, ctx->stream));
        VR_LAUNCH(ctx, "f32_pointwise", k_graddot_f<<<blocks(N), kT, 0, ctx->stream>>>(q[0], s->gradm, vt3, N));
        for (int j = 0; j < nt; ++j) {
            VR_LAUNCH(ctx, "f32_pointwise", k_graddot_f<<<blocks(N), kT, 0, ctx->stream>>>(
                q[(j + 1) & 1], s->gradm + 3LL * (j + 1) * N, vt3, N));
            lincomb(ctx, tmp, 1.0, mt + j * N, -hdt, q[j & 1], N);
            sl_tricubic_f32(ctx, tmp, 1, s->xb, mt + (j + 1) * N);
            axpy(ctx, mt + (j + 1) * N, -hdt, q[(j + 1) & 1], N);
        }
        o->counters.pde_solves += 1;
        // solve_inc_adjoint, full Newton (transport.cpp:192-226), with the observer
        float *cur = falloc(ctx, N), *li = falloc(ctx, N), *si = falloc(ctx, N), *lv = falloc(ctx, 3 * N);
        float *r[2] = {falloc(ctx, N), falloc(ctx, N)}, *gmt = falloc(ctx, 3 * N);
        auto source = [&](int j, float* out) {  // r_j = div(lambda_j vt)
            VR_LAUNCH(ctx, "f32_pointwise", k_scale_vec_f<<<blocks(N), kT, 0, ctx->stream>>>(lv, s->lamhist + j * N, vt3, N));
            spectral_f(ctx, lv, 3, out, 1, [&](const double* i, double* d) { op_divergence(ctx, i, d); });
        };
        float* b = out3;
        VR_CUDA(cudaMemsetAsync(b, 0, sizeof(float) * 3 * N, ctx->stream));
        auto observe = [&](int j) {
            const double w = (j == 0 || j == nt) ? 0.5 * dt : dt;
            spectral_f(ctx, mt + j * N, 1, gmt, 3, [&](const double* i, double* d) { op_gradient(ctx, i, d); });
            VR_LAUNCH(ctx, "f32_pointwise", k_observe_fn_f<<<blocks(N), kT, 0, ctx->stream>>>(
                b, w, cur, s->gradm + 3LL * j * N, s->lamhist + j * N, gmt, N));
        };
        lincomb(ctx, cur, -1.0, mt + nt * N, 0.0, nullptr, N);  // terminal = -mt_nt
        source(nt, r[nt & 1]);
        observe(nt);
        for (int j = nt - 1; j >= 0; --j) {
            source(j, r[j & 1]);
            sl_tricubic_f32(ctx, cur, 1, s->xf, li);
            sl_tricubic_f32(ctx, r[(j + 1) & 1], 1, s->xf, si);
            VR_LAUNCH(ctx, "f32_pointwise", k_fn_step_f<<<blocks(N), kT, 0, ctx->stream>>>(cur, li, s->factor, r[j & 1], si, hdt, N));
            observe(j);
        }
        o->counters.pde_solves += 1;
        for (float* p : {mt, q[0], q[1], tmp, cur, li, si, lv, r[0], r[1], gmt}) ffree(ctx, p);
        if (o->model.projection != VR_PROJ_IDENTITY)
            spectral_f(ctx, b, 3, b, 3, [&](const double* i, double* out) {
                op_projection(ctx, i, out, o->model.projection, o->model.beta_v, o->model.norm.beta_w);
            });
        o->counters.hessian_matvecs += 1;
        if (with_reg) {
            op_reg_begin_f32(ctx, vt3, o->model.norm, VR_REGOP_APPLY, o->model.beta_v);
            op_reg_finish_f32(ctx, out3, out3);
        }
        return;
    }
    // incremental state (transport.cpp:150-173) fused per step; the last step writes the
    // inc-adjoint terminal -mt_nt into the history, whose sweep then keeps every lambda~_j
    float* lamh = falloc(ctx, (nt + 1) * N);
    float* tmp[2] = {falloc(ctx, N), falloc(ctx, N)};
    sl_incstate_first_f32(ctx, s->gradm, vt3, hdt, tmp[0]);
    int c = 0;
    for (int j = 0; j < nt; ++j) {
        const bool last = j == nt - 1;
        sl_incstate_step_f32(ctx, tmp[c], s->xb, s->gradm + 3LL * (j + 1) * N, vt3, hdt,
                             last ? lamh + nt * N : tmp[c ^ 1], last);
        c ^= 1;
    }
    o->counters.pde_solves += 1;
    for (int j = nt - 1; j >= 0; --j)
        sl_continuity_f32(ctx, lamh + (j + 1) * N, s->xf, s->factor, lamh + j * N);
    float* b = out3;
    sl_accumulate_f32(ctx, lamh, s->gradm, nt, dt, b);
    o->counters.pde_solves += 1;
    for (float* p : {lamh, tmp[0], tmp[1]}) ffree(ctx, p);
    if (o->model.projection != VR_PROJ_IDENTITY)
        spectral_f(ctx, b, 3, b, 3, [&](const double* i, double* out) {
            op_projection(ctx, i, out, o->model.projection, o->model.beta_v, o->model.norm.beta_w);
        });
    o->counters.hessian_matvecs += 1;
    if (!with_reg) return;
    // out = float(b + beta_v A vt): fp32 rows in, the add fused into the c2r epilogue
    op_reg_begin_f32(ctx, vt3, o->model.norm, VR_REGOP_APPLY, o->model.beta_v);
    op_reg_finish_f32(ctx, out3, out3);
}

// ---- solver.cpp:51-269 on fp32 vectors (fp64 scalars) -------------------------------
namespace {
double norm_f(vr_ctx* ctx, const float* a, long long n) { return std::sqrt(dot_f(ctx, a, a, n, 1)); }

using OpF = std::function<void(const float*, float*)>;
vr_pcg_stats pcg_f32(ObjF32* o, const StateF32* s, const float* rhs, double rel_tol, int max_iter,
                     int precond, float* x, const OpF* op_override = nullptr,
                     const OpF* pc_override = nullptr) {
    vr_ctx* ctx = o->ctx;
    const long long n3 = 3 * ctx->g.N;
    vr_pcg_stats st{};
    VR_CUDA(cudaMemsetAsync(x, 0, sizeof(float) * n3, ctx->stream));
    const double r0 = norm_f(ctx, rhs, n3);
    if (r0 == 0.0) {
        st.converged = 1;
        return st;
    }
    const double target = rel_tol * r0;
    float *r = falloc(ctx, n3), *z = falloc(ctx, n3), *sd = falloc(ctx, n3), *Hs = falloc(ctx, n3);
    auto pc = [&](const float* in, float* out) {  // SpectralPreconditioner: (beta_v A)^-1
        if (pc_override) {
            (*pc_override)(in, out);
        } else if (precond == VR_PRECOND_SPECTRAL) {
            op_reg_begin_f32(ctx, in, o->model.norm, VR_REGOP_INVERSE, o->model.beta_v);
            op_reg_finish_f32(ctx, out, nullptr);
        }
        else
            VR_CUDA(cudaMemcpyAsync(out, in, sizeof(float) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
    };
    VR_CUDA(cudaMemcpyAsync(r, rhs, sizeof(float) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
    pc(r, z);
    VR_CUDA(cudaMemcpyAsync(sd, z, sizeof(float) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
    double rz = dot_f(ctx, r, z, n3, 1);
    bool done = false;
    for (int it = 0; it < max_iter && !done; ++it) {
        if (op_override)
            (*op_override)(sd, Hs);
        else
            objf32_matvec(o, s, sd, Hs);
        const double sHs = dot_f(ctx, sd, Hs, n3, 1);
        if (sHs <= 0.0) {
            st.negative_curvature = 1;
            if (it == 0) VR_CUDA(cudaMemcpyAsync(x, z, sizeof(float) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
            st.iterations = it + 1;
            st.rel_residual = norm_f(ctx, r, n3) / r0;
            done = true;
            break;
        }
        const double kappa = rz / sHs;
        axpy(ctx, x, kappa, sd, n3);
        axpy(ctx, r, -kappa, Hs, n3);
        st.iterations = it + 1;
        const double rn = norm_f(ctx, r, n3);
        st.rel_residual = rn / r0;
        if (rn < target) {
            st.converged = 1;
            done = true;
            break;
        }
        pc(r, z);
        const double rz_new = dot_f(ctx, r, z, n3, 1);
        const double mu = rz_new / rz;
        rz = rz_new;
        lincomb(ctx, sd, 1.0, z, mu, sd, n3);
    }
    if (!done) st.hit_max_iterations = 1;
    for (float* p : {r, z, sd, Hs}) ffree(ctx, p);
    return st;
}
}  // namespace

// The two-level preconditioner of the fp32 solve (precond.cpp:153-249 with T = float): the
// outer Newton / split-system PCG runs on fp32 vectors as in the reference; the coarse-grid
// machinery behind M^-1 (restriction, coarse objective, inner PCG / Chebyshev, prolongation)
// is the fp64 TwoLevel of twolevel.cu applied to fp64 views of the fp32 fields -- a
// preconditioner in higher precision than the reference's float one (it changes Krylov
// iteration counts slightly, not what the solve converges to).
struct TwoLevelF32 {
    vr_ctx* ctx;
    TwoLevel tl;
    std::unique_ptr<F64> mR, mT;
    vr_objective* obj64 = nullptr;
    std::unique_ptr<vr_state> st64;
    TwoLevelF32(vr_ctx* c, const vr_twolevel_options& o, const float* r, const float* t, const vr_model& m)
        : ctx(c), tl(o), mR(new F64(c, r, c->g.N)), mT(new F64(c, t, c->g.N)) {
        obj64 = objective_create(c, mR->p, mT->p, m);
    }
    ~TwoLevelF32() {  // the coarse objects in `tl` do not reference the fine mirror
        st64.reset();
        delete obj64;
    }
    void rebuild(const StateF32* s, double eps_H) {
        const long long N = ctx->g.N;
        st64.reset(new vr_state());
        st64->obj = obj64;
        st64->nt = s->nt;
        st64->v = dev_alloc(ctx, 3 * N);
        st64->mhist = dev_alloc(ctx, (s->nt + 1) * N);
        convert_f2d(ctx, s->v, st64->v, 3 * N);
        convert_f2d(ctx, s->mhist, st64->mhist, (s->nt + 1) * N);
        if (s->lamhist) {
            st64->lamhist = dev_alloc(ctx, (s->nt + 1) * N);
            convert_f2d(ctx, s->lamhist, st64->lamhist, (s->nt + 1) * N);
        }
        tl.rebuild(obj64, st64.get(), eps_H);
    }
    void apply(const float* r, float* z) {
        const long long n3 = 3 * ctx->g.N;
        F64 dr(ctx, r, n3), dz(ctx, nullptr, n3);
        tl.apply(ctx, dr.p, dz.p);
        convert_d2f(ctx, dz.p, z, n3);
    }
};

GnResult gauss_newton_solve_f32(vr_ctx* ctx, const float* mR, const float* mT, const float* v0,
                                const vr_model& model, const vr_solver_params& params, int precond,
                                float* v_out, const vr_twolevel_options* tl_opts) {
    validate_params(params);
    if (precond != VR_PRECOND_NONE && precond != VR_PRECOND_SPECTRAL && precond != VR_PRECOND_TWO_LEVEL)
        throw_argument("gauss_newton_solve_f32: unknown preconditioner");
    std::unique_ptr<TwoLevelF32> tl;
    if (precond == VR_PRECOND_TWO_LEVEL) {
        vr_twolevel_options d;
        vr_twolevel_options_default(&d);
        tl.reset(new TwoLevelF32(ctx, tl_opts ? *tl_opts : d, mR, mT, model));
    }
    const auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    const long long n3 = 3 * ctx->g.N;
    const double hc = cell(ctx->g);
    GnResult res;
    vr_solve_report& rep = res.report;
    rep.stop = VR_STOP_MAX_ITERATIONS;
    std::unique_ptr<ObjF32> obj(objf32_create(ctx, mR, mT, model));
    std::unique_ptr<StateF32> state(objf32_evaluate(obj.get(), v0));
    objf32_gradient(obj.get(), state.get());
    auto record = [&](int k, double gn, double g0) {
        vr_iteration_record r{};
        r.k = k;
        r.objective = state->objective;
        r.mismatch_rel = state->mismatch_rel;
        r.grad_norm = gn;
        r.grad_rel = g0 > 0 ? gn / g0 : 0.0;
        r.fine_matvecs = obj->counters.hessian_matvecs;
        r.pde_solves = obj->counters.pde_solves;
        r.wall_time_s = elapsed();
        return r;
    };
    const double g0 = norm_f(ctx, state->grad, n3);
    rep.grad0 = g0;
    res.records.push_back(record(0, g0, g0));
    float* dir = falloc(ctx, n3);
    float* rhs = falloc(ctx, n3);
    float* trial_v = falloc(ctx, n3);
    if (g0 == 0.0) {
        rep.stop = VR_STOP_ZERO_GRADIENT;
        rep.success = 1;
    } else {
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
            const double eps_H = std::min(0.5, std::sqrt(gk / g0));  // compute_forcing
            vr_pcg_stats pcg;
            if (tl) {
                // split system (solver.cpp:208-221): (I + R H_data R) w = -R g, v~ = R w, R = (beta_v A)^-1/2
                tl->rebuild(state.get(), eps_H);
                const bool zero_mode = reg_symbol(model.norm, 0.0) == 0.0;
                auto R = [&](const float* in, float* out) {
                    op_reg_begin_f32(ctx, in, model.norm, VR_REGOP_INVERSE_SQRT, model.beta_v);
                    op_reg_finish_f32(ctx, out, nullptr);
                };
                float* u = falloc(ctx, n3);
                float* du = falloc(ctx, n3);
                OpF sop = [&](const float* w, float* out) {  // Objective<float>::split_matvec (objective.cpp:158-176)
                    R(w, u);
                    objf32_matvec_impl(obj.get(), state.get(), u, du, false);
                    R(du, out);
                    axpy(ctx, out, 1.0, w, n3);
                    if (zero_mode) {  // + mean(w) per component: A has a zero singular value
                        const long long N = ctx->g.N;
                        for (int c = 0; c < 3; ++c) {
                            F64 dw(ctx, w + c * N, N);
                            double sum[1];
                            sum_components(ctx, dw.p, N, 1, sum);
                            F64 dout(ctx, out + c * N, N);
                            affine(ctx, dout.p, dout.p, N, sum[0] / static_cast<double>(ctx->g.Ng), 1.0);
                            convert_d2f(ctx, dout.p, out + c * N, N);
                        }
                    }
                };
                OpF spc = [&](const float* r, float* z) { tl->apply(r, z); };
                R(state->grad, rhs);
                lincomb(ctx, rhs, -1.0, rhs, 0.0, nullptr, n3);
                pcg = pcg_f32(obj.get(), state.get(), rhs, eps_H, params.max_krylov, precond, dir, &sop, &spc);
                R(dir, dir);
                ffree(ctx, u);
                ffree(ctx, du);
            } else {
                lincomb(ctx, rhs, -1.0, state->grad, 0.0, nullptr, n3);   // scale(rhs, -1)
                pcg = pcg_f32(obj.get(), state.get(), rhs, eps_H, params.max_krylov, precond, dir);
            }
            const double slope = dot_f(ctx, state->grad, dir, ctx->g.N, 3) * hc;  // inner_product
            if (slope >= 0.0) {
                rep.stop = VR_STOP_LINE_SEARCH_FAILURE;
                break;
            }
            // armijo_search (solver.cpp:104-129)
            double alpha = 1.0;
            std::unique_ptr<StateF32> accepted;
            for (int t = 0; t < params.armijo_max_trials; ++t) {
                lincomb(ctx, trial_v, 1.0, state->v, alpha, dir, n3);
                std::unique_ptr<StateF32> trial(objf32_evaluate(obj.get(), trial_v));
                if (trial->objective <= state->objective + params.armijo_c1 * alpha * slope) {
                    accepted = std::move(trial);
                    break;
                }
                alpha *= params.armijo_backtrack;
            }
            if (!accepted) {
                rep.stop = VR_STOP_LINE_SEARCH_FAILURE;
                break;
            }
            state = std::move(accepted);
            objf32_gradient(obj.get(), state.get());
            gk = norm_f(ctx, state->grad, n3);
            ++k;
            vr_iteration_record row = record(k, gk, g0);
            row.step_length = alpha;
            row.forcing = eps_H;
            row.inner_iterations = pcg.iterations;
            res.records.push_back(row);
        }
        rep.outer_iterations = k;
    }
    for (float* p : {dir, rhs, trial_v}) ffree(ctx, p);
    rep.final_objective = state->objective;
    rep.final_mismatch_rel = state->mismatch_rel;
    rep.final_grad_rel = g0 > 0 ? norm_f(ctx, state->grad, n3) / g0 : 0.0;
    rep.fine = obj->counters;
    if (tl) rep.coarse = tl->tl.counters();
    rep.n_records = static_cast<int>(res.records.size());
    VR_CUDA(cudaMemcpyAsync(v_out, state->v, sizeof(float) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
    VR_CUDA(cudaStreamSynchronize(ctx->stream));
    rep.wall_time_s = elapsed();
    state.reset();  // before the objective it points to
    return res;
}

// parameter continuation on the fp32 solve: beta_v 1, 1e-1, ... target
std::vector<GnResult> parameter_continuation_f32(vr_ctx* ctx, const float* mR, const float* mT,
                                                 const float* v0, const vr_model& model,
                                                 const vr_solver_params& params, int precond,
                                                 float* v_out) {
    if (!(model.beta_v <= 1.0)) throw_argument("parameter continuation: target beta_v > 1");
    std::vector<double> levels;
    for (int i = 0;; ++i) {
        const double b = std::pow(10.0, -i);
        if (b <= model.beta_v * (1.0 + 1e-9)) break;
        levels.push_back(b);
    }
    levels.push_back(model.beta_v);
    const long long n3 = 3 * ctx->g.N;
    float* v = falloc(ctx, n3);
    VR_CUDA(cudaMemcpyAsync(v, v0, sizeof(float) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
    std::vector<GnResult> out;
    try {
        for (double b : levels) {
            vr_model m = model;
            m.beta_v = b;
            out.push_back(gauss_newton_solve_f32(ctx, mR, mT, v, m, params, precond, v));
            if (out.back().report.stop == VR_STOP_LINE_SEARCH_FAILURE) break;
        }
        VR_CUDA(cudaMemcpyAsync(v_out, v, sizeof(float) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        ffree(ctx, v);
        throw;
    }
    ffree(ctx, v);
    return out;
}

void objf32_destroy(ObjF32* o) { delete o; }
void statef32_destroy(StateF32* s) { delete s; }
void statef32_scalars(const StateF32* s, double* J, double* mis, double* rel) {
    *J = s->objective;
    *mis = s->mismatch;
    *rel = s->mismatch_rel;
}
const float* statef32_gradient(const StateF32* s) { return s->grad; }
vr_counters objf32_counters(const ObjF32* o) { return o->counters; }
vr_ctx* objf32_ctx(ObjF32* o) { return o->ctx; }
void objf32_copy_gradient(ObjF32* o, const StateF32* s, float* g3) {
    if (!s->grad) throw_logic("gradient: not computed");
    VR_CUDA(cudaMemcpyAsync(g3, s->grad, sizeof(float) * 3 * o->ctx->g.N, cudaMemcpyDeviceToDevice,
                            o->ctx->stream));
    VR_CUDA(cudaStreamSynchronize(o->ctx->stream));
}

}  // namespace vr
