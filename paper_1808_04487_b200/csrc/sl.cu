// sl.cu -- semi-Lagrangian transport on sm_100a: tricubic Lagrange gathers,
// RK2 characteristics, continuity factor and the fused per-time-step kernels of
// the state / adjoint / incremental-state / incremental-adjoint sweeps.
//
// Reference: proj/include/veloreg/interp.hpp:10-126 (weights, stencil, gather),
// proj/src/transport.cpp:11-237 (trace, factor, steps, sweeps),
// proj/src/objective.cpp:9-32,96-99,143-148 (fused gradient accumulation).
//
// Every kernel is one thread per output grid point, consecutive threads along
// the contiguous x3 axis, so departure-point loads are coalesced and the 4x4x4
// stencil rows of neighbouring threads overlap in L1. The stencil arithmetic
// follows interp.hpp:32-53 exactly (u = x / h, 1e-12 node snap, floor, wrapped
// base (i-1) mod n); the gather keeps the reference's a -> b -> c nesting.
#include "vr_common.cuh"

namespace vr {
namespace {

// cubic_weights (interp.hpp:12-18)
__device__ __forceinline__ void cubic_weights(double s, double* w) {
    const double sm1 = s - 1.0, sm2 = s - 2.0, sp1 = s + 1.0;
    w[0] = -s * sm1 * sm2 * (1.0 / 6.0);
    w[1] = sp1 * sm1 * sm2 * 0.5;
    w[2] = -sp1 * s * sm2 * 0.5;
    w[3] = sp1 * s * sm1 * (1.0 / 6.0);
}

struct Stencil {
    long long o1[4];  // i1 * n2
    int i2[4];
    int i3[4];
    double w1[4], w2[4], w3[4];
    bool contig3;  // i3 indices consecutive (no wrap)
};

// TricubicStencil ctor, per axis (interp.hpp:32-53)
__device__ __forceinline__ void axis_stencil(double x, double h, int n, int* idx, double* w) {
    double u = x / h;
    const double r = rint(u);
    if (fabs(u - r) < 1e-12) u = r;
    const double fl = floor(u);
    const double s = u - fl;
    const int i = static_cast<int>(fl);
    cubic_weights(s, w);
    int base = i - 1;
    base %= n;
    if (base < 0) base += n;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int j = base + t;
        idx[t] = j < n ? j : j - n;
    }
}

__device__ __forceinline__ void make_stencil(const GridDims& g, double x1, double x2, double x3,
                                             Stencil& st) {
    int i1[4];
    axis_stencil(x1, g.h1, g.n1, i1, st.w1);
    axis_stencil(x2, g.h2, g.n2, st.i2, st.w2);
    axis_stencil(x3, g.h3, g.n3, st.i3, st.w3);
#pragma unroll
    for (int t = 0; t < 4; ++t) st.o1[t] = static_cast<long long>(i1[t]) * g.n2;
    st.contig3 = st.i3[3] == st.i3[0] + 3;
}

// gather (interp.hpp:55-72): sum_a w1[a] sum_b w2[b] sum_c w3[c] f
__device__ __forceinline__ double gather(const double* __restrict__ f, const GridDims& g,
                                         const Stencil& st) {
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double acc1 = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double* row = f + (st.o1[a] + st.i2[b]) * g.n3;
            double acc2 = 0.0;
            if (st.contig3) {
                const double* p = row + st.i3[0];
#pragma unroll
                for (int c = 0; c < 4; ++c) acc2 += st.w3[c] * __ldg(p + c);
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) acc2 += st.w3[c] * __ldg(row + st.i3[c]);
            }
            acc1 += st.w2[b] * acc2;
        }
        acc += st.w1[a] * acc1;
    }
    return acc;
}

__device__ __forceinline__ void load_point(const double* __restrict__ dep, long long i,
                                           long long N, double& x1, double& x2, double& x3) {
    x1 = __ldg(dep + i);
    x2 = __ldg(dep + N + i);
    x3 = __ldg(dep + 2 * N + i);
}

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
template <int NF>
__global__ void __launch_bounds__(kThreads)
    k_tricubic(const double* __restrict__ f, const double* __restrict__ pts, double* __restrict__ out,
               GridDims g) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    double x1, x2, x3;
    load_point(pts, i, g.N, x1, x2, x3);
    Stencil st;
    make_stencil(g, x1, x2, x3, st);
#pragma unroll
    for (int q = 0; q < NF; ++q) out[q * g.N + i] = gather(f + q * g.N, g, st);
}

// trace_characteristics (transport.cpp:11-42)
__global__ void __launch_bounds__(kThreads)
    k_trace(const double* __restrict__ v, double* __restrict__ dep, GridDims g, double sign,
            double dt) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    long long r = i;
    const int i3 = static_cast<int>(r % g.n3);
    r /= g.n3;
    const int i2 = static_cast<int>(r % g.n2);
    const int i1 = static_cast<int>(r / g.n2);
    const double x[3] = {g.h1 * i1, g.h2 * i2, g.h3 * i3};
    double mid[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) mid[c] = wrap_coord(x[c] + sign * 0.5 * dt * v[c * g.N + i]);
    Stencil st;
    make_stencil(g, mid[0], mid[1], mid[2], st);
#pragma unroll
    for (int c = 0; c < 3; ++c)
        dep[c * g.N + i] = wrap_coord(x[c] + sign * dt * gather(v + c * g.N, g, st));
}

// continuity_factor (transport.cpp:44-55)
__global__ void __launch_bounds__(kThreads)
    k_factor(const double* __restrict__ div, const double* __restrict__ dep,
             double* __restrict__ factor, GridDims g, double half_dt) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    Stencil st;
    make_stencil(g, x1, x2, x3, st);
    const double at_dep = gather(div, g, st);
    factor[i] = exp(half_dt * (div[i] + at_dep));
}

// advect_step / continuity_step (transport.cpp:57-68)
template <bool FACTOR>
__global__ void __launch_bounds__(kThreads)
    k_advect(const double* __restrict__ f, const double* __restrict__ dep,
             const double* __restrict__ factor, double* __restrict__ out, GridDims g) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    Stencil st;
    make_stencil(g, x1, x2, x3, st);
    double v = gather(f, g, st);
    if (FACTOR) v = v * factor[i];
    out[i] = v;
}

// q = grad m . vt (transport.cpp:126-148 accumulation order: ((0 + d0 w0) + d1 w1) + d2 w2)
__device__ __forceinline__ double qdot(const double* __restrict__ gm, const double* __restrict__ vt,
                                       long long i, long long N) {
    double q = 0.0;
    q = q + gm[i] * vt[i];
    q = q + gm[N + i] * vt[N + i];
    q = q + gm[2 * N + i] * vt[2 * N + i];
    return q;
}

// solve_inc_state, j = 0 (transport.cpp:159-167): tmp = 1.0 * 0 + (-hdt) * q_0
__global__ void __launch_bounds__(kThreads)
    k_incstate_first(const double* __restrict__ gm0, const double* __restrict__ vt,
                     double* __restrict__ tmp, GridDims g, double hdt, int* __restrict__ nonfinite) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    const double a = vt[i], b = vt[g.N + i], c = vt[2 * g.N + i];
    if (!(isfinite(a) && isfinite(b) && isfinite(c))) *nonfinite = 1;
    tmp[i] = 1.0 * 0.0 + (-hdt) * qdot(gm0, vt, i, g.N);
}

// solve_inc_state step j (transport.cpp:165-170):
//   mt_{j+1} = I[tmp_j](X_bwd) - hdt q_{j+1};  MODE 0: tmp_{j+1} = mt_{j+1} - hdt q_{j+1}
//   MODE 1 (last step): terminal = -mt_nt (objective.cpp:138-140)
template <int MODE>
__global__ void __launch_bounds__(kThreads)
    k_incstate_step(const double* __restrict__ src, const double* __restrict__ dep,
                    const double* __restrict__ gm, const double* __restrict__ vt,
                    double* __restrict__ dst, GridDims g, double hdt) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    Stencil st;
    make_stencil(g, x1, x2, x3, st);
    const double adv = gather(src, g, st);
    const double q = qdot(gm, vt, i, g.N);
    const double m = adv + (-hdt) * q;
    dst[i] = (MODE == 0) ? 1.0 * m + (-hdt) * q : -m;
}

// continuity step + optional fused accumulation b_a += (w * lam) * d_a m_j
template <bool ACC>
__global__ void __launch_bounds__(kThreads)
    k_adjoint_step(const double* __restrict__ src, const double* __restrict__ dep,
                   const double* __restrict__ factor, double* __restrict__ dst,
                   const double* __restrict__ gm, double w, double* __restrict__ b, GridDims g) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    Stencil st;
    make_stencil(g, x1, x2, x3, st);
    const double lam = gather(src, g, st) * factor[i];
    dst[i] = lam;
    if (ACC) {
        const double wl = w * lam;
#pragma unroll
        for (int a = 0; a < 3; ++a) b[a * g.N + i] = b[a * g.N + i] + wl * gm[a * g.N + i];
    }
}

// compute_gradient terminal (objective.cpp:91-99): lam = m_R - m_nt; b = (w lam) grad m_nt
__global__ void __launch_bounds__(kThreads)
    k_grad_terminal(const double* __restrict__ mR, const double* __restrict__ mfin,
                    const double* __restrict__ gm, double w, double* __restrict__ lam,
                    double* __restrict__ b, GridDims g) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    const double l = 1.0 * mR[i] + (-1.0) * mfin[i];
    lam[i] = l;
    const double wl = w * l;
#pragma unroll
    for (int a = 0; a < 3; ++a) b[a * g.N + i] = 0.0 + wl * gm[a * g.N + i];
}

// b_a = sum_{j = nt..0} (w_j lam_j) d_a m_j (observer order of objective.cpp:143-148)
__global__ void __launch_bounds__(kThreads)
    k_accumulate(const double* __restrict__ lam, const double* __restrict__ gm, int nt, double dt,
                 double* __restrict__ b, GridDims g) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int j = nt; j >= 0; --j) {
        const double w = (j == 0 || j == nt) ? 0.5 * dt : dt;
        const double wl = w * lam[j * g.N + i];
        const double* gj = gm + 3LL * j * g.N;
#pragma unroll
        for (int a = 0; a < 3; ++a) acc[a] = acc[a] + wl * gj[a * g.N + i];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) b[a * g.N + i] = acc[a];
}

__global__ void __launch_bounds__(kThreads)
    k_gradient_dot(const double* __restrict__ gm, const double* __restrict__ w,
                   double* __restrict__ out, GridDims g) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    out[i] = qdot(gm, w, i, g.N);
}

// generate_synthetic (synthetic.cpp:10-34): analytic m_T and v*
__global__ void __launch_bounds__(kThreads)
    k_synth(double amplitude, double* __restrict__ mT, double* __restrict__ v, GridDims g) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    long long r = i;
    const int i3 = static_cast<int>(r % g.n3);
    r /= g.n3;
    const int i2 = static_cast<int>(r % g.n2);
    const int i1 = static_cast<int>(r / g.n2);
    const double x1 = g.h1 * i1, x2 = g.h2 * i2, x3 = g.h3 * i3;
    const double s1 = sin(x1), s2 = sin(x2), s3 = sin(x3);
    mT[i] = (s1 * s1 + s2 * s2 + s3 * s3) / 3.0;
    const double v0 = sin(x3) * cos(x2) * sin(x2);
    const double v1 = sin(x1) * cos(x3) * sin(x3);
    const double v2 = sin(x2) * cos(x1) * sin(x1);
    v[i] = amplitude * v0;
    v[g.N + i] = amplitude * v1;
    v[2 * g.N + i] = amplitude * v2;
}

unsigned pgrid(const GridDims& g) { return grid_1d(g.N, kThreads); }

}  // namespace

void sl_tricubic(vr_ctx* ctx, const double* f, int nfields, const double* pts3, double* out) {
    const GridDims& g = ctx->g;
    switch (nfields) {
        case 1: VR_LAUNCH(ctx, "sl_gather", k_tricubic<1><<<pgrid(g), kThreads, 0, ctx->stream>>>(f, pts3, out, g)); break;
        case 2: VR_LAUNCH(ctx, "sl_gather", k_tricubic<2><<<pgrid(g), kThreads, 0, ctx->stream>>>(f, pts3, out, g)); break;
        case 3: VR_LAUNCH(ctx, "sl_gather", k_tricubic<3><<<pgrid(g), kThreads, 0, ctx->stream>>>(f, pts3, out, g)); break;
        default: throw_argument("tricubic_interpolate: nfields must be 1, 2 or 3");
    }
}

void sl_trace(vr_ctx* ctx, const double* v3, int nt, int direction, double* dep3) {
    if (nt < 1) throw_argument("trace_characteristics: n_t must be >= 1");
    const GridDims& g = ctx->g;
    const double dt = 1.0 / nt;
    const double sign = direction == VR_TRACE_BACKWARD ? -1.0 : 1.0;
    VR_LAUNCH(ctx, "sl_trace", k_trace<<<pgrid(g), kThreads, 0, ctx->stream>>>(v3, dep3, g, sign, dt));
}

void sl_factor(vr_ctx* ctx, const double* div_v, const double* dep3, double half_dt,
               double* factor) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_factor", k_factor<<<pgrid(g), kThreads, 0, ctx->stream>>>(div_v, dep3, factor, g, half_dt));
}

void sl_advect(vr_ctx* ctx, const double* f, const double* dep3, double* out) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_state_step", k_advect<false><<<pgrid(g), kThreads, 0, ctx->stream>>>(f, dep3, nullptr, out, g));
}

void sl_continuity(vr_ctx* ctx, const double* f, const double* dep3, const double* factor,
                   double* out) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_adjoint_step", k_advect<true><<<pgrid(g), kThreads, 0, ctx->stream>>>(f, dep3, factor, out, g));
}

void sl_incstate_first(vr_ctx* ctx, const double* gm0, const double* vt3, double hdt,
                       double* tmp0) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_pointwise", k_incstate_first<<<pgrid(g), kThreads, 0, ctx->stream>>>(gm0, vt3, tmp0, g, hdt, ctx->flag_dev));
}

void sl_incstate_step(vr_ctx* ctx, const double* src, const double* dep3, const double* gm,
                      const double* vt3, double hdt, double* dst, int mode) {
    const GridDims& g = ctx->g;
    if (mode == 0)
        VR_LAUNCH(ctx, "sl_incstate_step", k_incstate_step<0><<<pgrid(g), kThreads, 0, ctx->stream>>>(src, dep3, gm, vt3, dst, g, hdt));
    else
        VR_LAUNCH(ctx, "sl_incstate_step", k_incstate_step<1><<<pgrid(g), kThreads, 0, ctx->stream>>>(src, dep3, gm, vt3, dst, g, hdt));
}

void sl_adjoint_step(vr_ctx* ctx, const double* src, const double* dep3, const double* factor,
                     double* dst, const double* gm, double w, double* b3) {
    const GridDims& g = ctx->g;
    if (b3)
        VR_LAUNCH(ctx, "sl_adjoint_step_acc", k_adjoint_step<true><<<pgrid(g), kThreads, 0, ctx->stream>>>(src, dep3, factor, dst, gm, w, b3, g));
    else
        VR_LAUNCH(ctx, "sl_adjoint_step", k_adjoint_step<false><<<pgrid(g), kThreads, 0, ctx->stream>>>(src, dep3, factor, dst, nullptr, 0.0, nullptr, g));
}

void sl_grad_terminal(vr_ctx* ctx, const double* mR, const double* mfinal, const double* gm,
                      double w, double* lam, double* b3) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_pointwise", k_grad_terminal<<<pgrid(g), kThreads, 0, ctx->stream>>>(mR, mfinal, gm, w, lam, b3, g));
}

void sl_accumulate(vr_ctx* ctx, const double* lam_hist, const double* gm_hist, int nt, double dt,
                   double* b3) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_accumulate", k_accumulate<<<pgrid(g), kThreads, 0, ctx->stream>>>(lam_hist, gm_hist, nt, dt, b3, g));
}

void sl_gradient_dot(vr_ctx* ctx, const double* gm3, const double* w3, double* out) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_pointwise", k_gradient_dot<<<pgrid(g), kThreads, 0, ctx->stream>>>(gm3, w3, out, g));
}

void synth_fill(vr_ctx* ctx, double amplitude, double* m_T, double* v3) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "synth", k_synth<<<pgrid(g), kThreads, 0, ctx->stream>>>(amplitude, m_T, v3, g));
}

}  // namespace vr
