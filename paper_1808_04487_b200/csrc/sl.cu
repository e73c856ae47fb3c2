// sl.cu -- semi-Lagrangian transport on sm_100a: tricubic Lagrange gathers,
// RK2 characteristics, continuity factor and the fused per-time-step kernels of
// the state / adjoint / incremental-state / incremental-adjoint sweeps.
//
// Reference: proj/include/veloreg/interp.hpp:10-126 (weights, stencil, gather),
// proj/src/transport.cpp:11-237 (trace, factor, steps, sweeps),
// proj/src/objective.cpp:9-32,96-99,143-148 (fused gradient accumulation).
//
// Mapping. A CTA owns a 1 x 4 x 32 tile of output points (x1 x x2 x x3; one warp
// is one contiguous x3 run; 128 threads, ~28 resident warps/SM), so the 4x4x4
// stencils of a CTA touch a compact, heavily reused set of L1 lines (84% L1 hit
// rate measured at 256^3; the tile / occupancy sweep is in DESIGN.md). Each
// thread computes its stencil once (u = x / h, 1e-12 node snap, floor, cubic
// Lagrange weights; interp.hpp:32-53) and gathers through L1 with 32-bit
// per-axis offsets and immediate-offset loads for the x3 run. The summation
// keeps the reference's a -> b -> c nesting. (A shared-memory staging of the
// CTA's stencil box was measured slower: fp64 gathers under compressive flow
// cause ~2x bank-conflict wavefronts.)
#include <climits>

#include "vr_common.cuh"

namespace vr {
namespace {

#ifndef VR_TILE_T2
#define VR_TILE_T2 4  // x2 rows per CTA tile (x3 run of 32 per warp)
#endif
#ifndef VR_TILE_T1
#define VR_TILE_T1 1  // x1 planes per CTA tile (1 x 4 x 32, 128 threads: measured best)
#endif
constexpr int kBigT1 = VR_TILE_T1, kBigT2 = VR_TILE_T2;
constexpr int kTileThreads = 32 * kBigT1 * kBigT2;
constexpr int kThreads = 256;  // pointwise kernels
#ifndef VR_SL_WARPS
#define VR_SL_WARPS 28  // resident warps/SM targeted by the gather kernels (72-register cap)
#endif
#define VR_SL_MINB (VR_SL_WARPS * 32 / kTileThreads)

// cubic_weights (interp.hpp:12-18)
__device__ __forceinline__ void cubic_weights(double s, double* w) {
    const double sm1 = s - 1.0, sm2 = s - 2.0, sp1 = s + 1.0;
    w[0] = -s * sm1 * sm2 * (1.0 / 6.0);
    w[1] = sp1 * sm1 * sm2 * 0.5;
    w[2] = -sp1 * s * sm2 * 0.5;
    w[3] = sp1 * s * sm1 * (1.0 / 6.0);
}

// Stencil with UNWRAPPED base index b = floor(u) - 1 per axis; nodes b..b+3
// are taken modulo n (== the reference's ((i-1) mod n + t) mod n).
struct Stencil {
    int b[3];
    double w[3][4];
};

__device__ __forceinline__ void axis_stencil(double x, double h, int& b, double* w) {
    double u = x / h;
    const double r = rint(u);
    if (fabs(u - r) < 1e-12) u = r;
    const double fl = floor(u);
    cubic_weights(u - fl, w);
    b = static_cast<int>(fl) - 1;
}

// i1 is the point's LOCAL plane. On x1 slabs the x1 base becomes slab-relative:
// shifted by a whole period to the image nearest the point (departure points
// are wrapped into [0, 2pi); the shift is exact, the weights are untouched) and
// then offset by the slab origin, so gathers index the halo-padded slab directly.
__device__ __forceinline__ void make_stencil(const GridDims& g, double x1, double x2, double x3,
                                             int i1, Stencil& st) {
    axis_stencil(x1, g.h1, st.b[0], st.w[0]);
    axis_stencil(x2, g.h2, st.b[1], st.w[1]);
    axis_stencil(x3, g.h3, st.b[2], st.w[2]);
    if (g.dist) {
        const int own = g.off1 + i1;
        const int d = st.b[0] - own;
        if (d > g.n1 / 2) st.b[0] -= g.n1;
        if (d < -g.n1 / 2) st.b[0] += g.n1;
        st.b[0] -= g.off1;
    }
}

// power-of-two periodic wrap (two's complement handles negative j)
__device__ __forceinline__ int wrapi(int j, int n) { return j & (n - 1); }

// Gather through L1. Per-axis element offsets are formed once per point in
// 32-bit (a single field has N <= 2^30 elements), so each of the 16 stencil rows
// costs one add + one address and its 4 x3-neighbours are immediate-offset
// loads; only points whose x3 run crosses the periodic seam take the wrapped path.
// On x1 slabs `f` points at the interior of a halo-padded field and x1 planes
// b .. b+3 must lie in [-halo, L + halo); a violation raises flags[1] (checked
// by the host after the sweep) and clamps.
// TF = storage type of the gathered field (double, or float for the fp32 lane: the
// reference's Objective<float> stores fields in fp32 and interpolates in fp64,
// interp.hpp:55-70)
template <class TF>
__device__ __forceinline__ double gather(const TF* __restrict__ f, const GridDims& g,
                                         const Stencil& st) {
    const int n23 = g.n2 * g.n3;
    int b1 = st.b[0];
    if (g.dist && (b1 < -g.halo || b1 + 3 >= g.L + g.halo)) {
        g.flags[1] = 1;
        b1 = b1 < -g.halo ? -g.halo : g.L + g.halo - 4;
    }
    int o12[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int oa = (g.dist ? b1 + a : wrapi(b1 + a, g.n1)) * n23;
#pragma unroll
        for (int b = 0; b < 4; ++b) o12[a][b] = oa + wrapi(st.b[1] + b, g.n2) * g.n3;
    }
    const int b3 = st.b[2];
    double acc = 0.0;
    if (b3 >= 0 && b3 + 3 < g.n3) {
        const TF* f3 = f + b3;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            double acc1 = 0.0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const TF* p = f3 + o12[a][b];
                double acc2 = 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c) acc2 += st.w[2][c] * static_cast<double>(__ldg(p + c));
                acc1 += st.w[1][b] * acc2;
            }
            acc += st.w[0][a] * acc1;
        }
    } else {
        int i3[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) i3[c] = wrapi(b3 + c, g.n3);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            double acc1 = 0.0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const TF* p = f + o12[a][b];
                double acc2 = 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c) acc2 += st.w[2][c] * static_cast<double>(__ldg(p + i3[c]));
                acc1 += st.w[1][b] * acc2;
            }
            acc += st.w[0][a] * acc1;
        }
    }
    return acc;
}

// Tile geometry. BIG: the T1 x T2 x 32 tile (grids with n3 >= 32, n2 >= T2, L >= T1);
// otherwise a runtime tile that fits small test grids.
struct Tile {
    int t1, t2, t3;
};
template <bool BIG>
__device__ __forceinline__ bool tile_point(const GridDims& g, const Tile& t, int& i1, int& i2,
                                           int& i3, long long& idx) {
    const int tid = threadIdx.x;
    int l1, l2, l3, T1, T2, T3;
    if (BIG) {
        T1 = kBigT1, T2 = kBigT2, T3 = 32;
        l3 = tid & 31;
        l2 = (tid >> 5) % kBigT2;
        l1 = (tid >> 5) / kBigT2;
    } else {
        T1 = t.t1, T2 = t.t2, T3 = t.t3;
        l3 = tid % T3;
        l2 = (tid / T3) % T2;
        l1 = tid / (T3 * T2);
    }
    i3 = blockIdx.x * T3 + l3;
    i2 = blockIdx.y * T2 + l2;
    i1 = g.z0 + blockIdx.z * T1 + l1;
    const bool ok = l1 < T1 && i1 < g.z0 + g.zn && i2 < g.n2 && i3 < g.n3;
    idx = ok ? (static_cast<long long>(i1) * g.n2 + i2) * g.n3 + i3 : 0;
    return ok;
}

template <class TD>
__device__ __forceinline__ void load_point(const TD* __restrict__ dep, long long i,
                                           long long N, double& x1, double& x2, double& x3) {
    x1 = static_cast<double>(__ldg(dep + i));
    x2 = static_cast<double>(__ldg(dep + N + i));
    x3 = static_cast<double>(__ldg(dep + 2 * N + i));
}

// ---------------------------------------------------------------------------
// tricubic_interpolate{,2,3} (interp.hpp:80-126)
template <int NF, bool BIG>
__global__ void __launch_bounds__(kTileThreads, NF == 1 ? VR_SL_MINB : VR_SL_MINB * 2 / 3)
    k_tricubic(const double* __restrict__ f, const double* __restrict__ pts, double* __restrict__ out,
               GridDims g, Tile t) {
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    double x1, x2, x3;
    load_point(pts, i, g.N, x1, x2, x3);
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, st);
#pragma unroll
    for (int q = 0; q < NF; ++q) out[q * g.N + i] = gather(f + q * g.N, g, st);
}

// trace_characteristics (transport.cpp:11-42): midpoint from v at the grid
// point, one 3-field gather of v there, wrapped departure point.
template <bool BIG>
__global__ void __launch_bounds__(kTileThreads, VR_SL_MINB * 2 / 3)
    k_trace(const double* __restrict__ v, long long vs, double* __restrict__ dep, GridDims g,
            Tile t, double sign, double dt) {
    // v: component c at v + c*vs (vs = N, or the padded stride on x1 slabs)
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    const double x[3] = {g.h1 * (g.off1 + i1), g.h2 * i2, g.h3 * i3};
    double mid[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) mid[c] = wrap_coord(x[c] + sign * 0.5 * dt * v[c * vs + i]);
    Stencil st;
    make_stencil(g, mid[0], mid[1], mid[2], i1, st);
#pragma unroll
    for (int c = 0; c < 3; ++c)
        dep[c * g.N + i] = wrap_coord(x[c] + sign * dt * gather(v + c * vs, g, st));
}

// continuity_factor (transport.cpp:44-55)
template <bool BIG>
__global__ void __launch_bounds__(kTileThreads, VR_SL_MINB)
    k_factor(const double* __restrict__ div, const double* __restrict__ dep,
             double* __restrict__ factor, GridDims g, Tile t, double half_dt) {
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    const double d = div[i];
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, st);
    factor[i] = exp(half_dt * (d + gather(div, g, st)));
}

// advect_step / continuity_step (transport.cpp:57-68)
template <bool FACTOR, bool BIG>
__global__ void __launch_bounds__(kTileThreads, VR_SL_MINB)
    k_advect(const double* __restrict__ f, const double* __restrict__ dep,
             const double* __restrict__ factor, double* __restrict__ out, GridDims g, Tile t) {
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    const double fac = FACTOR ? factor[i] : 1.0;
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, st);
    const double r = gather(f, g, st);
    out[i] = FACTOR ? r * fac : r;
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
template <int MODE, bool BIG>
__global__ void __launch_bounds__(kTileThreads, VR_SL_MINB)
    k_incstate_step(const double* __restrict__ src, const double* __restrict__ dep,
                    const double* __restrict__ gm, const double* __restrict__ vt,
                    double* __restrict__ dst, GridDims g, Tile t, double hdt,
                    double* __restrict__ b, double wb, double* __restrict__ mt_out) {
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    const double q = qdot(gm, vt, i, g.N);
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, st);
    const double m = gather(src, g, st) + (-hdt) * q;
    const double r = (MODE == 0) ? 1.0 * m + (-hdt) * q : -m;
    dst[i] = r;
    if (mt_out) mt_out[i] = m;  // full Newton keeps the mt history
    if (MODE == 2) {  // b = 0 + (w lam_nt) grad m_nt (objective.cpp:143-148 at j = nt)
        const double wl = wb * r;
#pragma unroll
        for (int a = 0; a < 3; ++a) __stcs(b + a * g.N + i, 0.0 + wl * __ldcs(gm + a * g.N + i));
    }
}

// continuity step + optional fused accumulation bout_a = (b_a + (w * lam) * d_a m_j) [+ add_a]
// (streaming loads / stores for b, gm, add keep L1 for the gather)
template <bool ACC, bool BIG>
__global__ void __launch_bounds__(kTileThreads, VR_SL_MINB)
    k_adjoint_step(const double* __restrict__ src, const double* __restrict__ dep,
                   const double* __restrict__ factor, double* __restrict__ dst,
                   const double* __restrict__ gm, double w, const double* b,
                   const double* __restrict__ add, double* bout, GridDims g, Tile t) {
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    const double fac = factor[i];
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, st);
    const double lam = gather(src, g, st) * fac;
    dst[i] = lam;
    if (ACC) {
        const double wl = w * lam;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            double v = __ldcs(b + a * g.N + i) + wl * __ldcs(gm + a * g.N + i);
            if (add) v = v + __ldcs(add + a * g.N + i);
            __stcs(bout + a * g.N + i, v);
        }
    }
}

// full-Newton inc-adjoint step (transport.cpp:214-222): one stencil, two gathered fields
//   cur_j = I[cur_{j+1}](X) * factor + hdt * (r_j + I[r_{j+1}](X))
template <bool BIG>
__global__ void __launch_bounds__(kTileThreads, VR_SL_MINB * 2 / 3)
    k_adjoint_fn_step(const double* __restrict__ src, const double* __restrict__ rnext,
                      const double* __restrict__ dep, const double* __restrict__ factor,
                      const double* __restrict__ rcur, double hdt, double* __restrict__ dst,
                      GridDims g, Tile t) {
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, st);
    const double li = gather(src, g, st);
    const double si = gather(rnext, g, st);
    dst[i] = li * factor[i] + hdt * (rcur[i] + si);
}

// deformation_map step (postprocess.cpp:40-47): u <- I3[u](X) - half_dt (v(X) + v),
// one stencil for the three components
template <bool BIG>
__global__ void __launch_bounds__(kTileThreads, VR_SL_MINB * 2 / 3)
    k_defmap_step(const double* __restrict__ u, const double* __restrict__ dep,
                  const double* __restrict__ vdep, const double* __restrict__ v, double half_dt,
                  double* __restrict__ out, GridDims g, Tile t, long long ustride) {
    // u / out: component c at + c * ustride (N, or the halo-padded stride on x1 slabs)
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, st);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double ud = gather(u + c * ustride, g, st);
        out[c * ustride + i] = ud - half_dt * (vdep[c * g.N + i] + v[c * g.N + i]);
    }
}

// ---- fp32 lane: the semi-Lagrangian operators of Objective<float>:
// fields and departure points stored in fp32, stencils and sums in fp64, results
// rounded to fp32 (interp.hpp:55-126, transport.cpp:11-42 with T = float) -----------
#ifndef VR_SL_MINB_F32
#define VR_SL_MINB_F32 8  // resident CTAs/SM of the fp32 gathers (swept 4..8: 8 best, 480 vs 486-629 us)
#endif
template <int NF, bool BIG>
__global__ void __launch_bounds__(kTileThreads, NF == 1 ? VR_SL_MINB_F32 : VR_SL_MINB_F32 * 2 / 3)
    k_tricubic_f32(const float* __restrict__ f, const float* __restrict__ pts, float* __restrict__ out,
                   GridDims g, Tile t) {
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    double x1, x2, x3;
    load_point(pts, i, g.N, x1, x2, x3);
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, st);
#pragma unroll
    for (int q = 0; q < NF; ++q) out[q * g.N + i] = static_cast<float>(gather(f + q * g.N, g, st));
}

template <bool BIG>
__global__ void __launch_bounds__(kTileThreads, VR_SL_MINB_F32 * 2 / 3)
    k_trace_f32(const float* __restrict__ v, float* __restrict__ dep, GridDims g, Tile t,
                double sign, double dt) {
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    const double x[3] = {g.h1 * i1, g.h2 * i2, g.h3 * i3};
    double mid[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
        mid[c] = wrap_coord(x[c] + sign * 0.5 * dt * static_cast<double>(v[c * g.N + i]));
    Stencil st;
    make_stencil(g, mid[0], mid[1], mid[2], i1, st);
#pragma unroll
    for (int c = 0; c < 3; ++c)
        dep[c * g.N + i] = static_cast<float>(wrap_coord(x[c] + sign * dt * gather(v + c * g.N, g, st)));
}

// fp32-lane sweep steps, fused like the fp64 ones but with the reference's float
// rounding points (transport.cpp:126-180, objective.cpp:9-32 with T = float)
__device__ __forceinline__ float graddot_f32(const float* __restrict__ gm, const float* __restrict__ vt,
                                             long long i, long long N) {
    float o = 0.0f;  // gradient_dot<float>: out = float(out + d_a m * w_a), a = 0, 1, 2
#pragma unroll
    for (int a = 0; a < 3; ++a)
        o = static_cast<float>(static_cast<double>(o) +
                               static_cast<double>(gm[a * N + i]) * static_cast<double>(vt[a * N + i]));
    return o;
}
// tmp_0 = float(1.0 * 0 + (-hdt) q_0)
__global__ void __launch_bounds__(kThreads)
    k_incstate_first_f32(const float* __restrict__ gm0, const float* __restrict__ vt,
                         float* __restrict__ tmp, long long N, double hdt) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= N) return;
    const float q = graddot_f32(gm0, vt, i, N);
    tmp[i] = static_cast<float>(1.0 * 0.0 + (-hdt) * static_cast<double>(q));
}
// mt_{j+1} = float(float(I[tmp_j](X)) + (-hdt) q_{j+1}); LAST: dst = float(-mt_nt) (terminal),
// else dst = tmp_{j+1} = float(1.0 mt_{j+1} + (-hdt) q_{j+1})
template <bool LAST, bool BIG>
__global__ void __launch_bounds__(kTileThreads, VR_SL_MINB_F32)
    k_incstate_step_f32(const float* __restrict__ src, const float* __restrict__ dep,
                        const float* __restrict__ gm, const float* __restrict__ vt,
                        float* __restrict__ dst, GridDims g, Tile t, double hdt) {
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    const float q = graddot_f32(gm, vt, i, g.N);
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, st);
    const float gv = static_cast<float>(gather(src, g, st));
    const float m = static_cast<float>(static_cast<double>(gv) + (-hdt) * static_cast<double>(q));
    dst[i] = LAST ? static_cast<float>(-m)
                  : static_cast<float>(1.0 * static_cast<double>(m) + (-hdt) * static_cast<double>(q));
}
// continuity_step<float>: dst = float(I[src](X)) * factor (a float product)
template <bool BIG>
__global__ void __launch_bounds__(kTileThreads, VR_SL_MINB_F32)
    k_continuity_f32(const float* __restrict__ src, const float* __restrict__ dep,
                     const float* __restrict__ factor, float* __restrict__ dst, GridDims g, Tile t) {
    int i1, i2, i3;
    long long i;
    if (!tile_point<BIG>(g, t, i1, i2, i3, i)) return;
    double x1, x2, x3;
    load_point(dep, i, g.N, x1, x2, x3);
    const float fac = factor[i];
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, st);
    dst[i] = static_cast<float>(gather(src, g, st)) * fac;
}
// b_a = sum over j = nt..0 of float(b_a + w_j lam_j d_a m_j), the observer order
__global__ void __launch_bounds__(kThreads)
    k_accumulate_f32(const float* __restrict__ lam, const float* __restrict__ gm, int nt, double dt,
                     float* __restrict__ b, long long N) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= N) return;
    float acc[3] = {0.0f, 0.0f, 0.0f};
    for (int j = nt; j >= 0; --j) {
        const double w = (j == 0 || j == nt) ? 0.5 * dt : dt;
        const double wl = w * static_cast<double>(lam[j * N + i]);
        const float* gj = gm + 3LL * j * N;
#pragma unroll
        for (int a = 0; a < 3; ++a)
            acc[a] = static_cast<float>(static_cast<double>(acc[a]) + wl * static_cast<double>(gj[a * N + i]));
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) b[a * N + i] = acc[a];
}

// lv_c = lam * vt_c (transport.cpp:203-207)
__global__ void __launch_bounds__(kThreads)
    k_scale_vec(const double* __restrict__ lam, const double* __restrict__ vt, double* __restrict__ lv,
                GridDims g) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    const double l = lam[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) lv[c * g.N + i] = l * vt[c * g.N + i];
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
    if (!b) return;  // the observer term is accumulated later (sl_accumulate)
    const double wl = w * l;
#pragma unroll
    for (int a = 0; a < 3; ++a) b[a * g.N + i] = 0.0 + wl * gm[a * g.N + i];
}

// b_a = sum_{j = nt..0} (w_j lam_j) d_a m_j (observer order of objective.cpp:143-148)
__global__ void __launch_bounds__(kThreads)
    k_accumulate(const double* __restrict__ lam, long long ls, const double* __restrict__ gm,
                 int nt, double dt, double* __restrict__ b, GridDims g,
                 const double* __restrict__ add, const double* __restrict__ lam2,
                 const double* __restrict__ gm2) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i >= g.N) return;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int j = nt; j >= 0; --j) {
        const double w = (j == 0 || j == nt) ? 0.5 * dt : dt;
        const double wl = w * lam[j * ls + i];
        const double* gj = gm + 3LL * j * g.N;
#pragma unroll
        for (int a = 0; a < 3; ++a) acc[a] = acc[a] + wl * gj[a * g.N + i];
        if (lam2) {  // full Newton: + (w lam_j) d_a mt_j (objective.cpp:146-147)
            const double wl2 = w * lam2[j * ls + i];
            const double* g2 = gm2 + 3LL * j * g.N;
#pragma unroll
            for (int a = 0; a < 3; ++a) acc[a] = acc[a] + wl2 * g2[a * g.N + i];
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) b[a * g.N + i] = add ? acc[a] + add[a * g.N + i] : acc[a];
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
    const double x1 = g.h1 * (g.off1 + i1), x2 = g.h2 * i2, x3 = g.h3 * i3;
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

bool is_big(const GridDims& g) { return g.n3 >= 32 && g.n2 >= kBigT2 && g.L >= kBigT1; }
Tile tile_of(const GridDims& g) {
    Tile t;
    if (is_big(g)) {
        t.t1 = kBigT1, t.t2 = kBigT2, t.t3 = 32;
        return t;
    }
    t.t3 = g.n3 < 32 ? g.n3 : 32;
    t.t2 = g.n2 < 4 ? g.n2 : 4;
    const int rest = kTileThreads / (t.t3 * t.t2);
    t.t1 = g.L < rest ? g.L : rest;
    return t;
}
dim3 tgrid(const GridDims& g, const Tile& t) {
    return dim3(static_cast<unsigned>(g.n3 / t.t3), static_cast<unsigned>(g.n2 / t.t2),
                static_cast<unsigned>((g.zn + t.t1 - 1) / t.t1));
}
unsigned tthreads(const Tile& t) { return static_cast<unsigned>(t.t1 * t.t2 * t.t3); }

// launch KERN<..., BIG> on the tile grid of ctx (BIG chosen from the grid)
#define VR_TILE_LAUNCH(ctx, cat, KERN, ...)                                                        \
    do {                                                                                          \
        const GridDims& g_ = (ctx)->g;                                                            \
        const Tile t_ = tile_of(g_);                                                              \
        if (is_big(g_))                                                                           \
            VR_LAUNCH(ctx, cat, KERN(true)<<<tgrid(g_, t_), tthreads(t_), 0, (ctx)->stream>>>(__VA_ARGS__)); \
        else                                                                                      \
            VR_LAUNCH(ctx, cat, KERN(false)<<<tgrid(g_, t_), tthreads(t_), 0, (ctx)->stream>>>(__VA_ARGS__)); \
    } while (0)

#define K_TRICUBIC1(B) k_tricubic<1, B>
#define K_TRICUBIC2(B) k_tricubic<2, B>
#define K_TRICUBIC3(B) k_tricubic<3, B>
#define K_TRACE(B) k_trace<B>
#define K_FACTOR(B) k_factor<B>
#define K_ADVECT(B) k_advect<false, B>
#define K_CONTINUITY(B) k_advect<true, B>
#define K_INCSTATE0(B) k_incstate_step<0, B>
#define K_INCSTATE1(B) k_incstate_step<1, B>
#define K_INCSTATE2(B) k_incstate_step<2, B>
#define K_ADJ(B) k_adjoint_step<false, B>
#define K_ADJ_ACC(B) k_adjoint_step<true, B>
#define K_ADJ_FN(B) k_adjoint_fn_step<B>
#define K_DEFMAP(B) k_defmap_step<B>
#define K_TRICUBIC1F(B) k_tricubic_f32<1, B>
#define K_TRICUBIC2F(B) k_tricubic_f32<2, B>
#define K_TRICUBIC3F(B) k_tricubic_f32<3, B>
#define K_TRACEF(B) k_trace_f32<B>
#define K_INCSTATEF0(B) k_incstate_step_f32<false, B>
#define K_INCSTATEF1(B) k_incstate_step_f32<true, B>
#define K_CONTINUITYF(B) k_continuity_f32<B>

}  // namespace

void sl_tricubic(vr_ctx* ctx, const double* f, int nfields, const double* pts3, double* out) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    switch (nfields) {
        case 1: VR_TILE_LAUNCH(ctx, "sl_gather", K_TRICUBIC1, f, pts3, out, g, t); break;
        case 2: VR_TILE_LAUNCH(ctx, "sl_gather", K_TRICUBIC2, f, pts3, out, g, t); break;
        case 3: VR_TILE_LAUNCH(ctx, "sl_gather", K_TRICUBIC3, f, pts3, out, g, t); break;
        default: throw_argument("tricubic_interpolate: nfields must be 1, 2 or 3");
    }
}

void sl_trace(vr_ctx* ctx, const double* v3, long long vstride, int nt, int direction,
              double* dep3) {
    Range nvtx("trace_characteristics");
    if (nt < 1) throw_argument("trace_characteristics: n_t must be >= 1");
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    const double dt = 1.0 / nt;
    const double sign = direction == VR_TRACE_BACKWARD ? -1.0 : 1.0;
    VR_TILE_LAUNCH(ctx, "sl_trace", K_TRACE, v3, vstride, dep3, g, t, sign, dt);
}

void sl_factor(vr_ctx* ctx, const double* div_v, const double* dep3, double half_dt,
               double* factor) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    VR_TILE_LAUNCH(ctx, "sl_factor", K_FACTOR, div_v, dep3, factor, g, t, half_dt);
}

void sl_advect(vr_ctx* ctx, const double* f, const double* dep3, double* out) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    VR_TILE_LAUNCH(ctx, "sl_state_step", K_ADVECT, f, dep3, nullptr, out, g, t);
}

void sl_continuity(vr_ctx* ctx, const double* f, const double* dep3, const double* factor,
                   double* out) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    VR_TILE_LAUNCH(ctx, "sl_adjoint_step", K_CONTINUITY, f, dep3, factor, out, g, t);
}

void sl_incstate_first(vr_ctx* ctx, const double* gm0, const double* vt3, double hdt,
                       double* tmp0) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_pointwise", k_incstate_first<<<pgrid(g), kThreads, 0, ctx->stream>>>(gm0, vt3, tmp0, g, hdt, ctx->flag_dev));
}

void sl_incstate_step(vr_ctx* ctx, const double* src, const double* dep3, const double* gm,
                      const double* vt3, double hdt, double* dst, int mode, double* b3, double wb,
                      double* mt_out) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    if (mode == 0)
        VR_TILE_LAUNCH(ctx, "sl_incstate_step", K_INCSTATE0, src, dep3, gm, vt3, dst, g, t, hdt, nullptr, 0.0, mt_out);
    else if (mode == 1)
        VR_TILE_LAUNCH(ctx, "sl_incstate_step", K_INCSTATE1, src, dep3, gm, vt3, dst, g, t, hdt, nullptr, 0.0, mt_out);
    else
        VR_TILE_LAUNCH(ctx, "sl_incstate_step", K_INCSTATE2, src, dep3, gm, vt3, dst, g, t, hdt, b3, wb, mt_out);
}

void sl_adjoint_step(vr_ctx* ctx, const double* src, const double* dep3, const double* factor,
                     double* dst, const double* gm, double w, double* b3, const double* add3,
                     double* bout3) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    if (b3)
        VR_TILE_LAUNCH(ctx, "sl_adjoint_step_acc", K_ADJ_ACC, src, dep3, factor, dst, gm, w, b3, add3,
                       bout3 ? bout3 : b3, g, t);
    else
        VR_TILE_LAUNCH(ctx, "sl_adjoint_step", K_ADJ, src, dep3, factor, dst, nullptr, 0.0, nullptr,
                       nullptr, nullptr, g, t);
}

void sl_grad_terminal(vr_ctx* ctx, const double* mR, const double* mfinal, const double* gm,
                      double w, double* lam, double* b3) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_pointwise", k_grad_terminal<<<pgrid(g), kThreads, 0, ctx->stream>>>(mR, mfinal, gm, w, lam, b3, g));
}

void sl_accumulate(vr_ctx* ctx, const double* lam_hist, const double* gm_hist, int nt, double dt,
                   double* b3, const double* add3, const double* lam2_hist,
                   const double* gm2_hist) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_accumulate", k_accumulate<<<pgrid(g), kThreads, 0, ctx->stream>>>(lam_hist, ctx->hstride, gm_hist, nt, dt, b3, g, add3, lam2_hist, gm2_hist));
}

void sl_adjoint_fn_step(vr_ctx* ctx, const double* src, const double* rnext, const double* dep3,
                        const double* factor, const double* rcur, double hdt, double* dst) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    VR_TILE_LAUNCH(ctx, "sl_adjoint_step", K_ADJ_FN, src, rnext, dep3, factor, rcur, hdt, dst, g, t);
}

void sl_defmap_step(vr_ctx* ctx, const double* u3, const double* dep3, const double* vdep3,
                    const double* v3, double half_dt, double* out3) {
    // u3 / out3: interiors of 3-component fields with stride ctx->hstride (== N on one GPU)
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    VR_TILE_LAUNCH(ctx, "sl_defmap_step", K_DEFMAP, u3, dep3, vdep3, v3, half_dt, out3, g, t, ctx->hstride);
}

void sl_tricubic_f32(vr_ctx* ctx, const float* f, int nfields, const float* pts3, float* out) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    switch (nfields) {
        case 1: VR_TILE_LAUNCH(ctx, "sl_gather_f32", K_TRICUBIC1F, f, pts3, out, g, t); break;
        case 2: VR_TILE_LAUNCH(ctx, "sl_gather_f32", K_TRICUBIC2F, f, pts3, out, g, t); break;
        case 3: VR_TILE_LAUNCH(ctx, "sl_gather_f32", K_TRICUBIC3F, f, pts3, out, g, t); break;
        default: throw_argument("tricubic_interpolate: nfields must be 1, 2 or 3");
    }
}
__global__ void __launch_bounds__(kThreads)
    k_nonfinite_f32(const float* __restrict__ a, long long n, int* __restrict__ flag) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i < n && !isfinite(a[i])) *flag = 1;
}
__global__ void __launch_bounds__(kThreads)
    k_f2d(const float* __restrict__ a, double* __restrict__ b, long long n) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i < n) b[i] = static_cast<double>(a[i]);
}
__global__ void __launch_bounds__(kThreads)
    k_d2f(const double* __restrict__ a, float* __restrict__ b, long long n) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (i < n) b[i] = static_cast<float>(a[i]);
}
void convert_f2d(vr_ctx* ctx, const float* a, double* b, long long n) {
    VR_LAUNCH(ctx, "sl_pointwise", k_f2d<<<grid_1d(n, kThreads), kThreads, 0, ctx->stream>>>(a, b, n));
}
void convert_d2f(vr_ctx* ctx, const double* a, float* b, long long n) {
    VR_LAUNCH(ctx, "sl_pointwise", k_d2f<<<grid_1d(n, kThreads), kThreads, 0, ctx->stream>>>(a, b, n));
}
bool all_finite_f32(vr_ctx* ctx, const float* a, long long n) {
    drain_flags(ctx);
    VR_CUDA(cudaMemsetAsync(ctx->flag_dev, 0, sizeof(int), ctx->stream));
    VR_LAUNCH(ctx, "sl_pointwise", k_nonfinite_f32<<<grid_1d(n, kThreads), kThreads, 0, ctx->stream>>>(a, n, ctx->flag_dev));
    VR_CUDA(cudaMemcpyAsync(ctx->flag_host, ctx->flag_dev, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    VR_CUDA(cudaStreamSynchronize(ctx->stream));
    return ctx->flag_host[0] == 0;
}
void sl_incstate_first_f32(vr_ctx* ctx, const float* gm0, const float* vt3, double hdt, float* tmp0) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_pointwise", k_incstate_first_f32<<<pgrid(g), kThreads, 0, ctx->stream>>>(gm0, vt3, tmp0, g.N, hdt));
}
void sl_incstate_step_f32(vr_ctx* ctx, const float* src, const float* dep3, const float* gm,
                          const float* vt3, double hdt, float* dst, bool last) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    if (last)
        VR_TILE_LAUNCH(ctx, "sl_incstate_step_f32", K_INCSTATEF1, src, dep3, gm, vt3, dst, g, t, hdt);
    else
        VR_TILE_LAUNCH(ctx, "sl_incstate_step_f32", K_INCSTATEF0, src, dep3, gm, vt3, dst, g, t, hdt);
}
void sl_continuity_f32(vr_ctx* ctx, const float* src, const float* dep3, const float* factor, float* dst) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    VR_TILE_LAUNCH(ctx, "sl_adjoint_step_f32", K_CONTINUITYF, src, dep3, factor, dst, g, t);
}
void sl_accumulate_f32(vr_ctx* ctx, const float* lam_hist, const float* gm_hist, int nt, double dt,
                       float* b3) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_accumulate_f32", k_accumulate_f32<<<pgrid(g), kThreads, 0, ctx->stream>>>(lam_hist, gm_hist, nt, dt, b3, g.N));
}
void sl_trace_f32(vr_ctx* ctx, const float* v3, int nt, int direction, float* dep3) {
    if (nt < 1) throw_argument("trace_characteristics: n_t must be >= 1");
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    const double sign = direction == VR_TRACE_BACKWARD ? -1.0 : 1.0;
    VR_TILE_LAUNCH(ctx, "sl_trace_f32", K_TRACEF, v3, dep3, g, t, sign, 1.0 / nt);
}

void sl_scale_vec(vr_ctx* ctx, const double* lam, const double* vt3, double* out3) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_pointwise", k_scale_vec<<<pgrid(g), kThreads, 0, ctx->stream>>>(lam, vt3, out3, g));
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
