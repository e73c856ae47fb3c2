// sl.cu -- semi-Lagrangian transport on sm_100a: tricubic Lagrange gathers,
// RK2 characteristics, continuity factor and the fused per-time-step kernels of
// the state / adjoint / incremental-state / incremental-adjoint sweeps.
//
// Reference: proj/include/veloreg/interp.hpp:10-126 (weights, stencil, gather),
// proj/src/transport.cpp:11-237 (trace, factor, steps, sweeps),
// proj/src/objective.cpp:9-32,96-99,143-148 (fused gradient accumulation).
//
// Tile gather. A CTA owns a t1 x t2 x t3 tile of output points (t3 = 32 along
// the contiguous axis, so a warp is one x3 run). Every thread first computes
// its stencil (u = x / h, 1e-12 node snap, floor, weights; interp.hpp:32-53);
// the CTA then reduces the bounding box of all 4x4x4 stencils. Because the
// velocity is smooth the box is only a few voxels larger than the tile, so the
// CTA stages it in shared memory with coalesced loads (periodic wrap resolved
// once per box element) and the 64-point gathers read shared memory instead of
// going through L1/L2. If the box does not fit (arbitrary query points, huge
// CFL) the CTA falls back to direct wrapped global gathers. Both paths keep the
// reference's a -> b -> c summation order.
#include <climits>

#include "vr_common.cuh"

namespace vr {
namespace {

constexpr int kTileThreads = 256;
constexpr int kBoxCap = 6144;  // doubles of staged box per CTA (48 KB)
constexpr int kThreads = 256;  // pointwise kernels

// cubic_weights (interp.hpp:12-18)
__device__ __forceinline__ void cubic_weights(double s, double* w) {
    const double sm1 = s - 1.0, sm2 = s - 2.0, sp1 = s + 1.0;
    w[0] = -s * sm1 * sm2 * (1.0 / 6.0);
    w[1] = sp1 * sm1 * sm2 * 0.5;
    w[2] = -sp1 * s * sm2 * 0.5;
    w[3] = sp1 * s * sm1 * (1.0 / 6.0);
}

// Stencil with UNWRAPPED base index b = floor(u) - 1 per axis; the stencil
// nodes are b..b+3 taken modulo n (== the reference's ((i-1) mod n + t) mod n).
struct Stencil {
    int b[3];
    double w[3][4];
};

// `own` is the output point's grid index on this axis: the integer base is
// shifted by a whole period to the image nearest to it (exact; the weights are
// computed from the unshifted u exactly as the reference), so departure points
// wrapped across the seam still give compact CTA boxes.
__device__ __forceinline__ void axis_stencil(double x, double h, int n, int own, int& b,
                                             double* w) {
    double u = x / h;
    const double r = rint(u);
    if (fabs(u - r) < 1e-12) u = r;
    const double fl = floor(u);
    cubic_weights(u - fl, w);
    b = static_cast<int>(fl) - 1;
    const int d = b - own;
    if (d > n / 2)
        b -= n * ((d + n / 2) / n);
    else if (d < -n / 2)
        b += n * ((-d + n / 2) / n);
}

__device__ __forceinline__ void make_stencil(const GridDims& g, double x1, double x2, double x3,
                                             int o1, int o2, int o3, Stencil& st) {
    axis_stencil(x1, g.h1, g.n1, o1, st.b[0], st.w[0]);
    axis_stencil(x2, g.h2, g.n2, o2, st.b[1], st.w[1]);
    axis_stencil(x3, g.h3, g.n3, o3, st.b[2], st.w[2]);
}

// power-of-two periodic wrap (two's complement handles negative j)
__device__ __forceinline__ int wrapi(int j, int n) { return j & (n - 1); }

// direct gather from global memory (fallback path)
__device__ __forceinline__ double global_gather(const double* __restrict__ f, const GridDims& g,
                                                const Stencil& st) {
    int i3[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) i3[c] = wrapi(st.b[2] + c, g.n3);
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const long long o1 = static_cast<long long>(wrapi(st.b[0] + a, g.n1)) * g.n2;
        double acc1 = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double* row = f + (o1 + wrapi(st.b[1] + b, g.n2)) * g.n3;
            double acc2 = 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c) acc2 += st.w[2][c] * __ldg(row + i3[c]);
            acc1 += st.w[1][b] * acc2;
        }
        acc += st.w[0][a] * acc1;
    }
    return acc;
}

struct Box {
    int m[3];  // min unwrapped base per axis
    int e[3];  // extents (max base - min base + 4)
    int size;  // e0 * e1 * e2
};

// CTA-wide bounding box of the active threads' stencils (all threads call).
__device__ __forceinline__ Box block_box(const Stencil& st, bool active) {
    __shared__ int red[kTileThreads / 32][6];
    __shared__ Box box_s;
    int v[6];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        v[a] = active ? st.b[a] : INT_MAX;
        v[3 + a] = active ? st.b[a] : INT_MIN;
    }
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        v[a] = __reduce_min_sync(full, v[a]);
        v[3 + a] = __reduce_max_sync(full, v[3 + a]);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int k = 0; k < 6; ++k) red[warp][k] = v[k];
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        int r[6];
        for (int k = 0; k < 6; ++k) r[k] = red[0][k];
        for (int w = 1; w < nw; ++w)
            for (int a = 0; a < 3; ++a) {
                r[a] = min(r[a], red[w][a]);
                r[3 + a] = max(r[3 + a], red[w][3 + a]);
            }
        Box b;
        long long size = 1;
        for (int a = 0; a < 3; ++a) {
            b.m[a] = r[a];
            const long long e = static_cast<long long>(r[3 + a]) - r[a] + 4;
            b.e[a] = static_cast<int>(e < INT_MAX ? e : INT_MAX);
            size *= e;
        }
        b.size = static_cast<int>(size < INT_MAX ? size : INT_MAX);
        box_s = b;
    }
    __syncthreads();
    return box_s;
}

// stage one field's box in shared memory: one warp per (j1, j2) box row, lanes
// along the contiguous x3 run (coalesced), no per-element integer division
__device__ __forceinline__ void box_load(const double* __restrict__ f, const GridDims& g,
                                         const Box& bx, double* __restrict__ sbox) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = (blockDim.x + 31) >> 5;
    const int rows = bx.e[0] * bx.e[1];
    for (int row = warp; row < rows; row += nwarps) {
        const int j1 = row / bx.e[1];
        const int j2 = row - j1 * bx.e[1];
        const double* src = f + (static_cast<long long>(wrapi(bx.m[0] + j1, g.n1)) * g.n2 +
                                 wrapi(bx.m[1] + j2, g.n2)) * g.n3;
        double* dst = sbox + row * bx.e[2];
        for (int j3 = lane; j3 < bx.e[2]; j3 += 32) dst[j3] = __ldg(src + wrapi(bx.m[2] + j3, g.n3));
    }
}

__device__ __forceinline__ double box_gather(const double* __restrict__ sbox, const Box& bx,
                                             const Stencil& st) {
    const int e3 = bx.e[2], e23 = bx.e[1] * bx.e[2];
    const double* p0 = sbox + ((st.b[0] - bx.m[0]) * bx.e[1] + (st.b[1] - bx.m[1])) * e3 +
                       (st.b[2] - bx.m[2]);
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double acc1 = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double* p = p0 + a * e23 + b * e3;
            double acc2 = 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c) acc2 += st.w[2][c] * p[c];
            acc1 += st.w[1][b] * acc2;
        }
        acc += st.w[0][a] * acc1;
    }
    return acc;
}

// Gather NF fields at this thread's stencil; all threads of the CTA must call.
// g.sl_mode: 0 = stage the CTA box in shared memory, 1 = L1-cached global gathers
template <int NF>
__device__ __forceinline__ void tile_gather(const double* const (&f)[NF], const GridDims& g,
                                            const Stencil& st, bool active, double (&out)[NF]) {
    extern __shared__ double sbox[];
    if (g.sl_mode == 1) {
        if (active) {
#pragma unroll
            for (int q = 0; q < NF; ++q) out[q] = global_gather(f[q], g, st);
        }
        return;
    }
    const Box bx = block_box(st, active);
    if (bx.size <= kBoxCap / NF) {  // uniform across the CTA
#pragma unroll
        for (int q = 0; q < NF; ++q) box_load(f[q], g, bx, sbox + q * bx.size);
        __syncthreads();
        if (active) {
#pragma unroll
            for (int q = 0; q < NF; ++q) out[q] = box_gather(sbox + q * bx.size, bx, st);
        }
    } else if (active) {
#pragma unroll
        for (int q = 0; q < NF; ++q) out[q] = global_gather(f[q], g, st);
    }
}

// tile geometry: CTA (bx, by, bz) covers i3 in [bx t3, ...), i2 in [by t2, ...), i1 in [bz t1, ...)
struct Tile {
    int t1, t2, t3;
};
__device__ __forceinline__ bool tile_point(const GridDims& g, const Tile& t, int& i1, int& i2,
                                           int& i3, long long& idx) {
    const int tid = threadIdx.x;
    const int l3 = tid % t.t3;
    const int l2 = (tid / t.t3) % t.t2;
    const int l1 = tid / (t.t3 * t.t2);
    i3 = blockIdx.x * t.t3 + l3;
    i2 = blockIdx.y * t.t2 + l2;
    i1 = blockIdx.z * t.t1 + l1;
    const bool ok = l1 < t.t1 && i1 < g.n1 && i2 < g.n2 && i3 < g.n3;
    idx = ok ? (static_cast<long long>(i1) * g.n2 + i2) * g.n3 + i3 : 0;
    return ok;
}

__device__ __forceinline__ void load_point(const double* __restrict__ dep, long long i,
                                           long long N, double& x1, double& x2, double& x3) {
    x1 = __ldg(dep + i);
    x2 = __ldg(dep + N + i);
    x3 = __ldg(dep + 2 * N + i);
}

// ---------------------------------------------------------------------------
// tricubic_interpolate{,2,3} (interp.hpp:80-126)
template <int NF>
__global__ void __launch_bounds__(kTileThreads, NF == 1 ? 3 : 2)
    k_tricubic(const double* __restrict__ f, const double* __restrict__ pts, double* __restrict__ out,
               GridDims g, Tile t) {
    int i1, i2, i3;
    long long i;
    const bool act = tile_point(g, t, i1, i2, i3, i);
    double x1 = 0, x2 = 0, x3 = 0;
    if (act) load_point(pts, i, g.N, x1, x2, x3);
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, i2, i3, st);
    const double* fs[NF];
#pragma unroll
    for (int q = 0; q < NF; ++q) fs[q] = f + q * g.N;
    double r[NF];
    tile_gather<NF>(fs, g, st, act, r);
    if (act) {
#pragma unroll
        for (int q = 0; q < NF; ++q) out[q * g.N + i] = r[q];
    }
}

// trace_characteristics (transport.cpp:11-42): midpoint from v at the grid
// point, one 3-field gather of v there, wrapped departure point.
__global__ void __launch_bounds__(kTileThreads, 2)
    k_trace(const double* __restrict__ v, double* __restrict__ dep, GridDims g, Tile t,
            double sign, double dt) {
    int i1, i2, i3;
    long long i;
    const bool act = tile_point(g, t, i1, i2, i3, i);
    const double x[3] = {g.h1 * i1, g.h2 * i2, g.h3 * i3};
    double mid[3] = {0, 0, 0};
    if (act) {
#pragma unroll
        for (int c = 0; c < 3; ++c) mid[c] = wrap_coord(x[c] + sign * 0.5 * dt * v[c * g.N + i]);
    }
    Stencil st;
    make_stencil(g, mid[0], mid[1], mid[2], i1, i2, i3, st);
    const double* fs[3] = {v, v + g.N, v + 2 * g.N};
    double r[3];
    tile_gather<3>(fs, g, st, act, r);
    if (act) {
#pragma unroll
        for (int c = 0; c < 3; ++c) dep[c * g.N + i] = wrap_coord(x[c] + sign * dt * r[c]);
    }
}

// continuity_factor (transport.cpp:44-55)
__global__ void __launch_bounds__(kTileThreads, 3)
    k_factor(const double* __restrict__ div, const double* __restrict__ dep,
             double* __restrict__ factor, GridDims g, Tile t, double half_dt) {
    int i1, i2, i3;
    long long i;
    const bool act = tile_point(g, t, i1, i2, i3, i);
    double x1 = 0, x2 = 0, x3 = 0, d = 0;
    if (act) {
        load_point(dep, i, g.N, x1, x2, x3);
        d = div[i];
    }
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, i2, i3, st);
    const double* fs[1] = {div};
    double r[1];
    tile_gather<1>(fs, g, st, act, r);
    if (act) factor[i] = exp(half_dt * (d + r[0]));
}

// advect_step / continuity_step (transport.cpp:57-68)
template <bool FACTOR>
__global__ void __launch_bounds__(kTileThreads, 3)
    k_advect(const double* __restrict__ f, const double* __restrict__ dep,
             const double* __restrict__ factor, double* __restrict__ out, GridDims g, Tile t) {
    int i1, i2, i3;
    long long i;
    const bool act = tile_point(g, t, i1, i2, i3, i);
    double x1 = 0, x2 = 0, x3 = 0, fac = 1.0;
    if (act) {
        load_point(dep, i, g.N, x1, x2, x3);
        if (FACTOR) fac = factor[i];
    }
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, i2, i3, st);
    const double* fs[1] = {f};
    double r[1];
    tile_gather<1>(fs, g, st, act, r);
    if (act) out[i] = FACTOR ? r[0] * fac : r[0];
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
__global__ void __launch_bounds__(kTileThreads, 3)
    k_incstate_step(const double* __restrict__ src, const double* __restrict__ dep,
                    const double* __restrict__ gm, const double* __restrict__ vt,
                    double* __restrict__ dst, GridDims g, Tile t, double hdt) {
    int i1, i2, i3;
    long long i;
    const bool act = tile_point(g, t, i1, i2, i3, i);
    double x1 = 0, x2 = 0, x3 = 0, q = 0;
    if (act) {
        load_point(dep, i, g.N, x1, x2, x3);
        q = qdot(gm, vt, i, g.N);  // independent loads issued before the box staging
    }
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, i2, i3, st);
    const double* fs[1] = {src};
    double r[1];
    tile_gather<1>(fs, g, st, act, r);
    if (act) {
        const double m = r[0] + (-hdt) * q;
        dst[i] = (MODE == 0) ? 1.0 * m + (-hdt) * q : -m;
    }
}

// continuity step + optional fused accumulation b_a += (w * lam) * d_a m_j
template <bool ACC>
__global__ void __launch_bounds__(kTileThreads, 3)
    k_adjoint_step(const double* __restrict__ src, const double* __restrict__ dep,
                   const double* __restrict__ factor, double* __restrict__ dst,
                   const double* __restrict__ gm, double w, double* __restrict__ b, GridDims g,
                   Tile t) {
    int i1, i2, i3;
    long long i;
    const bool act = tile_point(g, t, i1, i2, i3, i);
    double x1 = 0, x2 = 0, x3 = 0, fac = 0;
    if (act) {
        load_point(dep, i, g.N, x1, x2, x3);
        fac = factor[i];
    }
    Stencil st;
    make_stencil(g, x1, x2, x3, i1, i2, i3, st);
    const double* fs[1] = {src};
    double r[1];
    tile_gather<1>(fs, g, st, act, r);
    if (act) {
        const double lam = r[0] * fac;
        dst[i] = lam;
        if (ACC) {
            const double wl = w * lam;
#pragma unroll
            for (int a = 0; a < 3; ++a) b[a * g.N + i] = b[a * g.N + i] + wl * gm[a * g.N + i];
        }
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

Tile tile_of(const GridDims& g) {
    Tile t;
    t.t3 = g.n3 < 32 ? g.n3 : 32;
    t.t2 = g.n2 < 4 ? g.n2 : 4;
    const int rest = kTileThreads / (t.t3 * t.t2);
    t.t1 = g.n1 < rest ? g.n1 : rest;
    return t;
}
dim3 tgrid(const GridDims& g, const Tile& t) {
    return dim3(static_cast<unsigned>(g.n3 / t.t3), static_cast<unsigned>(g.n2 / t.t2),
                static_cast<unsigned>(g.n1 / t.t1));
}
unsigned tthreads(const Tile& t) { return static_cast<unsigned>(t.t1 * t.t2 * t.t3); }
constexpr size_t kBoxBytes = sizeof(double) * kBoxCap;

// opt every tile kernel into > 48 KB of shared memory once per (kernel, device)
template <class K>
void set_box_smem(K kern) {
    static std::vector<std::pair<const void*, int>> done;
    int dev = 0;
    VR_CUDA(cudaGetDevice(&dev));
    const void* key = reinterpret_cast<const void*>(kern);
    for (const auto& d : done)
        if (d.first == key && d.second == dev) return;
    VR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kBoxBytes)));
    done.emplace_back(key, dev);
}

#define VR_TILE_LAUNCH(ctx, cat, kern, ...)                                                       \
    do {                                                                                         \
        const GridDims& g_ = (ctx)->g;                                                           \
        const Tile t_ = tile_of(g_);                                                             \
        set_box_smem(kern);                                                                      \
        VR_LAUNCH(ctx, cat, kern<<<tgrid(g_, t_), tthreads(t_), kBoxBytes, (ctx)->stream>>>(__VA_ARGS__)); \
    } while (0)

}  // namespace

void sl_tricubic(vr_ctx* ctx, const double* f, int nfields, const double* pts3, double* out) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    switch (nfields) {
        case 1: VR_TILE_LAUNCH(ctx, "sl_gather", k_tricubic<1>, f, pts3, out, g, t); break;
        case 2: VR_TILE_LAUNCH(ctx, "sl_gather", k_tricubic<2>, f, pts3, out, g, t); break;
        case 3: VR_TILE_LAUNCH(ctx, "sl_gather", k_tricubic<3>, f, pts3, out, g, t); break;
        default: throw_argument("tricubic_interpolate: nfields must be 1, 2 or 3");
    }
}

void sl_trace(vr_ctx* ctx, const double* v3, int nt, int direction, double* dep3) {
    if (nt < 1) throw_argument("trace_characteristics: n_t must be >= 1");
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    const double dt = 1.0 / nt;
    const double sign = direction == VR_TRACE_BACKWARD ? -1.0 : 1.0;
    VR_TILE_LAUNCH(ctx, "sl_trace", k_trace, v3, dep3, g, t, sign, dt);
}

void sl_factor(vr_ctx* ctx, const double* div_v, const double* dep3, double half_dt,
               double* factor) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    VR_TILE_LAUNCH(ctx, "sl_factor", k_factor, div_v, dep3, factor, g, t, half_dt);
}

void sl_advect(vr_ctx* ctx, const double* f, const double* dep3, double* out) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    VR_TILE_LAUNCH(ctx, "sl_state_step", k_advect<false>, f, dep3, nullptr, out, g, t);
}

void sl_continuity(vr_ctx* ctx, const double* f, const double* dep3, const double* factor,
                   double* out) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    VR_TILE_LAUNCH(ctx, "sl_adjoint_step", k_advect<true>, f, dep3, factor, out, g, t);
}

void sl_incstate_first(vr_ctx* ctx, const double* gm0, const double* vt3, double hdt,
                       double* tmp0) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "sl_pointwise", k_incstate_first<<<pgrid(g), kThreads, 0, ctx->stream>>>(gm0, vt3, tmp0, g, hdt, ctx->flag_dev));
}

void sl_incstate_step(vr_ctx* ctx, const double* src, const double* dep3, const double* gm,
                      const double* vt3, double hdt, double* dst, int mode) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    if (mode == 0)
        VR_TILE_LAUNCH(ctx, "sl_incstate_step", k_incstate_step<0>, src, dep3, gm, vt3, dst, g, t, hdt);
    else
        VR_TILE_LAUNCH(ctx, "sl_incstate_step", k_incstate_step<1>, src, dep3, gm, vt3, dst, g, t, hdt);
}

void sl_adjoint_step(vr_ctx* ctx, const double* src, const double* dep3, const double* factor,
                     double* dst, const double* gm, double w, double* b3) {
    const GridDims& g = ctx->g;
    const Tile t = tile_of(g);
    if (b3)
        VR_TILE_LAUNCH(ctx, "sl_adjoint_step_acc", k_adjoint_step<true>, src, dep3, factor, dst, gm, w, b3, g, t);
    else
        VR_TILE_LAUNCH(ctx, "sl_adjoint_step", k_adjoint_step<false>, src, dep3, factor, dst, nullptr, 0.0, nullptr, g, t);
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
