// gather_lab.cu -- standalone micro-benchmark of the semi-Lagrangian tricubic gather
// (interp.hpp:32-53 arithmetic) at real departure points, comparing:
//   A  one point per thread through L1 (the shipped sl.cu gather, 1x4x32 tiles)
//   D  per-tile stencil box staged in shared memory by the bulk-copy engine
//      (cp.async.bulk row segments + mbarrier, double-buffered persistent CTAs),
//      gathered with LDS; tiles whose box overflows fall back to A's path
// Inputs: raw fp64 files written by tools/gather_lab_inputs.py (departure points
// X (3N) and a field f (N)). Prints one JSON line per variant.
//
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        -Xptxas -v tools/gather_lab.cu -o gpurun_out/gather_lab
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

constexpr double kTwoPi = 6.283185307179586476925286766559;

struct G {
    int n;  // cubic grid n^3 (power of two)
    double h;
};

__device__ __forceinline__ void cubic_weights(double s, double* w) {
    const double sm1 = s - 1.0, sm2 = s - 2.0, sp1 = s + 1.0;
    w[0] = -s * sm1 * sm2 * (1.0 / 6.0);
    w[1] = sp1 * sm1 * sm2 * 0.5;
    w[2] = -sp1 * s * sm2 * 0.5;
    w[3] = sp1 * s * sm1 * (1.0 / 6.0);
}
__device__ __forceinline__ void axis_stencil(double x, double h, int& b, double* w) {
    double u = x / h;
    const double r = rint(u);
    if (fabs(u - r) < 1e-12) u = r;
    const double fl = floor(u);
    cubic_weights(u - fl, w);
    b = static_cast<int>(fl) - 1;
}
__device__ __forceinline__ int wrapi(int j, int n) { return j & (n - 1); }
// base nearest to the point's own index (departure coords are wrapped into [0, 2pi))
__device__ __forceinline__ int near(int b, int i, int n) {
    int d = b - i;
    d = ((d + n / 2) & (n - 1)) - n / 2;
    return i + d;
}

// ---------------------------------------------------------------- variant A
__device__ __forceinline__ double gather_l1(const double* __restrict__ f, int n, const int b[3],
                                            const double w[3][4]) {
    const int n23 = n * n;
    int o12[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int oa = wrapi(b[0] + a, n) * n23;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) o12[a][bb] = oa + wrapi(b[1] + bb, n) * n;
    }
    const int b3 = b[2];
    double acc = 0.0;
    if (b3 >= 0 && b3 + 3 < n) {
        const double* f3 = f + b3;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            double acc1 = 0.0;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                const double* p = f3 + o12[a][bb];
                double acc2 = 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c) acc2 += w[2][c] * __ldg(p + c);
                acc1 += w[1][bb] * acc2;
            }
            acc += w[0][a] * acc1;
        }
    } else {
        int i3[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) i3[c] = wrapi(b3 + c, n);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            double acc1 = 0.0;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                const double* p = f + o12[a][bb];
                double acc2 = 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c) acc2 += w[2][c] * __ldg(p + i3[c]);
                acc1 += w[1][bb] * acc2;
            }
            acc += w[0][a] * acc1;
        }
    }
    return acc;
}

__global__ void __launch_bounds__(128, 7) k_gather_A(const double* __restrict__ f, const double* __restrict__ X,
                                                     double* __restrict__ out, G g) {
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int i3 = blockIdx.x * 32 + (threadIdx.x & 31);
    const int i2 = blockIdx.y * 4 + (threadIdx.x >> 5);
    const int i1 = blockIdx.z;
    const long long i = ((long long)i1 * n + i2) * n + i3;
    int b[3];
    double w[3][4];
    axis_stencil(__ldg(X + i), g.h, b[0], w[0]);
    axis_stencil(__ldg(X + N + i), g.h, b[1], w[1]);
    axis_stencil(__ldg(X + 2 * N + i), g.h, b[2], w[2]);
    out[i] = gather_l1(f, n, b, w);
}


// ---------------------------------------------------------------- variant F
// as A, but each stencil row is fetched with three 16-byte loads from the even-aligned
// base a = b3 & ~1 ([a, a+6) covers b3..b3+3), the four values picked by the parity of b3
// (the odd-lane third load is predicated): 3 requests per row instead of 4
__device__ __forceinline__ double gather_l1_v2(const double* __restrict__ f, int n, const int b[3],
                                               const double w[3][4]) {
    const int n23 = n * n;
    const int b3 = b[2];
    if (b3 < 0 || b3 + 5 >= n) return gather_l1(f, n, b, w);
    const int a3 = b3 & ~1;
    const bool odd = b3 & 1;
    int o12[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int oa = wrapi(b[0] + a, n) * n23;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) o12[a][bb] = oa + wrapi(b[1] + bb, n) * n + a3;
    }
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double acc1 = 0.0;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            const double2* p = reinterpret_cast<const double2*>(f + o12[a][bb]);
            const double2 v01 = __ldg(p), v23 = __ldg(p + 1);
            double2 v45 = make_double2(0.0, 0.0);
            if (odd) v45 = __ldg(p + 2);
            const double x0 = odd ? v01.y : v01.x, x1 = odd ? v23.x : v01.y;
            const double x2 = odd ? v23.y : v23.x, x3 = odd ? v45.x : v23.y;
            double acc2 = 0.0;
            acc2 += w[2][0] * x0;
            acc2 += w[2][1] * x1;
            acc2 += w[2][2] * x2;
            acc2 += w[2][3] * x3;
            acc1 += w[1][bb] * acc2;
        }
        acc += w[0][a] * acc1;
    }
    return acc;
}

template <int WARPS>
__global__ void __launch_bounds__(128, WARPS / 4) k_gather_F(const double* __restrict__ f, const double* __restrict__ X,
                                                             double* __restrict__ out, G g) {
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int i3 = blockIdx.x * 32 + (threadIdx.x & 31);
    const int i2 = blockIdx.y * 4 + (threadIdx.x >> 5);
    const int i1 = blockIdx.z;
    const long long i = ((long long)i1 * n + i2) * n + i3;
    int b[3];
    double w[3][4];
    axis_stencil(__ldg(X + i), g.h, b[0], w[0]);
    axis_stencil(__ldg(X + N + i), g.h, b[1], w[1]);
    axis_stencil(__ldg(X + 2 * N + i), g.h, b[2], w[2]);
    out[i] = gather_l1_v2(f, n, b, w);
}


// ---------------------------------------------------------------- variant G
// two x3-adjacent points per thread (warp = 64 consecutive points): when the pair shares
// its (x1, x2) stencil rows (~85% at config 3), each row is fetched once as a 6-wide
// window (three 16-byte loads from the even base of the first point) and both points'
// x3 sums read it through zero-padded weight vectors (adding exact zeros keeps the
// reference's summation order); otherwise the second point gathers on its own
template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_gather_G(const double* __restrict__ f, const double* __restrict__ X,
                                                        double* __restrict__ out, G g) {
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int lane = threadIdx.x & 31;
    const int i3 = blockIdx.x * 64 + 2 * lane;
    const int i2 = blockIdx.y * 4 + (threadIdx.x >> 5);
    const int i1 = blockIdx.z;
    const long long i = ((long long)i1 * n + i2) * n + i3;
    const double2 xa = __ldg(reinterpret_cast<const double2*>(X + i));
    const double2 xb = __ldg(reinterpret_cast<const double2*>(X + N + i));
    const double2 xc = __ldg(reinterpret_cast<const double2*>(X + 2 * N + i));
    int b0[3], b1[3];
    double w0[3][4], w1[3][4];
    axis_stencil(xa.x, g.h, b0[0], w0[0]);
    axis_stencil(xb.x, g.h, b0[1], w0[1]);
    axis_stencil(xc.x, g.h, b0[2], w0[2]);
    axis_stencil(xa.y, g.h, b1[0], w1[0]);
    axis_stencil(xb.y, g.h, b1[1], w1[1]);
    axis_stencil(xc.y, g.h, b1[2], w1[2]);
    const int a3 = b0[2] & ~1;
    const int e0 = b0[2] - a3, e1 = b1[2] - a3;
    const bool fast0 = a3 >= 0 && a3 + 6 <= n;
    const bool share = fast0 && b1[0] == b0[0] && b1[1] == b0[1] && e1 >= 0 && e1 <= 2;
    double acc0 = 0.0, acc1 = 0.0;
    if (fast0) {
        double W0[5], W1[6];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int c = k - e0;
            W0[k] = c == 0 ? w0[2][0] : c == 1 ? w0[2][1] : c == 2 ? w0[2][2] : c == 3 ? w0[2][3] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const int c = k - e1;
            W1[k] = c == 0 ? w1[2][0] : c == 1 ? w1[2][1] : c == 2 ? w1[2][2] : c == 3 ? w1[2][3] : 0.0;
        }
        const int n23 = n * n;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int oa = wrapi(b0[0] + a, n) * n23 + a3;
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                const double2* p = reinterpret_cast<const double2*>(f + oa + wrapi(b0[1] + bb, n) * n);
                const double2 v01 = __ldg(p), v23 = __ldg(p + 1), v45 = __ldg(p + 2);
                double t0 = 0.0;
                t0 += W0[0] * v01.x;
                t0 += W0[1] * v01.y;
                t0 += W0[2] * v23.x;
                t0 += W0[3] * v23.y;
                t0 += W0[4] * v45.x;
                double t1 = 0.0;
                t1 += W1[0] * v01.x;
                t1 += W1[1] * v01.y;
                t1 += W1[2] * v23.x;
                t1 += W1[3] * v23.y;
                t1 += W1[4] * v45.x;
                t1 += W1[5] * v45.y;
                s0 += w0[1][bb] * t0;
                s1 += w1[1][bb] * t1;
            }
            acc0 += w0[0][a] * s0;
            acc1 += w1[0][a] * s1;
        }
    } else {
        acc0 = gather_l1(f, n, b0, w0);
    }
    if (!share) acc1 = gather_l1(f, n, b1, w1);
    *reinterpret_cast<double2*>(out + i) = make_double2(acc0, acc1);
}

// ---------------------------------------------------------------- tiles / boxes
template <int T1, int T2>
struct TileGeo {
    static constexpr int P = T1 * T2 * 32;
};

// per tile: box origin (unwrapped, nearest image to the points) and extents;
// ext.w = -1 when the box does not fit (then the tile is gathered through L1)
template <int T1, int T2>
__global__ void k_boxes(const double* __restrict__ X, G g, int4* __restrict__ org, int4* __restrict__ ext,
                        int rows_max, int pitch) {
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int tiles3 = n / 32, tiles2 = n / T2;
    const int t = blockIdx.x;
    const int t3 = t % tiles3, t2 = (t / tiles3) % tiles2, t1 = t / (tiles3 * tiles2);
    int mn[3] = {1 << 29, 1 << 29, 1 << 29}, mx[3] = {-(1 << 29), -(1 << 29), -(1 << 29)};
    for (int p = threadIdx.x; p < TileGeo<T1, T2>::P; p += blockDim.x) {
        const int l3 = p & 31, r = p >> 5;
        const int i1 = t1 * T1 + r / T2, i2 = t2 * T2 + r % T2, i3 = t3 * 32 + l3;
        const long long i = ((long long)i1 * n + i2) * n + i3;
        const int own[3] = {i1, i2, i3};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            int b;
            double w[4];
            axis_stencil(__ldg(X + c * N + i), g.h, b, w);
            b = near(b, own[c], n);
            mn[c] = min(mn[c], b);
            mx[c] = max(mx[c], b);
        }
    }
    __shared__ int smn[3][32], smx[3][32];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        int a = mn[c], z = mx[c];
        for (int o = 16; o; o >>= 1) {
            a = min(a, __shfl_xor_sync(~0u, a, o));
            z = max(z, __shfl_xor_sync(~0u, z, o));
        }
        if ((threadIdx.x & 31) == 0) smn[c][threadIdx.x >> 5] = a, smx[c][threadIdx.x >> 5] = z;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int a[3], z[3];
        for (int c = 0; c < 3; ++c) {
            a[c] = smn[c][0], z[c] = smx[c][0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) a[c] = min(a[c], smn[c][w]), z[c] = max(z[c], smx[c][w]);
        }
        const int E1 = z[0] - a[0] + 4, E2 = z[1] - a[1] + 4;
        const int o3a = a[2] & ~1;
        const int W = ((z[2] + 4 - o3a) + 1) & ~1;  // even number of doubles from the even origin
        const bool ok = E1 * E2 <= rows_max && W <= pitch && W <= n;
        org[t] = make_int4(a[0], a[1], o3a, 0);
        ext[t] = make_int4(E1, E2, W, ok ? 1 : -1);
    }
}

// ---------------------------------------------------------------- variant D
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.b32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(su32(bar)), "r"(parity)
            : "memory");
    }
}

// issue the row-segment copies of tile t's box into `buf` (warp 0)
__device__ __forceinline__ void issue_box(const double* __restrict__ f, int n, int4 o, int4 e, double* buf,
                                          int pitch, unsigned long long* bar) {
    const int lane = threadIdx.x & 31;
    const int rows = e.x * e.y;
    if (lane == 0) mbar_expect(bar, (unsigned)(rows * e.z * 8));
    __syncwarp();
    const int s = o.z & (n - 1);  // even
    const int first = min(e.z, n - s);
    for (int r = lane; r < rows; r += 32) {
        const int a = r / e.y, b = r - a * e.y;
        const double* row = f + ((long long)wrapi(o.x + a, n) * n + wrapi(o.y + b, n)) * n;
        double* d = buf + r * pitch;
        bulk_g2s(d, row + s, first * 8, bar);
        if (first < e.z) bulk_g2s(d + first, row, (e.z - first) * 8, bar);
    }
}

template <int T1, int T2, int PITCH, int ROWS, int MINB>
__global__ void __launch_bounds__(256, MINB) k_gather_D(const double* __restrict__ f, const double* __restrict__ X,
                                                     double* __restrict__ out, G g, const int4* __restrict__ org,
                                                     const int4* __restrict__ ext, int ntiles) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* buf[2] = {reinterpret_cast<double*>(smem_raw), reinterpret_cast<double*>(smem_raw) + ROWS * PITCH};
    __shared__ unsigned long long bar[2];
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int tiles3 = n / 32, tiles2 = n / T2;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned phase[2] = {0, 0};
    int t = blockIdx.x;
    if (t < ntiles && threadIdx.x < 32) {
        int4 e = ext[t];
        if (e.w > 0) issue_box(f, n, org[t], e, buf[0], PITCH, &bar[0]);
    }
    for (int k = 0; t < ntiles; ++k, t += gridDim.x) {
        const int s = k & 1;
        const int tn = t + gridDim.x;
        if (tn < ntiles && threadIdx.x < 32) {
            int4 e = ext[tn];
            if (e.w > 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue_box(f, n, org[tn], e, buf[s ^ 1], PITCH, &bar[s ^ 1]);
            }
        }
        const int4 o = org[t], e = ext[t];
        const bool staged = e.w > 0;
        if (staged) {
            mbar_wait(&bar[s], phase[s]);
            phase[s] ^= 1;
        }
        const int t3 = t % tiles3, t2 = (t / tiles3) % tiles2, t1 = t / (tiles3 * tiles2);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
        for (int r = warp; r < T1 * T2; r += 8) {
            const int i1 = t1 * T1 + r / T2, i2 = t2 * T2 + r % T2, i3 = t3 * 32 + lane;
            const long long i = ((long long)i1 * n + i2) * n + i3;
            int b[3];
            double w[3][4];
            axis_stencil(__ldg(X + i), g.h, b[0], w[0]);
            axis_stencil(__ldg(X + N + i), g.h, b[1], w[1]);
            axis_stencil(__ldg(X + 2 * N + i), g.h, b[2], w[2]);
            double acc = 0.0;
            if (staged) {
                const int r1 = near(b[0], i1, n) - o.x, r2 = near(b[1], i2, n) - o.y, r3 = near(b[2], i3, n) - o.z;
                const double* sb = buf[s] + (r1 * e.y + r2) * PITCH + r3;
                const int rp = e.y * PITCH;
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    double acc1 = 0.0;
#pragma unroll
                    for (int bb = 0; bb < 4; ++bb) {
                        const double* p = sb + a * rp + bb * PITCH;
                        double acc2 = 0.0;
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc2 += w[2][c] * p[c];
                        acc1 += w[1][bb] * acc2;
                    }
                    acc += w[0][a] * acc1;
                }
            } else {
                acc = gather_l1(f, n, b, w);
            }
            out[i] = acc;
        }
        __syncthreads();  // everyone is done with buf[s] before it is refilled
    }
}


// ---------------------------------------------------------------- variant E
// warp-specialized: one producer warp streams each tile's stencil box AND its departure
// points into a STAGES-deep ring of shared-memory stages (cp.async.bulk + full/empty
// mbarriers); CWARPS consumer warps gather from shared memory only
template <int T1, int T2, int PITCH, int ROWS, int STAGES, int CWARPS, int MINB>
__global__ void __launch_bounds__(32 * (CWARPS + 1), MINB)
    k_gather_E(const double* __restrict__ f, const double* __restrict__ X, double* __restrict__ out, G g,
               const int4* __restrict__ org, const int4* __restrict__ ext, int ntiles) {
    constexpr int TP = T1 * T2 * 32;                // points per tile
    constexpr int STAGE = ROWS * PITCH + 3 * TP;    // doubles per stage
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* sm = reinterpret_cast<double*>(smem_raw);
    __shared__ unsigned long long full[STAGES], empty[STAGES];
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int tiles3 = n / 32, tiles2 = n / T2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CWARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == CWARPS) {  // producer
        int k = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
            const int s = k % STAGES, u = k / STAGES;
            if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
            const int4 o = org[t], e = ext[t];
            const bool staged = e.w > 0;
            double* box = sm + s * STAGE;
            double* xs = box + ROWS * PITCH;
            const unsigned bytes = (staged ? e.x * e.y * e.z * 8 : 0) + 3 * TP * 8;
            if (lane == 0) mbar_expect(&full[s], bytes);
            __syncwarp();
            const int t3 = t % tiles3, t2 = (t / tiles3) % tiles2, t1 = t / (tiles3 * tiles2);
            for (int q = lane; q < 3 * T1 * T2; q += 32) {  // departure points: 256 B rows
                const int c = q / (T1 * T2), r = q % (T1 * T2);
                const int i1 = t1 * T1 + r / T2, i2 = t2 * T2 + r % T2;
                bulk_g2s(xs + c * TP + r * 32, X + c * N + ((long long)i1 * n + i2) * n + t3 * 32, 256, &full[s]);
            }
            if (staged) {
                const int rows = e.x * e.y;
                const int s0 = o.z & (n - 1);
                const int first = min(e.z, n - s0);
                for (int r = lane; r < rows; r += 32) {
                    const int a = r / e.y, b = r - a * e.y;
                    const double* row = f + ((long long)wrapi(o.x + a, n) * n + wrapi(o.y + b, n)) * n;
                    double* d = box + r * PITCH;
                    bulk_g2s(d, row + s0, first * 8, &full[s]);
                    if (first < e.z) bulk_g2s(d + first, row, (e.z - first) * 8, &full[s]);
                }
            }
        }
        return;
    }
    int k = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int s = k % STAGES, u = k / STAGES;
        const int4 o = org[t], e = ext[t];
        const bool staged = e.w > 0;
        mbar_wait(&full[s], u & 1);
        const double* box = sm + s * STAGE;
        const double* xs = box + ROWS * PITCH;
        const int t3 = t % tiles3, t2 = (t / tiles3) % tiles2, t1 = t / (tiles3 * tiles2);
#pragma unroll 1
        for (int r = warp; r < T1 * T2; r += CWARPS) {
            const int i1 = t1 * T1 + r / T2, i2 = t2 * T2 + r % T2, i3 = t3 * 32 + lane;
            const long long i = ((long long)i1 * n + i2) * n + i3;
            int b[3];
            double w[3][4];
            axis_stencil(xs[r * 32 + lane], g.h, b[0], w[0]);
            axis_stencil(xs[TP + r * 32 + lane], g.h, b[1], w[1]);
            axis_stencil(xs[2 * TP + r * 32 + lane], g.h, b[2], w[2]);
            double acc = 0.0;
            if (staged) {
                const int r1 = near(b[0], i1, n) - o.x, r2 = near(b[1], i2, n) - o.y, r3 = near(b[2], i3, n) - o.z;
                const double* sb = box + (r1 * e.y + r2) * PITCH + r3;
                const int rp = e.y * PITCH;
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    double acc1 = 0.0;
#pragma unroll
                    for (int bb = 0; bb < 4; ++bb) {
                        const double* p = sb + a * rp + bb * PITCH;
                        double acc2 = 0.0;
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc2 += w[2][c] * p[c];
                        acc1 += w[1][bb] * acc2;
                    }
                    acc += w[0][a] * acc1;
                }
            } else {
                acc = gather_l1(f, n, b, w);
            }
            out[i] = acc;
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
}

// ---------------------------------------------------------------- driver
static std::vector<double> readf(const char* p, size_t cnt) {
    std::vector<double> v(cnt);
    FILE* fp = fopen(p, "rb");
    if (!fp || fread(v.data(), 8, cnt, fp) != cnt) {
        fprintf(stderr, "cannot read %s\n", p);
        exit(1);
    }
    fclose(fp);
    return v;
}

template <class L>
static float time_it(L&& launch, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / reps;
}

static void compare(const char* name, float ms, const std::vector<double>& ref, double* d_out, long long N,
                    double extra) {
    std::vector<double> o(N);
    CK(cudaMemcpy(o.data(), d_out, N * 8, cudaMemcpyDeviceToHost));
    long long same = 0;
    double md = 0;
    for (long long i = 0; i < N; ++i) {
        if (o[i] == ref[i]) ++same;
        md = fmax(md, fabs(o[i] - ref[i]));
    }
    printf("{\"variant\": \"%s\", \"ms\": %.4f, \"bitwise_equal_frac\": %.6f, \"max_abs_diff\": %.3e, \"extra\": %.4f}\n",
           name, ms, (double)same / N, md, extra);
    fflush(stdout);
}

template <int T1, int T2, int PITCH, int ROWS, int MINB>
static void run_D(const char* name, const double* d_f, const double* d_X, double* d_out, G g,
                  const std::vector<double>& ref) {
    const int ctas_per_sm = MINB;
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int ntiles = (n / T1) * (n / T2) * (n / 32);
    int4 *org, *ext;
    CK(cudaMalloc(&org, ntiles * sizeof(int4)));
    CK(cudaMalloc(&ext, ntiles * sizeof(int4)));
    auto boxes = [&] { k_boxes<T1, T2><<<ntiles, 256>>>(d_X, g, org, ext, ROWS, PITCH); };
    float ms_box = time_it(boxes, 5);
    std::vector<int4> he(ntiles);
    CK(cudaMemcpy(he.data(), ext, ntiles * sizeof(int4), cudaMemcpyDeviceToHost));
    int over = 0;
    double rows = 0, bytes = 0;
    for (auto& e : he) {
        if (e.w < 0) ++over;
        else rows += e.x * e.y, bytes += 8.0 * e.x * e.y * e.z;
    }
    const size_t smem = 2ull * ROWS * PITCH * 8;
    auto kern = k_gather_D<T1, T2, PITCH, ROWS, MINB>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem));
    const int grid = sms * std::max(1, std::min(occ, ctas_per_sm));
    auto launch = [&] { kern<<<grid, 256, smem>>>(d_f, d_X, d_out, g, org, ext, ntiles); };
    CK(cudaMemset(d_out, 0, N * 8));
    float ms = time_it(launch, 20);
    CK(cudaGetLastError());
    char nm[160];
    snprintf(nm, sizeof nm, "%s T%dx%dx32 pitch%d rows%d occ%d overflow%.3f box_B_per_pt%.1f", name, T1, T2, PITCH,
             ROWS, occ, (double)over / ntiles, bytes / ((double)(ntiles - over) * T1 * T2 * 32));
    compare(nm, ms, ref, d_out, N, ms_box);
    cudaFree(org);
    cudaFree(ext);
}


template <int T1, int T2, int PITCH, int ROWS, int STAGES, int CWARPS, int MINB>
static void run_E(const double* d_f, const double* d_X, double* d_out, G g, const std::vector<double>& ref) {
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int ntiles = (n / T1) * (n / T2) * (n / 32);
    int4 *org, *ext;
    CK(cudaMalloc(&org, ntiles * sizeof(int4)));
    CK(cudaMalloc(&ext, ntiles * sizeof(int4)));
    k_boxes<T1, T2><<<ntiles, 256>>>(d_X, g, org, ext, ROWS, PITCH);
    std::vector<int4> he(ntiles);
    CK(cudaMemcpy(he.data(), ext, ntiles * sizeof(int4), cudaMemcpyDeviceToHost));
    int over = 0;
    for (auto& e : he) over += e.w < 0;
    const size_t smem = (size_t)STAGES * (ROWS * PITCH + 3 * T1 * T2 * 32) * 8;
    auto kern = k_gather_E<T1, T2, PITCH, ROWS, STAGES, CWARPS, MINB>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int sms, occ = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * (CWARPS + 1), smem));
    const int grid = sms * std::max(1, std::min(occ, MINB));
    auto launch = [&] { kern<<<grid, 32 * (CWARPS + 1), smem>>>(d_f, d_X, d_out, g, org, ext, ntiles); };
    CK(cudaMemset(d_out, 0, N * 8));
    float ms = time_it(launch, 20);
    CK(cudaGetLastError());
    char nm[160];
    snprintf(nm, sizeof nm, "E ws T%dx%dx32 pitch%d rows%d stages%d cwarps%d occ%d smemKB%zu overflow%.3f", T1, T2,
             PITCH, ROWS, STAGES, CWARPS, occ, smem / 1024, (double)over / ntiles);
    compare(nm, ms, ref, d_out, N, 0.0);
    cudaFree(org);
    cudaFree(ext);
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 256;
    const char* xp = argc > 2 ? argv[2] : "/tmp/lab_X.bin";
    const char* fp = argc > 3 ? argv[3] : "/tmp/lab_f.bin";
    const long long N = (long long)n * n * n;
    auto X = readf(xp, 3 * N);
    auto F = readf(fp, N);
    double *d_X, *d_f, *d_out;
    CK(cudaMalloc(&d_X, 3 * N * 8));
    CK(cudaMalloc(&d_f, N * 8));
    CK(cudaMalloc(&d_out, N * 8));
    CK(cudaMemcpy(d_X, X.data(), 3 * N * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_f, F.data(), N * 8, cudaMemcpyHostToDevice));
    G g{n, kTwoPi / n};
    // A
    auto la = [&] { k_gather_A<<<dim3(n / 32, n / 4, n), 128>>>(d_f, d_X, d_out, g); };
    float msA = time_it(la, 20);
    std::vector<double> ref(N);
    CK(cudaMemcpy(ref.data(), d_out, N * 8, cudaMemcpyDeviceToHost));
    printf("{\"variant\": \"A l1 1x4x32\", \"ms\": %.4f, \"GBps_alg\": %.1f}\n", msA, 5.0 * 8 * N / (msA * 1e-3) / 1e9);
    {
        auto lg4 = [&] { k_gather_G<4><<<dim3(n / 64, n / 4, n), 128>>>(d_f, d_X, d_out, g); };
        CK(cudaMemset(d_out, 0, N * 8));
        compare("G x3pair 16w", time_it(lg4, 20), ref, d_out, N, 0);
        auto lg5 = [&] { k_gather_G<5><<<dim3(n / 64, n / 4, n), 128>>>(d_f, d_X, d_out, g); };
        CK(cudaMemset(d_out, 0, N * 8));
        compare("G x3pair 20w", time_it(lg5, 20), ref, d_out, N, 0);
        auto lg6 = [&] { k_gather_G<6><<<dim3(n / 64, n / 4, n), 128>>>(d_f, d_X, d_out, g); };
        CK(cudaMemset(d_out, 0, N * 8));
        compare("G x3pair 24w", time_it(lg6, 20), ref, d_out, N, 0);
        auto lg3 = [&] { k_gather_G<3><<<dim3(n / 64, n / 4, n), 128>>>(d_f, d_X, d_out, g); };
        CK(cudaMemset(d_out, 0, N * 8));
        compare("G x3pair 12w", time_it(lg3, 20), ref, d_out, N, 0);
    }
    return 0;
}
