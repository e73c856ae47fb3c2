// gather_lab2.cu -- round-2b gather lab: several lanes per point.
//
// Motivation (B300_MICROARCH "L1tex wavefront queue"): an LDG request costs about
// 1 + 2.07 (lines - 1) L1 data-pipe cycles, so a warp-wide fp64 load of 32 adjacent points
// (35 doubles, 3 lines) costs ~5.2 cycles while a load that stays inside 1-2 lines costs
// 1-3. Variant A (shipped in round 2a): 64 requests x 3.1 lines per 32 points. Here the
// stencil's x3 columns are split over L lanes of the same point, so a request covers
// 32 / L adjacent points and spans fewer lines:
//   H   2 lanes per point: lane h reads columns {h, h+2} (or {2h, 2h+1}), 32 requests of
//       ~2.1 lines per 16 points
//   H4  4 lanes per point: lane c reads column c, 16 requests of ~1.6 lines per 8 points
// Partial sums are combined with xor-shuffles. Same inputs as tools/gather_lab.cu.
//
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        -Xptxas -v tools/gather_lab2.cu -o /tmp/gather_lab2
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
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
    int n;
    double h;
    int skip_fallback = 0;
};

__device__ __forceinline__ void cubic_weights(double s, double* w) {
    const double sm1 = s - 1.0, sm2 = s - 2.0, sp1 = s + 1.0;
    w[0] = -s * sm1 * sm2 * (1.0 / 6.0);
    w[1] = sp1 * sm1 * sm2 * 0.5;
    w[2] = -sp1 * s * sm2 * 0.5;
    w[3] = sp1 * s * sm1 * (1.0 / 6.0);
}
__device__ __forceinline__ double axis_frac(double x, double h, int& b) {
    double u = x / h;
    const double r = rint(u);
    if (fabs(u - r) < 1e-12) u = r;
    const double fl = floor(u);
    b = static_cast<int>(fl) - 1;
    return u - fl;
}
__device__ __forceinline__ void axis_stencil(double x, double h, int& b, double* w) {
    cubic_weights(axis_frac(x, h, b), w);
}
__device__ __forceinline__ int wrapi(int j, int n) { return j & (n - 1); }

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

// ---------------------------------------------------------------- variant H (2 lanes / point)
// CTA tile: T2 x2-rows x T3 x3-points, 2*T3 threads per row. lane = 2 p + h (LM = 0) or
// p + 16 h (LM = 1). SPLIT 0: lane h reads columns {h, h + 2}; SPLIT 1: {2h, 2h + 1}.
template <int T2, int T3, int MINB, int SPLIT, int LM>
__global__ void __launch_bounds__(2 * T2 * T3, MINB)
    k_gather_H(const double* __restrict__ f, const double* __restrict__ X, double* __restrict__ out, G g) {
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    const int h = LM == 0 ? (lane & 1) : (lane >> 4);
    const int pl = LM == 0 ? (lane >> 1) : (lane & 15);
    constexpr int WPR = T3 / 16;  // warps per x2 row
    const int i3 = blockIdx.x * T3 + (wid % WPR) * 16 + pl;
    const int i2 = blockIdx.y * T2 + wid / WPR;
    const int i1 = blockIdx.z;
    const long long i = ((long long)i1 * n + i2) * n + i3;
    int b[3];
    double w[3][4];
    axis_stencil(__ldg(X + i), g.h, b[0], w[0]);
    axis_stencil(__ldg(X + N + i), g.h, b[1], w[1]);
    axis_stencil(__ldg(X + 2 * N + i), g.h, b[2], w[2]);
    const int c0 = SPLIT == 0 ? h : 2 * h, c1 = SPLIT == 0 ? h + 2 : 2 * h + 1;
    const double wc0 = h ? (SPLIT == 0 ? w[2][1] : w[2][2]) : w[2][0];
    const double wc1 = h ? w[2][3] : (SPLIT == 0 ? w[2][2] : w[2][1]);
    const int n23 = n * n;
    const int b3 = b[2];
    int k0, k1;
    if (b3 >= 0 && b3 + 3 < n) {
        k0 = b3 + c0;
        k1 = b3 + c1;
    } else {
        k0 = wrapi(b3 + c0, n);
        k1 = wrapi(b3 + c1, n);
    }
    const double* f0 = f + k0;
    const int d1 = k1 - k0;
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int oa = wrapi(b[0] + a, n) * n23;
        double acc1 = 0.0;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            const double* p = f0 + (oa + wrapi(b[1] + bb, n) * n);
            double acc2 = wc0 * __ldg(p);
            acc2 += wc1 * __ldg(p + d1);
            acc1 += w[1][bb] * acc2;
        }
        acc += w[0][a] * acc1;
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, LM == 0 ? 1 : 16);
    if (h == 0) out[i] = acc;
}

// ---------------------------------------------------------------- variant H4 (4 lanes / point)
// lane = 4 p + c; a warp covers 8 adjacent x3 points; each lane reads column c of the 16 rows.
template <int T2, int T3, int MINB>
__global__ void __launch_bounds__(4 * T2 * T3, MINB)
    k_gather_H4(const double* __restrict__ f, const double* __restrict__ X, double* __restrict__ out, G g) {
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    const int c = lane & 3, pl = lane >> 2;
    constexpr int WPR = T3 / 8;
    const int i3 = blockIdx.x * T3 + (wid % WPR) * 8 + pl;
    const int i2 = blockIdx.y * T2 + wid / WPR;
    const int i1 = blockIdx.z;
    const long long i = ((long long)i1 * n + i2) * n + i3;
    int b[3];
    double w[3][4];
    axis_stencil(__ldg(X + i), g.h, b[0], w[0]);
    axis_stencil(__ldg(X + N + i), g.h, b[1], w[1]);
    // own column weight: Lagrange basis c on nodes -1, 0, 1, 2
    const double s = axis_frac(__ldg(X + 2 * N + i), g.h, b[2]);
    double w3[4];
    cubic_weights(s, w3);
    const double wc = c == 0 ? w3[0] : c == 1 ? w3[1] : c == 2 ? w3[2] : w3[3];
    const int n23 = n * n;
    const double* f0 = f + wrapi(b[2] + c, n);
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int oa = wrapi(b[0] + a, n) * n23;
        double acc1 = 0.0;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) acc1 += w[1][bb] * __ldg(f0 + (oa + wrapi(b[1] + bb, n) * n));
        acc += w[0][a] * acc1;
    }
    acc *= wc;
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (c == 0) out[i] = acc;
}


// ---------------------------------------------------------------- variant T (TMA stencil box)
// Persistent CTAs walk T1 x T2 x 32 tiles. Per tile ONE cp.async.bulk.tensor 3D box
// (BX1 x BX2 x BW doubles at the tile's stencil origin, two stages, mbarrier) stages the
// union of the tile's stencils in shared memory; the points gather with LDS.64. Tiles whose
// stencils leave the box or cross the periodic boundary take A's L1 path.
__device__ __forceinline__ int near_img(int b, int i, int n) {
    int d = b - i;
    d = ((d + n / 2) & (n - 1)) - n / 2;
    return i + d;
}
template <int T1, int T2>
__global__ void k_tile_boxes(const double* __restrict__ X, G g, int4* __restrict__ org, int bx1, int bx2, int bw) {
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int tiles3 = n / 32, tiles2 = n / T2;
    const int t = blockIdx.x;
    const int t3 = t % tiles3, t2 = (t / tiles3) % tiles2, t1 = t / (tiles3 * tiles2);
    int mn[3] = {1 << 29, 1 << 29, 1 << 29}, mx[3] = {-(1 << 29), -(1 << 29), -(1 << 29)};
    for (int p = threadIdx.x; p < T1 * T2 * 32; p += blockDim.x) {
        const int l3 = p & 31, r = p >> 5;
        const int i1 = t1 * T1 + r / T2, i2 = t2 * T2 + r % T2, i3 = t3 * 32 + l3;
        const long long i = ((long long)i1 * n + i2) * n + i3;
        const int own[3] = {i1, i2, i3};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            int b;
            axis_frac(__ldg(X + c * N + i), g.h, b);
            b = near_img(b, own[c], n);
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
        const int o3 = a[2] & ~1;  // 16-byte aligned box rows
        const bool fits = z[0] + 4 - a[0] <= bx1 && z[1] + 4 - a[1] <= bx2 && z[2] + 4 - o3 <= bw;
        const bool inside = a[0] >= 0 && z[0] + 4 <= n && a[1] >= 0 && z[1] + 4 <= n && o3 >= 0 && z[2] + 4 <= n;
        org[t] = make_int4(a[0], a[1], o3, fits && inside ? 1 : 0);
    }
}
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait_t(unsigned long long* bar, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.b32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(su32(bar)), "r"(parity)
            : "memory");
    }
}
template <int T1, int T2, int BX1, int BX2, int BW, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
    k_gather_T(const __grid_constant__ CUtensorMap tmap, const double* __restrict__ f, const double* __restrict__ X,
               double* __restrict__ out, G g, const int4* __restrict__ org, int ntiles) {
    constexpr int STAGE = BX1 * BX2 * BW;  // doubles
    extern __shared__ __align__(128) double sm[];
    __shared__ unsigned long long bar[2];
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int tiles3 = n / 32, tiles2 = n / T2;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[s])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int t, int s) {
        const int4 o = org[t];
        if (!o.w) return;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])),
                     "r"((unsigned)(STAGE * 8))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            ::"r"(su32(sm + s * STAGE)), "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(o.z), "r"(o.y),
            "r"(o.x), "r"(su32(&bar[s]))
            : "memory");
    };
    int t = blockIdx.x;
    if (threadIdx.x == 0 && t < ntiles) issue(t, 0);
    unsigned ph[2] = {0, 0};
    for (int k = 0; t < ntiles; ++k, t += gridDim.x) {
        const int s = k & 1;
        const int tn = t + gridDim.x;
        if (threadIdx.x == 0 && tn < ntiles) issue(tn, s ^ 1);
        const int4 o = org[t];
        if (o.w) {
            mbar_wait_t(&bar[s], ph[s]);
            ph[s] ^= 1;
        }
        const double* box = sm + s * STAGE;
        const int t3 = t % tiles3, t2 = (t / tiles3) % tiles2, t1 = t / (tiles3 * tiles2);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
        for (int r = warp; r < T1 * T2; r += THREADS / 32) {
            const int i1 = t1 * T1 + r / T2, i2 = t2 * T2 + r % T2, i3 = t3 * 32 + lane;
            const long long i = ((long long)i1 * n + i2) * n + i3;
            int b[3];
            double w[3][4];
            axis_stencil(__ldg(X + i), g.h, b[0], w[0]);
            axis_stencil(__ldg(X + N + i), g.h, b[1], w[1]);
            axis_stencil(__ldg(X + 2 * N + i), g.h, b[2], w[2]);
            double acc = 0.0;
            if (o.w) {
                const int r1 = near_img(b[0], i1, n) - o.x, r2 = near_img(b[1], i2, n) - o.y,
                          r3 = near_img(b[2], i3, n) - o.z;
                const double* sb = box + (r1 * BX2 + r2) * BW + r3;
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    double acc1 = 0.0;
#pragma unroll
                    for (int bb = 0; bb < 4; ++bb) {
                        const double* p = sb + (a * BX2 + bb) * BW;
                        double acc2 = 0.0;
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc2 += w[2][c] * p[c];
                        acc1 += w[1][bb] * acc2;
                    }
                    acc += w[0][a] * acc1;
                }
            } else {
                if (g.skip_fallback) continue;  // lab: time the staged tiles alone
                acc = gather_l1(f, n, b, w);
            }
            out[i] = acc;
        }
        __syncthreads();  // everyone is done with this stage before the copy engine refills it
    }
}

using TmapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmapEncodeFn tmap_encoder() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    return reinterpret_cast<TmapEncodeFn>(p);
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
    CK(cudaGetLastError());
    return ms / reps;
}

static void compare(const char* name, float ms, const std::vector<double>& ref, double* d_out, long long N) {
    std::vector<double> o(N);
    CK(cudaMemcpy(o.data(), d_out, N * 8, cudaMemcpyDeviceToHost));
    long long same = 0;
    double md = 0;
    for (long long i = 0; i < N; ++i) {
        if (o[i] == ref[i]) ++same;
        md = fmax(md, fabs(o[i] - ref[i]));
    }
    printf("{\"variant\": \"%s\", \"ms\": %.4f, \"bitwise_equal_frac\": %.6f, \"max_abs_diff\": %.3e}\n", name, ms,
           (double)same / N, md);
    fflush(stdout);
}

template <int T2, int T3, int MINB, int SPLIT, int LM>
static void run_H(const double* d_f, const double* d_X, double* d_out, G g, const std::vector<double>& ref) {
    const int n = g.n;
    const long long N = (long long)n * n * n;
    auto l = [&] {
        k_gather_H<T2, T3, MINB, SPLIT, LM><<<dim3(n / T3, n / T2, n), 2 * T2 * T3>>>(d_f, d_X, d_out, g);
    };
    CK(cudaMemset(d_out, 0, N * 8));
    char nm[128];
    snprintf(nm, sizeof nm, "H 2lanes T1x%dx%d minb%d split%d lm%d", T2, T3, MINB, SPLIT, LM);
    compare(nm, time_it(l, 20), ref, d_out, N);
}
template <int T2, int T3, int MINB>
static void run_H4(const double* d_f, const double* d_X, double* d_out, G g, const std::vector<double>& ref) {
    const int n = g.n;
    const long long N = (long long)n * n * n;
    auto l = [&] { k_gather_H4<T2, T3, MINB><<<dim3(n / T3, n / T2, n), 4 * T2 * T3>>>(d_f, d_X, d_out, g); };
    CK(cudaMemset(d_out, 0, N * 8));
    char nm[128];
    snprintf(nm, sizeof nm, "H4 4lanes T1x%dx%d minb%d", T2, T3, MINB);
    compare(nm, time_it(l, 20), ref, d_out, N);
}


template <int T1, int T2, int BX1, int BX2, int BW, int THREADS, int MINB>
static void run_T(const double* d_f, const double* d_X, double* d_out, G g, const std::vector<double>& ref) {
    const int n = g.n;
    const long long N = (long long)n * n * n;
    const int ntiles = (n / T1) * (n / T2) * (n / 32);
    int4* org;
    CK(cudaMalloc(&org, ntiles * sizeof(int4)));
    auto boxes = [&] { k_tile_boxes<T1, T2><<<ntiles, 256>>>(d_X, g, org, BX1, BX2, BW); };
    float ms_box = time_it(boxes, 5);
    std::vector<int4> ho(ntiles);
    CK(cudaMemcpy(ho.data(), org, ntiles * sizeof(int4), cudaMemcpyDeviceToHost));
    int staged = 0;
    for (auto& o : ho) staged += o.w;
    CUtensorMap tm;
    const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)n};
    const cuuint64_t strides[2] = {(cuuint64_t)n * 8, (cuuint64_t)n * n * 8};
    const cuuint32_t box[3] = {BW, BX2, BX1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = tmap_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)d_f, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        fprintf(stderr, "tensor map encode failed %d\n", (int)r);
        exit(1);
    }
    const size_t smem = 2ull * BX1 * BX2 * BW * 8;
    auto kern = k_gather_T<T1, T2, BX1, BX2, BW, THREADS, MINB>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int sms, occ = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, smem));
    const int grid = sms * std::max(1, std::min(occ, MINB));
    auto launch = [&] { kern<<<grid, THREADS, smem>>>(tm, d_f, d_X, d_out, g, org, ntiles); };
    CK(cudaMemset(d_out, 0, N * 8));
    char nm[200];
    float ms = time_it(launch, 20);
    snprintf(nm, sizeof nm, "T tma-box T%dx%dx32 box%dx%dx%d thr%d occ%d smemKB%zu staged%.3f boxes_ms%.3f", T1, T2,
             BX1, BX2, BW, THREADS, occ, smem / 1024, (double)staged / ntiles, ms_box);
    compare(nm, ms, ref, d_out, N);
    G g2 = g;
    g2.skip_fallback = 1;
    auto launch2 = [&] { kern<<<grid, THREADS, smem>>>(tm, d_f, d_X, d_out, g2, org, ntiles); };
    float ms2 = time_it(launch2, 20);
    printf("{\"variant\": \"%s staged tiles only\", \"ms\": %.4f, \"ms_per_full_grid_equiv\": %.4f}\n", nm, ms2,
           ms2 / ((double)staged / ntiles));
    cudaFree(org);
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
    if (argc > 4) {  // ncu mode: one launch of each kernel of interest
        k_gather_A<<<dim3(n / 32, n / 4, n), 128>>>(d_f, d_X, d_out, g);
        k_gather_H<4, 16, 8, 0, 0><<<dim3(n / 16, n / 4, n), 128>>>(d_f, d_X, d_out, g);
        k_gather_H4<4, 16, 4><<<dim3(n / 16, n / 4, n), 256>>>(d_f, d_X, d_out, g);
        CK(cudaDeviceSynchronize());
        return 0;
    }
    auto la = [&] { k_gather_A<<<dim3(n / 32, n / 4, n), 128>>>(d_f, d_X, d_out, g); };
    float msA = time_it(la, 20);
    std::vector<double> ref(N);
    CK(cudaMemcpy(ref.data(), d_out, N * 8, cudaMemcpyDeviceToHost));
    printf("{\"variant\": \"A l1 1x4x32\", \"ms\": %.4f}\n", msA);
    if (getenv("LAB_T")) {
        run_T<2, 4, 8, 12, 48, 256, 3>(d_f, d_X, d_out, g, ref);
        run_T<1, 4, 8, 12, 48, 128, 3>(d_f, d_X, d_out, g, ref);
        run_T<1, 4, 6, 10, 48, 128, 4>(d_f, d_X, d_out, g, ref);
        run_T<2, 2, 8, 8, 48, 128, 4>(d_f, d_X, d_out, g, ref);
        run_T<2, 4, 8, 10, 48, 256, 3>(d_f, d_X, d_out, g, ref);
        run_T<2, 4, 7, 10, 40, 256, 4>(d_f, d_X, d_out, g, ref);
        run_T<2, 4, 8, 12, 48, 128, 3>(d_f, d_X, d_out, g, ref);
        run_T<4, 4, 10, 10, 48, 512, 2>(d_f, d_X, d_out, g, ref);
        return 0;
    }
    // 2 lanes per point: tile / occupancy / split / lane-map sweep
    run_H<4, 32, 4, 0, 0>(d_f, d_X, d_out, g, ref);
    run_H<4, 32, 4, 1, 0>(d_f, d_X, d_out, g, ref);
    run_H<4, 32, 4, 0, 1>(d_f, d_X, d_out, g, ref);
    run_H<4, 32, 3, 0, 0>(d_f, d_X, d_out, g, ref);
    run_H<4, 32, 5, 0, 0>(d_f, d_X, d_out, g, ref);
    run_H<4, 16, 8, 0, 0>(d_f, d_X, d_out, g, ref);
    run_H<4, 16, 6, 0, 0>(d_f, d_X, d_out, g, ref);
    run_H<4, 16, 10, 0, 0>(d_f, d_X, d_out, g, ref);
    run_H<8, 16, 4, 0, 0>(d_f, d_X, d_out, g, ref);
    run_H<2, 32, 8, 0, 0>(d_f, d_X, d_out, g, ref);
    run_H<2, 64, 4, 0, 0>(d_f, d_X, d_out, g, ref);
    run_H<8, 32, 2, 0, 0>(d_f, d_X, d_out, g, ref);
    // 4 lanes per point
    run_H4<4, 32, 3>(d_f, d_X, d_out, g, ref);
    run_H4<4, 32, 2>(d_f, d_X, d_out, g, ref);
    run_H4<4, 16, 6>(d_f, d_X, d_out, g, ref);
    run_H4<4, 16, 4>(d_f, d_X, d_out, g, ref);
    run_H4<4, 8, 12>(d_f, d_X, d_out, g, ref);
    run_H4<8, 8, 6>(d_f, d_X, d_out, g, ref);
    run_H4<2, 32, 6>(d_f, d_X, d_out, g, ref);
    return 0;
}
