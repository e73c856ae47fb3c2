// fft.cu -- hand-written fp64 3D r2c/c2r FFTs for power-of-two periodic grids,
// fused with the spectral multipliers of the reference's spectral module.
//
// Replaces proj/src/fft.cpp (FFTW r2c/c2r 3D, forward unnormalized, inverse
// scaled by 1/N after the c2r, fft.cpp:66-115) and the serial bin loops of
// proj/src/spectral.cpp:13-214 (gradient, divergence, laplacian, (-lap+1),
// beta*A^{1,-1,-1/2}, Leray / near-incompressible K, Gaussian).
//
// Decomposition (all passes HBM-streaming, each CTA owns whole 1D lines):
//   x3 (contiguous):  k_r2c_rows / k_c2r_rows. A real row of n3 is packed as
//                     n3/2 complex values, transformed in shared memory and
//                     split/merged into the n3/2+1 half-spectrum bins.
//   x2, x1 (strided): k_fft_axis. A CTA loads TB adjacent columns (coalesced
//                     along the contiguous index) straight into registers,
//                     runs a Stockham radix-16 FFT with shared-memory exchanges,
//                     and stores straight back. The x1 pass optionally runs
//                     forward -> multiplier -> inverse in one kernel, so a
//                     scalar spectral operator costs 5 passes instead of 6.
// In-register butterflies are radix-2 DIT networks of size <= 16 with
// literal twiddles; inter-stage twiddles come from per-axis long-double
// tables (exactly rounded), so the transform error is O(eps log n).
#include "fft_core.cuh"

namespace vr {
namespace {

#ifndef VR_ROW_THREADS
#define VR_ROW_THREADS 128
#endif
// --------------------------------------------------------------------------
// x3 row kernels (real rows <-> half-spectrum rows)
// --------------------------------------------------------------------------
// Persistent CTAs walk tiles of RB rows with a two-stage cp.async pipeline: the
// next tile's rows stream into the other shared-memory stage while this tile is
// transformed, so HBM reads overlap the butterflies (the one-tile-per-CTA
// version sat at ~2 TB/s, latency bound at 25% occupancy).
template <int M>
struct RowCfg {
    static constexpr int RMAX = rmax_of(M);
    static constexpr int T = M / RMAX;
    // threads per tile: 128 (16 rows at M = 128); at M = 256 (n3 = 512) 64-thread tiles of 4 rows
    // measured 4-7 % faster (more, smaller CTAs per SM: barriers stall fewer warps)
    static constexpr int ROW_THREADS = M == 256 ? VR_ROW_THREADS / 2 : VR_ROW_THREADS;
    static constexpr int RB0 = ROW_THREADS / T;
    static constexpr int RB = RB0 < 1 ? 1 : (RB0 > 64 ? 64 : RB0);
    static constexpr int THREADS = RB * T;
    static constexpr int LD = (M + 1) + ((M + 1) >> 4) + 1;  // padded row length
    static constexpr int STAGE = LD * RB;                     // one pipeline stage (double2)
    // 2 stages + W_M, W_2M. At M = 128 three CTAs fill the SM's 228 KB exactly, so the two
    // mbarriers live in stage 0's last 16 bytes (pad slot LD - 1 of its last row: never a
    // padded position, and past the end of the linear RB x (M + 1) landing area)
    static constexpr size_t SMEM = sizeof(double2) * (2 * STAGE + 3 * M);
};
// A tile of RB consecutive rows of W double2 is one contiguous block in global memory: one
// bulk copy (cp.async.bulk, issued by one thread, completing on an mbarrier) lands it
// LINEARLY (row pitch W) at the start of the stage. The first butterfly stage reads that
// linear layout into registers, and after its barrier every later access uses the padded
// layout (row pitch LD, padi), so the bank-conflict-free exchange layout is kept.
template <int M, int W>
__device__ __forceinline__ void bulk_rows(double2* stage, const double2* src, long long tile,
                                          long long nrows, unsigned long long* bar) {
    using C = RowCfg<M>;
    if (threadIdx.x == 0) {
        const long long rows = nrows - tile * C::RB;
        const unsigned bytes =
            static_cast<unsigned>((rows < C::RB ? rows : C::RB) * W * sizeof(double2));
        mbar_expect_tx(bar, bytes);
        bulk_load(stage, src + tile * C::RB * W, bytes, bar);
    }
}
// stage the W_M and W_N (N = 2M) twiddle tables in shared memory after the rows
template <int M>
__device__ __forceinline__ void stage_row_tables(double2* smem, const double2* twM_g,
                                                 const double2* twN_g, double2*& twM,
                                                 double2*& twN) {
    using C = RowCfg<M>;
    twM = smem + 2 * C::STAGE;
    twN = twM + M;
    for (int i = threadIdx.x; i < M; i += C::THREADS) twM[i] = __ldg(twM_g + i);
    for (int i = threadIdx.x; i < 2 * M; i += C::THREADS) twN[i] = __ldg(twN_g + i);
}
__device__ __forceinline__ int padi(int i) { return i + (i >> 4); }

// async copy of tile `tile` (RB rows of W double2 each, row-contiguous in src)
// into a padded stage; rows past nrows are zero-filled
template <int M, int W>
__device__ __forceinline__ void load_rows_async(double2* stage, const double2* src, long long tile,
                                                long long nrows) {
    using C = RowCfg<M>;
    const long long base = tile * C::RB * W;
    const long long avail = (nrows - tile * C::RB) * W;
#pragma unroll 4
    for (int e = threadIdx.x; e < C::RB * W; e += C::THREADS) {
        const int r = e / W, i = e % W;
        const bool ok = e < avail;
        cp_async16(stage + r * C::LD + padi(i), src + base + (ok ? e : 0), ok);
    }
}

// r2c input rows into a stage: fp64 rows stream in with cp.async; fp32 rows (the fp32
// lane) are loaded and widened to fp64 pairs in the same padded layout (synchronously)
template <int M, class TI>
__device__ __forceinline__ void load_rows_in(double2* stage, const TI* in, long long tile,
                                             long long nrows) {
    if constexpr (std::is_same<TI, double>::value) {
        load_rows_async<M, M>(stage, reinterpret_cast<const double2*>(in), tile, nrows);
    } else {
        using C = RowCfg<M>;
        const float2* src = reinterpret_cast<const float2*>(in);
        const long long base = tile * C::RB * M;
        const long long avail = (nrows - tile * C::RB) * M;
        for (int e = threadIdx.x; e < C::RB * M; e += C::THREADS) {
            const int r = e / M, i = e % M;
            double2 v = make_double2(0.0, 0.0);
            if (e < avail) {
                const float2 f = __ldg(src + base + e);
                v = make_double2(static_cast<double>(f.x), static_cast<double>(f.y));
            }
            stage[r * C::LD + padi(i)] = v;
        }
    }
}

// r2c along x3: in nrows x 2M reals -> out nrows x (M+1) complex.
// z[m] = x[2m] + i x[2m+1]; Z = FFT_M(z); X[k] = A[k] + W_N^k B[k] with
// A = (Z[k] + conj Z[M-k]) / 2, B = (Z[k] - conj Z[M-k]) / 2i.
template <int M, class TI>
__global__ void __launch_bounds__(RowCfg<M>::THREADS)
    k_r2c_rows(const TI* __restrict__ in, double2* __restrict__ out, long long nrows,
               const double2* __restrict__ twM_g, const double2* __restrict__ twN_g) {
    using C = RowCfg<M>;
    constexpr bool LIN = std::is_same<TI, double>::value;  // fp64 rows arrive by bulk copy
    extern __shared__ __align__(128) double2 smem[];
    double2 *twM, *twN;
    stage_row_tables<M>(smem, twM_g, twN_g, twM, twN);
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + C::STAGE - 1);
    mbar_init_pair(full);
    const long long ntiles = (nrows + C::RB - 1) / C::RB;
    auto issue = [&](long long tl, int b) {
        if constexpr (LIN)
            bulk_rows<M, M>(smem + b * C::STAGE, reinterpret_cast<const double2*>(in), tl, nrows, full + b);
        else
            load_rows_in<M, TI>(smem + b * C::STAGE, in, tl, nrows);
    };
    long long tile = blockIdx.x;
    if (tile < ntiles) issue(tile, 0);
    unsigned it = 0;
    for (int b = 0; tile < ntiles; tile += gridDim.x, b ^= 1, ++it) {
        const long long next = tile + gridDim.x;
        if (next < ntiles) issue(next, b ^ 1);
        if constexpr (LIN)
            mbar_wait(full + b, (it >> 1) & 1);
        else
            __syncthreads();
        double2* buf = smem + b * C::STAGE;
        {
            const int t = threadIdx.x % C::T, r = threadIdx.x / C::T;
            auto sm = [&](int i) -> double2& { return buf[r * C::LD + padi(i)]; };
            auto load = [&](int i) -> double2 { return LIN ? buf[r * M + i] : sm(i); };
            auto store = [&](int i, double2 v) { sm(i) = v; };
            fft_line<M, -1, true, true>(t, twM, load, store, sm);
        }
        __syncthreads();
        double2* dstp = out + tile * C::RB * (M + 1);
        const long long avail_out = (nrows - tile * C::RB) * (M + 1);
        for (int e = threadIdx.x; e < C::RB * (M + 1); e += C::THREADS) {
            if (e >= avail_out) break;
            const int r = e / (M + 1), k = e % (M + 1);
            const double2* Z = buf + r * C::LD;
            double2 X;
            if (k == 0 || k == M) {
                const double2 z0 = Z[0];
                X = make_double2(k == 0 ? z0.x + z0.y : z0.x - z0.y, 0.0);
            } else {
                const double2 zk = Z[padi(k)];
                const double2 zc = cconj(Z[padi(M - k)]);
                const double2 A = make_double2(0.5 * (zk.x + zc.x), 0.5 * (zk.y + zc.y));
                const double2 D = make_double2(0.5 * (zk.x - zc.x), 0.5 * (zk.y - zc.y));
                const double2 B = make_double2(D.y, -D.x);  // D / i
                double2 w = twN[k];
                w.y = -w.y;  // exp(-2 pi i k / N)
                X = cadd(A, cmul(w, B));
            }
            dstp[e] = X;
        }
        fence_proxy_async();  // butterfly stages wrote this stage; the next TMA box overwrites it
        __syncthreads();      // this stage is refilled by the next iteration's prefetch
    }
}

// c2r along x3: in nrows x (M+1) complex -> out nrows x 2M reals,
// out = add + scale * x. Z[k] = E + i O, E = X[k] + conj X[M-k],
// O = (X[k] - conj X[M-k]) exp(+2 pi i k / N); z = IFFT_M(Z); x[2m] = Re, x[2m+1] = Im.
// Imaginary parts of the self-conjugate bins X[0], X[M] are ignored (c2r semantics).
// TO = output / add element type (float for the fp32 lane: out = float(add + scale x))
// ADD = false (plain transform: no prefetched add field) is built for 3 CTAs/SM where the
// stages allow three (M <= 128: 76.8 KB each); with the add field's 64 prefetch registers
// that cap spills and measured slower (104 vs 89 us at 256^3), so ADD = true keeps 2.
template <int M, bool ADD>
struct C2rOcc {
    static constexpr int MINB = (!ADD && 3 * (RowCfg<M>::SMEM + 1024) <= 233472) ? 3 : 2;
};
template <int M, class TO, bool ADD>
__global__ void __launch_bounds__(RowCfg<M>::THREADS, C2rOcc<M, ADD>::MINB)
    k_c2r_rows(const double2* __restrict__ in, TO* __restrict__ out, long long nrows,
               const double2* __restrict__ twM_g, const double2* __restrict__ twN_g, double scale,
               const TO* __restrict__ add_in) {
    const TO* __restrict__ add = ADD ? add_in : nullptr;
    using C = RowCfg<M>;
    using TO2 = typename std::conditional<std::is_same<TO, float>::value, float2, double2>::type;
    constexpr int PER = C::RB * M / C::THREADS;  // output double2 per thread per tile
    extern __shared__ __align__(128) double2 smem[];
    double2 *twM, *twN;
    stage_row_tables<M>(smem, twM_g, twN_g, twM, twN);
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + C::STAGE - 1);
    mbar_init_pair(full);
    const long long ntiles = (nrows + C::RB - 1) / C::RB;
    long long tile = blockIdx.x;
    if (tile < ntiles) bulk_rows<M, M + 1>(smem, in, tile, nrows, full);
    unsigned it = 0;
    for (int b = 0; tile < ntiles; tile += gridDim.x, b ^= 1, ++it) {
        const long long next = tile + gridDim.x;
        if (next < ntiles) bulk_rows<M, M + 1>(smem + (b ^ 1) * C::STAGE, in, next, nrows, full + (b ^ 1));
        const long long avail_out = (nrows - tile * C::RB) * M;
        TO2* dstp = reinterpret_cast<TO2*>(out) + tile * C::RB * M;
        // the add field's loads are issued now and land while the rows transform
        double2 addv[ADD ? PER : 1];
        if constexpr (ADD) {
            const TO2* addp = reinterpret_cast<const TO2*>(add) + tile * C::RB * M;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int e = threadIdx.x + j * C::THREADS;
                if (e < avail_out) {
                    const TO2 a = __ldcs(addp + e);
                    addv[j] = make_double2(static_cast<double>(a.x), static_cast<double>(a.y));
                } else {
                    addv[j] = make_double2(0.0, 0.0);
                }
            }
        }
        mbar_wait(full + b, (it >> 1) & 1);
        double2* buf = smem + b * C::STAGE;
        // form Z in place in the linear layout (row pitch M + 1): thread handles the pair
        // (k, M-k), k in [0, M/2]
        for (int e = threadIdx.x; e < C::RB * (M / 2 + 1); e += C::THREADS) {
            const int r = e / (M / 2 + 1), k = e % (M / 2 + 1);
            double2* X = buf + r * (M + 1);
            if (k == 0) {
                const double a = X[0].x, bb = X[M].x;
                X[0] = make_double2(a + bb, a - bb);
            } else {
                const double2 xk = X[k], xm = X[M - k];
                const double2 wk = twN[k];     // exp(+2 pi i k / N)
                const double2 wm = twN[M - k]; // exp(+2 pi i (M-k) / N)
                {
                    const double2 E = cadd(xk, cconj(xm));
                    const double2 O = cmul(csub(xk, cconj(xm)), wk);
                    X[k] = make_double2(E.x - O.y, E.y + O.x);
                }
                if (k != M - k) {
                    const double2 E = cadd(xm, cconj(xk));
                    const double2 O = cmul(csub(xm, cconj(xk)), wm);
                    X[M - k] = make_double2(E.x - O.y, E.y + O.x);
                }
            }
        }
        __syncthreads();
        {
            const int t = threadIdx.x % C::T, r = threadIdx.x / C::T;
            auto sm = [&](int i) -> double2& { return buf[r * C::LD + padi(i)]; };
            auto load = [&](int i) -> double2 { return buf[r * (M + 1) + i]; };  // linear (first stage only)
            auto store = [&](int i, double2 v) { sm(i) = v; };
            fft_line<M, +1, true, true>(t, twM, load, store, sm);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int e = threadIdx.x + j * C::THREADS;
            if (e >= avail_out) break;
            const int r = e / M, i = e % M;
            const double2 z = buf[r * C::LD + padi(i)];
            double2 o;
            if constexpr (ADD)
                o = make_double2(addv[j].x + scale * z.x, addv[j].y + scale * z.y);
            else
                o = make_double2(z.x * scale, z.y * scale);
            TO2 ot;
            ot.x = static_cast<TO>(o.x);
            ot.y = static_cast<TO>(o.y);
            dstp[e] = ot;
        }
        fence_proxy_async();  // butterfly stages wrote this stage; the next TMA box overwrites it
        __syncthreads();      // this stage is refilled by the next iteration's prefetch
    }
}

// --------------------------------------------------------------------------
// elementwise spectral kernels on fully transformed spectra in the x1-pass
// layout [n1][n2s][nh] (== (n1, n2, nh) on one GPU)
// --------------------------------------------------------------------------
__device__ __forceinline__ void bin_coords(long long b, const GridDims& g, int& i1, int& i2,
                                           int& i3) {
    i3 = static_cast<int>(b % g.nh);
    long long r = b / g.nh;
    i2 = static_cast<int>(r % g.n2s) + g.k2_off;
    i1 = static_cast<int>(r / g.n2s);
}

// <A v_c, v_c> per component by Parseval on the half spectrum (fft_freq symbol, bins with
// 0 < k3 < n3/2 stand for their conjugate partner too); per-block partials, fixed grid
__global__ void __launch_bounds__(kRedThreads)
    k_reg_energy(const double2* __restrict__ s0, const double2* __restrict__ s1,
                 const double2* __restrict__ s2, MultDev m, GridDims g, double* __restrict__ partials) {
    const double2* sp = blockIdx.y == 0 ? s0 : (blockIdx.y == 1 ? s1 : s2);
    double acc = 0.0;
    for (long long b = blockIdx.x * (long long)kRedThreads + threadIdx.x; b < g.NC;
         b += (long long)gridDim.x * kRedThreads) {
        int i1, i2, i3;
        bin_coords(b, g, i1, i2, i3);
        const double a = fft_freq(i1, g.n1), c = fft_freq(i2, g.n2), d = fft_freq(i3, g.n3);
        const double w = (i3 == 0 || 2 * i3 == g.n3) ? 1.0 : 2.0;
        const double2 v = sp[b];
        acc += w * symbol_dev(m, a * a + c * c + d * d) * (v.x * v.x + v.y * v.y);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    __shared__ double sh[kRedThreads / 32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = sh[0];
        for (int q = 1; q < kRedThreads / 32; ++q) t += sh[q];
        partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

// x3 derivative on the row spectrum [rows][nh]: c *= i deriv_freq(k3)
__global__ void k_rows_deriv(double2* __restrict__ spec, long long nbins, int nh, int n3) {
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nbins;
         b += (long long)gridDim.x * blockDim.x)
        spec[b] = cmul(make_double2(0.0, (double)deriv_freq(static_cast<int>(b % nh), n3)), spec[b]);
}

// divergence (spectral.cpp:124-140): acc = sum_a i k_a c_a, deriv_freq
__global__ void k_spec_div(const double2* __restrict__ c0, const double2* __restrict__ c1,
                           const double2* __restrict__ c2, double2* __restrict__ out, GridDims g) {
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < g.NC;
         b += (long long)gridDim.x * blockDim.x) {
        int i1, i2, i3;
        bin_coords(b, g, i1, i2, i3);
        double2 acc = make_double2(0.0, 0.0);
        acc = cadd(acc, cmul(make_double2(0.0, (double)deriv_freq(i1, g.n1)), c0[b]));
        acc = cadd(acc, cmul(make_double2(0.0, (double)deriv_freq(i2, g.n2)), c1[b]));
        acc = cadd(acc, cmul(make_double2(0.0, (double)deriv_freq(i3, g.n3)), c2[b]));
        out[b] = acc;
    }
}

// projections (spectral.cpp:190-214)
__global__ void k_spec_project(double2* __restrict__ c0, double2* __restrict__ c1,
                               double2* __restrict__ c2, GridDims g, int kind, double beta_v,
                               double beta_w) {
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < g.NC;
         b += (long long)gridDim.x * blockDim.x) {
        int i1, i2, i3;
        bin_coords(b, g, i1, i2, i3);
        const double k[3] = {(double)deriv_freq(i1, g.n1), (double)deriv_freq(i2, g.n2),
                             (double)deriv_freq(i3, g.n3)};
        const double kk = k[0] * k[0] + k[1] * k[1] + k[2] * k[2];
        if (kk == 0.0) continue;
        double s = 1.0;
        if (kind == VR_PROJ_NEAR_INCOMPRESSIBLE)
            s = beta_w * (kk + 1.0) / (beta_v + beta_w * (kk + 1.0));
        const double2 a0 = c0[b], a1 = c1[b], a2 = c2[b];
        double2 kdotf = make_double2(k[0] * a0.x, k[0] * a0.y);
        kdotf = cadd(kdotf, make_double2(k[1] * a1.x, k[1] * a1.y));
        kdotf = cadd(kdotf, make_double2(k[2] * a2.x, k[2] * a2.y));
        const double f = s / kk;
        const double2 corr = make_double2(kdotf.x * f, kdotf.y * f);
        c0[b] = csub(a0, make_double2(k[0] * corr.x, k[0] * corr.y));
        c1[b] = csub(a1, make_double2(k[1] * corr.x, k[1] * corr.y));
        c2[b] = csub(a2, make_double2(k[2] * corr.x, k[2] * corr.y));
    }
}

template <int M>
void launch_rows_f32in(vr_ctx* ctx, const float* in, double* spec) {
    using C = RowCfg<M>;
    const long long nrows = static_cast<long long>(ctx->g.L) * ctx->g.n2;
    const long long ntiles = (nrows + C::RB - 1) / C::RB;
    static int occ[64] = {0};
    const unsigned grid = persistent_grid(ctx, k_r2c_rows<M, float>, C::THREADS, C::SMEM, ntiles, occ);
    VR_LAUNCH(ctx, "fft_x3_r2c", k_r2c_rows<M, float><<<grid, C::THREADS, C::SMEM, ctx->stream>>>(
        in, reinterpret_cast<double2*>(spec), nrows, ctx->fft->tw3h, ctx->fft->tw3));
}

template <int M>
void launch_rows_f32out(vr_ctx* ctx, const void* in, float* out, double scale, const float* add) {
    using C = RowCfg<M>;
    const long long nrows = static_cast<long long>(ctx->g.L) * ctx->g.n2;
    const long long ntiles = (nrows + C::RB - 1) / C::RB;
    if (add) {
        static int occ[64] = {0};
        const unsigned grid = persistent_grid(ctx, k_c2r_rows<M, float, true>, C::THREADS, C::SMEM, ntiles, occ);
        VR_LAUNCH(ctx, "fft_x3_c2r", k_c2r_rows<M, float, true><<<grid, C::THREADS, C::SMEM, ctx->stream>>>(
            static_cast<const double2*>(in), out, nrows, ctx->fft->tw3h, ctx->fft->tw3, scale, add));
    } else {
        static int occ[64] = {0};
        const unsigned grid = persistent_grid(ctx, k_c2r_rows<M, float, false>, C::THREADS, C::SMEM, ntiles, occ);
        VR_LAUNCH(ctx, "fft_x3_c2r", k_c2r_rows<M, float, false><<<grid, C::THREADS, C::SMEM, ctx->stream>>>(
            static_cast<const double2*>(in), out, nrows, ctx->fft->tw3h, ctx->fft->tw3, scale, nullptr));
    }
}

template <int M>
void launch_rows_t(vr_ctx* ctx, bool forward, const void* in, void* out, double scale,
                   const double* add) {
    using C = RowCfg<M>;
    const long long nrows = static_cast<long long>(ctx->g.L) * ctx->g.n2;  // local rows
    const long long ntiles = (nrows + C::RB - 1) / C::RB;
    if (forward) {
        static int occ[64] = {0};
        const unsigned grid = persistent_grid(ctx, k_r2c_rows<M, double>, C::THREADS, C::SMEM, ntiles, occ);
        VR_LAUNCH(ctx, "fft_x3_r2c", k_r2c_rows<M, double><<<grid, C::THREADS, C::SMEM, ctx->stream>>>(
            static_cast<const double*>(in), static_cast<double2*>(out), nrows, ctx->fft->tw3h,
            ctx->fft->tw3));
    } else if (add) {
        static int occ[64] = {0};
        const unsigned grid = persistent_grid(ctx, k_c2r_rows<M, double, true>, C::THREADS, C::SMEM, ntiles, occ);
        VR_LAUNCH(ctx, "fft_x3_c2r", k_c2r_rows<M, double, true><<<grid, C::THREADS, C::SMEM, ctx->stream>>>(
            static_cast<const double2*>(in), static_cast<double*>(out), nrows, ctx->fft->tw3h,
            ctx->fft->tw3, scale, add));
    } else {
        static int occ[64] = {0};
        const unsigned grid = persistent_grid(ctx, k_c2r_rows<M, double, false>, C::THREADS, C::SMEM, ntiles, occ);
        VR_LAUNCH(ctx, "fft_x3_c2r", k_c2r_rows<M, double, false><<<grid, C::THREADS, C::SMEM, ctx->stream>>>(
            static_cast<const double2*>(in), static_cast<double*>(out), nrows, ctx->fft->tw3h,
            ctx->fft->tw3, scale, nullptr));
    }
}

void launch_rows(vr_ctx* ctx, bool forward, const void* in, void* out, double scale,
                 const double* add) {
    switch (ctx->g.n3 / 2) {
#define VR_CASE(MM) \
    case MM: launch_rows_t<MM>(ctx, forward, in, out, scale, add); break;
        VR_CASE(2)
        VR_CASE(4)
        VR_CASE(8)
        VR_CASE(16)
        VR_CASE(32)
        VR_CASE(64)
        VR_CASE(128)
        VR_CASE(256)
        VR_CASE(512)
#undef VR_CASE
        default: throw_dimension("fft: unsupported n3 " + std::to_string(ctx->g.n3));
    }
}

unsigned spec_grid(const GridDims& g) {
    return static_cast<unsigned>(std::min<long long>((g.NC + 255) / 256, 148LL * 16));
}

void upload_table(double2** dst, int n) {
    std::vector<double2> h(n);
    const long double two_pi_l = 6.283185307179586476925286766559005768L;
    for (int k = 0; k < n; ++k) {
        long double a = two_pi_l * static_cast<long double>(k) / static_cast<long double>(n);
        h[k] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(sinl(a)));
    }
    VR_CUDA(cudaMalloc(dst, sizeof(double2) * n));
    VR_CUDA(cudaMemcpy(*dst, h.data(), sizeof(double2) * n, cudaMemcpyHostToDevice));
}

}  // namespace

// ============================================================================
// pass-level primitives (spectral.cu composes them, incl. the slab transposes)
// ============================================================================
void fft_plan_create(vr_ctx* ctx) {
    auto* p = new FftPlan();
    ctx->fft = p;
    upload_table(&p->tw1, ctx->g.n1);
    upload_table(&p->tw2, ctx->g.n2);
    upload_table(&p->tw3h, ctx->g.n3 / 2);
    upload_table(&p->tw3, ctx->g.n3);
}
void fft_plan_destroy(vr_ctx* ctx) {
    if (!ctx->fft) return;
    cudaFree(ctx->fft->tw1);
    cudaFree(ctx->fft->tw2);
    cudaFree(ctx->fft->tw3h);
    cudaFree(ctx->fft->tw3);
    delete ctx->fft;
    ctx->fft = nullptr;
}

void pass_rows_forward(vr_ctx* ctx, const double* in, double* spec) {
    launch_rows(ctx, true, in, spec, 1.0, nullptr);
}
void pass_rows_inverse(vr_ctx* ctx, const double* spec, double* out, double scale,
                       const double* add) {
    launch_rows(ctx, false, spec, out, scale, add);
}
void pass_rows_forward_f32(vr_ctx* ctx, const float* in, double* spec) {
    switch (ctx->g.n3 / 2) {
#define VR_CASE(MM) \
    case MM: launch_rows_f32in<MM>(ctx, in, spec); break;
        VR_CASE(2)
        VR_CASE(4)
        VR_CASE(8)
        VR_CASE(16)
        VR_CASE(32)
        VR_CASE(64)
        VR_CASE(128)
        VR_CASE(256)
        VR_CASE(512)
#undef VR_CASE
        default: throw_dimension("fft: unsupported n3 " + std::to_string(ctx->g.n3));
    }
}
void pass_rows_inverse_f32(vr_ctx* ctx, const double* spec, float* out, double scale,
                           const float* add) {
    switch (ctx->g.n3 / 2) {
#define VR_CASE(MM) \
    case MM: launch_rows_f32out<MM>(ctx, spec, out, scale, add); break;
        VR_CASE(2)
        VR_CASE(4)
        VR_CASE(8)
        VR_CASE(16)
        VR_CASE(32)
        VR_CASE(64)
        VR_CASE(128)
        VR_CASE(256)
        VR_CASE(512)
#undef VR_CASE
        default: throw_dimension("fft: unsupported n3 " + std::to_string(ctx->g.n3));
    }
}
// d f / d x_axis of a real field on one GPU, one axis only: the derivative is a
// 1D spectral operator along that axis (the other axes' transforms cancel), so x1
// and x2 are one fused pass over f viewed as complex pairs and x3 is a row
// r2c -> i k3 -> c2r round trip (spec: scratch of NC complex)
void deriv_axis(vr_ctx* ctx, int axis, const double* f, double* out, double* spec) {
    const GridDims& g = ctx->g;
    if (axis < 2) {
        deriv_axis_strided(ctx, axis, f, out);  // fft_axis.cu
    } else {
        launch_rows(ctx, true, f, spec, 1.0, nullptr);
        const long long nb = static_cast<long long>(g.L) * g.n2 * g.nh;
        VR_LAUNCH(ctx, "fft_spectral", k_rows_deriv<<<spec_grid(g), 256, 0, ctx->stream>>>(
            reinterpret_cast<double2*>(spec), nb, g.nh, g.n3));
        launch_rows(ctx, false, spec, out, 1.0 / g.n3, nullptr);
    }
}
// <A v, v>_h = h1 h2 h3 sum_c sum_x (A v_c) v_c (A at beta = 1, apply mode) by Parseval:
// three forward transforms and a spectrum reduction instead of three transform round
// trips and a real-space inner product (one GPU)
double reg_energy(vr_ctx* ctx, const double* v3, const vr_regnorm& norm) {
    const GridDims& g = ctx->g;
    double* sp[3];
    for (int c = 0; c < 3; ++c) {
        sp[c] = spec_buf(ctx, 1 + c);
        fft_r2c(ctx, v3 + c * g.N, sp[c]);
    }
    MultDev m{};
    m.reg_kind = norm.kind;
    m.gamma = norm.gamma;
    m.helm_sq = norm.helmholtz_squared;
    VR_LAUNCH(ctx, "reduce", k_reg_energy<<<dim3(kRedBlocks, 3), kRedThreads, 0, ctx->stream>>>(
        reinterpret_cast<const double2*>(sp[0]), reinterpret_cast<const double2*>(sp[1]),
        reinterpret_cast<const double2*>(sp[2]), m, g, ctx->red_partials));
    double part[3];
    finalize_sums(ctx, kRedBlocks, 3, part);
    return (part[0] + part[1] + part[2]) / static_cast<double>(g.Ng) * (g.h1 * g.h2 * g.h3);
}
void pass_spec_div(vr_ctx* ctx, const double* s0, const double* s1, const double* s2, double* acc) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "fft_spectral", k_spec_div<<<spec_grid(g), 256, 0, ctx->stream>>>(
        reinterpret_cast<const double2*>(s0), reinterpret_cast<const double2*>(s1),
        reinterpret_cast<const double2*>(s2), reinterpret_cast<double2*>(acc), g));
}
void pass_spec_project(vr_ctx* ctx, double* s0, double* s1, double* s2, int kind, double beta_v,
                       double beta_w) {
    const GridDims& g = ctx->g;
    VR_LAUNCH(ctx, "fft_spectral", k_spec_project<<<spec_grid(g), 256, 0, ctx->stream>>>(
        reinterpret_cast<double2*>(s0), reinterpret_cast<double2*>(s1),
        reinterpret_cast<double2*>(s2), g, kind, beta_v, beta_w));
}

}  // namespace vr
