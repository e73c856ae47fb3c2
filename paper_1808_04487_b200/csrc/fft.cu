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
#include <cuda.h>  // CUtensorMap types; cuTensorMapEncodeTiled is resolved at run time (no -lcuda)

#include <cmath>
#include <type_traits>

#include "vr_common.cuh"

namespace vr {

struct FftPlan {
    double2* tw1 = nullptr;   // exp(2 pi i k / n1), k < n1 (cos, sin)
    double2* tw2 = nullptr;   // n2
    double2* tw3h = nullptr;  // n3 / 2
    double2* tw3 = nullptr;   // n3
};

namespace {

// --------------------------------------------------------------------------
// complex helpers
// --------------------------------------------------------------------------
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

constexpr int bitrev_c(int i, int r) {
    int out = 0;
    for (int b = 1; b < r; b <<= 1) {
        out = (out << 1) | (i & 1);
        i >>= 1;
    }
    return out;
}

// exp(DIR * 2 pi i k / 16), k in [0, 8)
template <int DIR>
__device__ __forceinline__ double2 w16(int k) {
    constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173,
                     R2 = 0.70710678118654752440;
    const double c[8] = {1.0, C1, R2, S1, 0.0, -S1, -R2, -C1};
    const double s[8] = {0.0, S1, R2, C1, 1.0, C1, R2, S1};
    return make_double2(c[k], DIR * s[k]);
}

// In-register DFT of size R (<= 16): X[k] = sum_n x[n] exp(DIR 2 pi i n k / R)
template <int R, int DIR>
__device__ __forceinline__ void dft_reg(double2* x) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int j = bitrev_c(i, R);
        if (j > i) {
            double2 t = x[i];
            x[i] = x[j];
            x[j] = t;
        }
    }
    constexpr int LOG2R = R >= 16 ? 4 : R >= 8 ? 3 : R >= 4 ? 2 : 1;
#pragma unroll
    for (int s = 0; s < LOG2R; ++s) {  // constant trip count: fully unrolled, literal twiddles
        const int len = 2 << s;
#pragma unroll
        for (int start = 0; start < R; start += len) {
#pragma unroll
            for (int k = 0; k < len / 2; ++k) {
                const int widx = k * (16 / len);
                double2 b = x[start + k + len / 2];
                double2 t;
                if (widx == 0) {
                    t = b;
                } else if (widx == 4) {
                    t = make_double2(-DIR * b.y, DIR * b.x);  // b * (DIR i)
                } else {
                    t = cmul(b, w16<DIR>(widx));
                }
                const double2 a = x[start + k];
                x[start + k] = cadd(a, t);
                x[start + k + len / 2] = csub(a, t);
            }
        }
    }
}

__host__ __device__ constexpr int rmax_of(int n) { return n < 16 ? n : 16; }

// One Stockham stage of radix R for a length-N transform with Ns = product of
// previous radices; this thread handles butterflies j = t + b*T, b < RMAX/R.
// SRC(i) reads element i, DST(i, v) writes element i. Caller handles syncs.
template <int N, int R, int DIR, class Src, class Dst>
__device__ __forceinline__ void stockham_stage(int Ns, int t, const double2* __restrict__ tw,
                                               Src src, Dst dst, bool sync_between) {
    constexpr int RMAX = rmax_of(N);
    constexpr int T = N / RMAX;
    constexpr int NB = RMAX / R;
    double2 x[RMAX];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = t + b * T;
#pragma unroll
        for (int r = 0; r < R; ++r) x[b * R + r] = src(j + r * (N / R));
    }
    if (sync_between) __syncthreads();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = t + b * T;
        const int k = j & (Ns - 1);
        if (Ns > 1) {
            const int step = N / (Ns * R);
#pragma unroll
            for (int r = 1; r < R; ++r) {
                double2 w = tw[r * k * step];  // shared-memory table
                if (DIR < 0) w.y = -w.y;
                x[b * R + r] = cmul(x[b * R + r], w);
            }
        }
        dft_reg<R, DIR>(x + b * R);
        const int out = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) dst(out + r * Ns, x[b * R + r]);
    }
}

// Full length-N transform. The first stage reads LOAD(i), the last writes
// STORE(i, v); intermediate stages exchange through shared memory via SM(i)
// (a reference to this column's element i). SRC_SM / DST_SM say whether LOAD /
// STORE alias that shared buffer, which decides where barriers are needed.
// Must be called by all threads of the CTA (barriers inside).
template <int N, int DIR, bool SRC_SM, bool DST_SM, class Load, class Store, class Sm>
__device__ __forceinline__ void fft_line(int t, const double2* __restrict__ tw, Load load,
                                         Store store, Sm sm) {
    auto sm_src = [&](int i) { return sm(i); };
    auto sm_dst = [&](int i, double2 v) { sm(i) = v; };
    int Ns = 1;
    bool first = true;
    while (Ns < N) {
        const int rem = N / Ns;
        const bool last = rem <= 16;
        const int R = rem >= 16 ? 16 : rem;
        const bool reads_sm = !first || SRC_SM;
        const bool writes_sm = !last || DST_SM;
        const bool sync_between = reads_sm && writes_sm;
        // R is uniform across the CTA; dispatch to compile-time radices
#define VR_STAGE(RR)                                                                           \
    if (R == RR) {                                                                             \
        if (first && last)                                                                     \
            stockham_stage<N, RR, DIR>(Ns, t, tw, load, store, sync_between);                  \
        else if (first)                                                                        \
            stockham_stage<N, RR, DIR>(Ns, t, tw, load, sm_dst, sync_between);                 \
        else if (last)                                                                         \
            stockham_stage<N, RR, DIR>(Ns, t, tw, sm_src, store, sync_between);                \
        else                                                                                   \
            stockham_stage<N, RR, DIR>(Ns, t, tw, sm_src, sm_dst, sync_between);               \
    }
        if constexpr (N >= 16) { VR_STAGE(16) }
        if constexpr (N >= 8) { VR_STAGE(8) }
        if constexpr (N >= 4) { VR_STAGE(4) }
        VR_STAGE(2)
#undef VR_STAGE
        if (!last) __syncthreads();
        first = false;
        Ns *= R;
    }
}

// --------------------------------------------------------------------------
// spectral multipliers (spectral.cpp:23-39, 84-184)
// --------------------------------------------------------------------------
struct MultDev {
    int kind;
    int reg_kind, reg_mode, helm_sq;
    double gamma, beta;
    double sig2h2[3];
};

__device__ __forceinline__ double symbol_dev(const MultDev& m, double k2) {
    switch (m.reg_kind) {
        case VR_REG_H1: return k2;
        case VR_REG_H2: return k2 * k2;
        case VR_REG_H3: return k2 * k2 * k2;
        default: {
            double s = k2 + m.gamma;
            return m.helm_sq ? s * s : s;
        }
    }
}

// returns the complex multiplier at bin (i1, i2, i3)
__device__ __forceinline__ double2 mult_at(const MultDev& m, const GridDims& g, int i1, int i2,
                                           int i3) {
    switch (m.kind) {
        case static_cast<int>(Mult::deriv0): return make_double2(0.0, (double)deriv_freq(i1, g.n1));
        case static_cast<int>(Mult::deriv1): return make_double2(0.0, (double)deriv_freq(i2, g.n2));
        case static_cast<int>(Mult::deriv2): return make_double2(0.0, (double)deriv_freq(i3, g.n3));
        default: break;
    }
    const double a = fft_freq(i1, g.n1), b = fft_freq(i2, g.n2), c = fft_freq(i3, g.n3);
    const double k2 = a * a + b * b + c * c;
    double v = 1.0;
    switch (m.kind) {
        case static_cast<int>(Mult::laplacian): v = -k2; break;
        case static_cast<int>(Mult::helmholtz1): v = k2 + 1.0; break;
        case static_cast<int>(Mult::reg): {
            const double s = symbol_dev(m, k2);
            if (m.reg_mode == VR_REGOP_APPLY)
                v = m.beta * s;
            else if (m.reg_mode == VR_REGOP_INVERSE)
                v = 1.0 / (m.beta * (s == 0.0 ? 1.0 : s));
            else
                v = 1.0 / sqrt(m.beta * (s == 0.0 ? 1.0 : s));
            break;
        }
        case static_cast<int>(Mult::gaussian): {
            const double e = m.sig2h2[0] * a * a + m.sig2h2[1] * b * b + m.sig2h2[2] * c * c;
            v = exp(-0.5 * e);
            break;
        }
        default: break;
    }
    return make_double2(v, 0.0);
}

// beta * A^{1,-1,-1/2} at |k|^2 = k2 (the Mult::reg branch of mult_at, same arithmetic)
__device__ __forceinline__ double reg_mult_k2(const MultDev& m, double k2) {
    const double s = symbol_dev(m, k2);
    if (m.reg_mode == VR_REGOP_APPLY) return m.beta * s;
    if (m.reg_mode == VR_REGOP_INVERSE) return 1.0 / (m.beta * (s == 0.0 ? 1.0 : s));
    return 1.0 / sqrt(m.beta * (s == 0.0 ? 1.0 : s));
}

__device__ __forceinline__ double2 apply_mult(double2 m, double2 c) {
    // real multipliers: c * m.x (exactly like complex<double> *= double);
    // imaginary (derivative) multipliers: (0, k) * c
    if (m.y == 0.0) return make_double2(c.x * m.x, c.y * m.x);
    return cmul(m, c);
}


// --------------------------------------------------------------------------
// strided-axis kernel (x1 / x2 passes)
// --------------------------------------------------------------------------
#ifndef VR_ROW_THREADS
#define VR_ROW_THREADS 128
#endif
// async global -> shared copies (16 B, zero-fill when !pred) for the pipelined passes
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc),
                 "r"(pred ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

#ifndef VR_AXIS_COLS
#define VR_AXIS_COLS 2048  // TB = VR_AXIS_COLS / N columns per tile (8 at N = 256)
#endif
template <int N>
struct AxisCfg {
    static constexpr int RMAX = rmax_of(N);
    static constexpr int T = N / RMAX;
    static constexpr int TB0 = VR_AXIS_COLS / N;
    static constexpr int TB = TB0 < 1 ? 1 : (TB0 > 64 ? 64 : TB0);
    static constexpr int THREADS = TB * T;
    static constexpr int STAGE = N * TB;  // one pipeline stage (double2)
    static constexpr int BOX_ROWS = N < 256 ? N : 256;  // TMA box height (<= 256 per dimension)
    static constexpr size_t SMEM = sizeof(double2) * (2 * STAGE + N) + 16;  // 2 stages + W_N + 2 mbarriers
};

// ---- TMA (cp.async.bulk.tensor) + mbarrier helpers for the strided passes ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// one 5D box (columns x rows x row groups x peer blocks x outer block) global -> shared,
// completing on `bar`
__device__ __forceinline__ void tma_load_5d(void* sdst, const CUtensorMap* tmap, int x, int outer,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %3, %3, %4}], [%5];"
        ::"r"(smem_u32(sdst)), "l"(reinterpret_cast<unsigned long long>(tmap)), "r"(x), "r"(0), "r"(outer),
        "r"(smem_u32(bar))
        : "memory");
}
// generic-proxy shared-memory accesses before this fence are ordered before later
// async-proxy (TMA) writes to the same locations
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// contiguous global -> shared bulk copy (bytes: multiple of 16), completing on `bar`
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_init_pair(unsigned long long* bars) {
    if (threadIdx.x == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
}

// Strided-axis pass over tiles of TB adjacent columns x N elements, persistent
// CTAs with a two-stage cp.async pipeline (the next tile streams in while this
// one is transformed; the last butterfly stage stores straight to HBM).
// MODE 0: transform in direction DIR (src may equal dst)
// MODE 1: forward -> multiplier -> inverse (x1 pass only), src -> dst (may alias)
// MODE 3: as MODE 1 for the regularisation multiplier (Mult::reg), applied in the last
//         forward butterfly stage's stores (no separate multiplier sweep over shared memory)
// MODE 2: forward -> i deriv_freq(k) * m.beta -> inverse along this axis: the spectral
//         derivative of a REAL field viewed as complex pairs (x3 = 2j, 2j+1 as re, im);
//         i k (Nyquist 0) maps real lines to real lines, so the pair never mixes
// SC (x1 slabs, forward x2 pass): the last stage stores row i of block `ob` straight into the
//         all-to-all send layout, dst + (i >> sc_shift) * sc_blk + ((ob << sc_shift) + (i & mask)) * inner
//         (block q = rows [q n2s, (q+1) n2s) of every plane), so the transpose needs no pack copy.
//         The matching unpack of the inverse direction is done by the tensor map of the loads.
template <int N, int DIR, int MODE, bool SC>
__global__ void __launch_bounds__(AxisCfg<N>::THREADS, 1)
    k_fft_axis(const __grid_constant__ CUtensorMap tmap, double2* dst, long long inner, long long outer,
               long long outer_stride, const double2* __restrict__ tw_g, MultDev m, GridDims g,
               int sc_shift, long long sc_blk) {
    using C = AxisCfg<N>;
    extern __shared__ __align__(128) double2 smem[];
    double2* tw = smem + 2 * C::STAGE;  // W_N table staged once per CTA (broadcast reads)
    unsigned long long* full = reinterpret_cast<unsigned long long*>(tw + N);  // one mbarrier per stage
    for (int i = threadIdx.x; i < N; i += C::THREADS) tw[i] = __ldg(tw_g + i);
    const long long ncb = (inner + C::TB - 1) / C::TB;
    const long long ntiles = ncb * outer;
    const int col = threadIdx.x % C::TB;
    const int t = threadIdx.x / C::TB;
    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        mbar_init(full + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // tile = TB adjacent columns x N rows of block `ob`: one TMA box per 256 rows, issued by
    // one thread; columns past `inner` are zero-filled by the copy engine
    auto issue = [&](long long tile, int b) {
        const long long ob = tile / ncb, c0 = (tile - ob * ncb) * C::TB;
        mbar_expect_tx(full + b, static_cast<unsigned>(C::STAGE * sizeof(double2)));
        tma_load_5d(smem + b * C::STAGE, &tmap, static_cast<int>(2 * c0), static_cast<int>(ob), full + b);
    };
    long long tile = blockIdx.x;
    if (threadIdx.x == 0 && tile < ntiles) issue(tile, 0);
    unsigned it = 0;
    for (int b = 0; tile < ntiles; tile += gridDim.x, b ^= 1, ++it) {
        const long long next = tile + gridDim.x;
        if (threadIdx.x == 0 && next < ntiles) issue(next, b ^ 1);
        mbar_wait(full + b, (it >> 1) & 1);
        double2* buf = smem + b * C::STAGE;
        const long long ob = tile / ncb;
        const long long cc = (tile - ob * ncb) * C::TB + col;
        const bool valid = cc < inner;
        double2* d = dst + (SC ? (ob << sc_shift) * inner : ob * outer_stride) + (valid ? cc : 0);
        auto sm = [&](int i) -> double2& { return buf[i * C::TB + col]; };
        auto load_sm = [&](int i) -> double2 { return sm(i); };
        auto store = [&](int i, double2 v) {
            if (!valid) return;
            if constexpr (SC)
                d[(i >> sc_shift) * sc_blk + static_cast<long long>(i & ((1 << sc_shift) - 1)) * inner] = v;
            else
                d[static_cast<long long>(i) * inner] = v;
        };
        if constexpr (MODE == 0) {
            fft_line<N, DIR, true, false>(t, tw, load_sm, store, sm);
        } else if constexpr (MODE == 2) {
            auto store_sm = [&](int i, double2 v) { sm(i) = v; };
            fft_line<N, -1, true, true>(t, tw, load_sm, store_sm, sm);
            __syncthreads();
#pragma unroll 1
            for (int i = t; i < N; i += C::T) {
                const double2 c = cmul(make_double2(0.0, (double)deriv_freq(i, N)), sm(i));
                sm(i) = make_double2(c.x * m.beta, c.y * m.beta);
            }
            __syncthreads();
            fft_line<N, +1, true, false>(t, tw, load_sm, store, sm);
        } else if constexpr (MODE == 3) {
            // x1 pass: column cc = i2 * nh + i3; |k|^2 = fft_freq(i1)^2 + kk23 (integers: exact)
            const int i2 = static_cast<int>(cc / g.nh) + g.k2_off;
            const int i3 = static_cast<int>(cc % g.nh);
            const double b2 = fft_freq(i2, g.n2), b3 = fft_freq(i3, g.n3);
            const double kk23 = b2 * b2 + b3 * b3;
            auto store_mult = [&](int i, double2 v) {
                const double a = fft_freq(i, N);
                const double mk = reg_mult_k2(m, a * a + kk23);
                sm(i) = make_double2(v.x * mk, v.y * mk);
            };
            fft_line<N, -1, true, true>(t, tw, load_sm, store_mult, sm);
            __syncthreads();
            fft_line<N, +1, true, false>(t, tw, load_sm, store, sm);
        } else {
            // x1 pass: column cc = i2 * nh + i3
            const int i2 = static_cast<int>(cc / g.nh) + g.k2_off;  // k2-slab on x1 slabs
            const int i3 = static_cast<int>(cc % g.nh);
            auto store_sm = [&](int i, double2 v) { sm(i) = v; };
            fft_line<N, -1, true, true>(t, tw, load_sm, store_sm, sm);
            __syncthreads();
            // one (not unrolled) copy of the multiplier code: inlining mult_at into
            // every butterfly store made this kernel ~40k instructions (i-cache bound)
#pragma unroll 1
            for (int i = t; i < N; i += C::T) sm(i) = apply_mult(mult_at(m, g, i, i2, i3), sm(i));
            __syncthreads();
            fft_line<N, +1, true, false>(t, tw, load_sm, store, sm);
        }
        fence_proxy_async();  // butterfly stages wrote this stage; the next TMA box overwrites it
        __syncthreads();      // this stage is refilled by the next iteration's prefetch
    }
}

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
    static constexpr int RB0 = VR_ROW_THREADS / T;
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

MultDev to_dev(const MultParams& p) {
    MultDev m;
    m.kind = static_cast<int>(p.kind);
    m.reg_kind = p.reg_kind;
    m.reg_mode = p.reg_mode;
    m.helm_sq = p.helm_sq;
    m.gamma = p.gamma;
    m.beta = p.beta;
    for (int a = 0; a < 3; ++a) m.sig2h2[a] = p.sig2h2[a];
    return m;
}

// ---- host-side launchers ----------------------------------------------------
// persistent grid: as many CTAs as fit on the device at once (<= one per tile).
// `occ` is the caller's per-kernel cache (kernels of one signature share a
// function-pointer type, so the cache cannot live in a template on K).
template <class K>
unsigned persistent_grid(vr_ctx* ctx, K kern, int threads, size_t smem, long long ntiles,
                         int (&occ)[64]) {
    const int d = ctx->device & 63;
    if (!occ[d]) {
        VR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
        int o = 0;
        VR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem));
        occ[d] = o > 0 ? o : 1;
    }
    const long long g = static_cast<long long>(occ[d]) * ctx->sms;
    return static_cast<unsigned>(ntiles < g ? ntiles : g);
}

// Tensor map of one strided pass: (2 inner doubles) x N rows x outer blocks, box = TB columns
// x min(N, 256) rows. Encoded on the host per launch (the source buffer changes per call).
using TmapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
inline TmapEncodeFn tmap_encoder() {
    static TmapEncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
        VR_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            throw_resource("fft: the CUDA driver does not export cuTensorMapEncodeTiled");
        return reinterpret_cast<TmapEncodeFn>(p);
    }();
    return fn;
}
// Row layout of a strided pass's SOURCE: the N rows of one block are Q2 peer blocks of Q1
// groups of R rows (R <= 256, the box limit per dimension); row r of group q1 of peer block q2
// sits at (q2 * q2_stride + q1 * R * inner + r * inner) double2 from the block's base. Plain
// layout: Q2 = 1. All-to-all receive layout on x1 slabs: Q2 = P peer blocks of n2s = Q1 * R
// rows each, q2_stride = the block size, and consecutive planes n2s * inner apart.
struct RowGroups {
    int rows_per_block = 0;      // 0: plain layout (one block of N rows)
    long long q2_stride = 0;
    long long outer_stride = 0;  // of the source blocks (0: same as the destination's)
};
template <int N>
CUtensorMap axis_tmap(const double2* src, long long inner, long long outer, long long outer_stride,
                      RowGroups rg) {
    using C = AxisCfg<N>;
    const int rows = rg.rows_per_block ? rg.rows_per_block : N;
    const int R = rows < 256 ? rows : 256, Q1 = rows / R, Q2 = N / rows;
    if (R * Q1 * Q2 != N || Q1 > 256 || Q2 > 256) throw_logic("fft: bad row grouping for the tensor map");
    if (rg.outer_stride) outer_stride = rg.outer_stride;
    CUtensorMap tm;
    const cuuint64_t dims[5] = {static_cast<cuuint64_t>(2 * inner), static_cast<cuuint64_t>(R),
                                static_cast<cuuint64_t>(Q1), static_cast<cuuint64_t>(Q2),
                                static_cast<cuuint64_t>(outer)};
    // strides of dimensions 1..4 in bytes (dimension 0 is contiguous)
    const cuuint64_t strides[4] = {
        static_cast<cuuint64_t>(inner) * sizeof(double2), static_cast<cuuint64_t>(R) * inner * sizeof(double2),
        static_cast<cuuint64_t>(Q2 > 1 ? rg.q2_stride : static_cast<long long>(rows) * inner) * sizeof(double2),
        static_cast<cuuint64_t>(outer > 1 ? outer_stride : inner * N) * sizeof(double2)};
    const cuuint32_t box[5] = {2u * C::TB, static_cast<cuuint32_t>(R), static_cast<cuuint32_t>(Q1),
                               static_cast<cuuint32_t>(Q2), 1u};
    const cuuint32_t estr[5] = {1u, 1u, 1u, 1u, 1u};
    const CUresult r = tmap_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double2*>(src), dims,
                                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw_resource("fft: cuTensorMapEncodeTiled failed (code " + std::to_string(static_cast<int>(r)) + ")");
    return tm;
}

// sc_blk > 0: scatter the stores into all-to-all blocks of sc_blk double2 (rows per block = 1 << sc_shift)
template <int N, int DIR, int MODE, bool SC = false>
void launch_axis_t(vr_ctx* ctx, const double2* src, double2* dst, long long inner, long long outer,
                   long long outer_stride, const double2* tw, const MultDev& m, RowGroups rg = {},
                   int sc_shift = 0, long long sc_blk = 0) {
    using C = AxisCfg<N>;
    static int occ[64] = {0};
    const long long ntiles = (inner + C::TB - 1) / C::TB * outer;
    const unsigned grid =
        persistent_grid(ctx, k_fft_axis<N, DIR, MODE, SC>, C::THREADS, C::SMEM, ntiles, occ);
    const CUtensorMap tm = axis_tmap<N>(src, inner, outer, outer_stride, rg);
    VR_LAUNCH(ctx, MODE == 0 ? "fft_axis" : (MODE == 1 || MODE == 3 ? "fft_x1_mult" : "fft_deriv"),
              k_fft_axis<N, DIR, MODE, SC><<<grid, C::THREADS, C::SMEM, ctx->stream>>>(
                  tm, dst, inner, outer, outer_stride, tw, m, ctx->g, sc_shift, sc_blk));
}

template <int DIR, int MODE>
void launch_axis(vr_ctx* ctx, int n, const double2* src, double2* dst, long long inner,
                 long long outer, long long outer_stride, const double2* tw, const MultDev& m) {
    switch (n) {
#define VR_CASE(NN) \
    case NN: launch_axis_t<NN, DIR, MODE>(ctx, src, dst, inner, outer, outer_stride, tw, m); break;
        VR_CASE(4)
        VR_CASE(8)
        VR_CASE(16)
        VR_CASE(32)
        VR_CASE(64)
        VR_CASE(128)
        VR_CASE(256)
        VR_CASE(512)
        VR_CASE(1024)
#undef VR_CASE
        default: throw_dimension("fft: unsupported axis length " + std::to_string(n));
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
void pass_x2(vr_ctx* ctx, double* spec, int dir) {
    const GridDims& g = ctx->g;
    auto* s = reinterpret_cast<double2*>(spec);
    MultDev none{};
    if (dir < 0)
        launch_axis<-1, 0>(ctx, g.n2, s, s, g.nh, g.L, (long long)g.n2 * g.nh, ctx->fft->tw2, none);
    else
        launch_axis<+1, 0>(ctx, g.n2, s, s, g.nh, g.L, (long long)g.n2 * g.nh, ctx->fft->tw2, none);
}
namespace {
int ilog2(int v) {
    int s = 0;
    while ((1 << s) < v) ++s;
    return s;
}
}  // namespace
// x1 slabs: forward x2 pass of the slab spectrum [L][n2][nh], stored straight into the
// all-to-all send layout (block q = [L][n2s][nh], the k2 rows of rank q)
void pass_x2_to_blocks(vr_ctx* ctx, const double* slab, double* send) {
    const GridDims& g = ctx->g;
    const auto* s = reinterpret_cast<const double2*>(slab);
    auto* d = reinterpret_cast<double2*>(send);
    MultDev none{};
    const long long blk = static_cast<long long>(g.L) * g.n2s * g.nh;
    const int sh = ilog2(g.n2s);
    switch (g.n2) {
#define VR_CASE(NN)                                                                                  \
    case NN:                                                                                         \
        launch_axis_t<NN, -1, 0, true>(ctx, s, d, g.nh, g.L, (long long)g.n2 * g.nh, ctx->fft->tw2, none, \
                                       RowGroups{}, sh, blk);                                       \
        break;
        VR_CASE(4)
        VR_CASE(8)
        VR_CASE(16)
        VR_CASE(32)
        VR_CASE(64)
        VR_CASE(128)
        VR_CASE(256)
        VR_CASE(512)
        VR_CASE(1024)
#undef VR_CASE
        default: throw_dimension("fft: unsupported axis length " + std::to_string(g.n2));
    }
}
// x1 slabs: inverse x2 pass reading the all-to-all receive layout (block q = [L][n2s][nh] from
// rank q) through a tensor map whose row groups are the peer blocks, into the slab [L][n2][nh]
void pass_x2_from_blocks(vr_ctx* ctx, const double* recv, double* slab) {
    const GridDims& g = ctx->g;
    const auto* s = reinterpret_cast<const double2*>(recv);
    auto* d = reinterpret_cast<double2*>(slab);
    MultDev none{};
    const long long blk = static_cast<long long>(g.L) * g.n2s * g.nh;
    const RowGroups rg{g.n2s, blk, static_cast<long long>(g.n2s) * g.nh};
    switch (g.n2) {
#define VR_CASE(NN)                                                                                   \
    case NN:                                                                                          \
        launch_axis_t<NN, +1, 0>(ctx, s, d, g.nh, g.L, (long long)g.n2 * g.nh, ctx->fft->tw2, none, rg);  \
        break;
        VR_CASE(4)
        VR_CASE(8)
        VR_CASE(16)
        VR_CASE(32)
        VR_CASE(64)
        VR_CASE(128)
        VR_CASE(256)
        VR_CASE(512)
        VR_CASE(1024)
#undef VR_CASE
        default: throw_dimension("fft: unsupported axis length " + std::to_string(g.n2));
    }
}
void pass_x1(vr_ctx* ctx, const double* src, double* dst, int dir, const MultParams* mult) {
    const GridDims& g = ctx->g;
    const auto* s = reinterpret_cast<const double2*>(src);
    auto* d = reinterpret_cast<double2*>(dst);
    const long long inner = (long long)g.n2s * g.nh;
    MultDev none{};
    if (mult && mult->kind == Mult::reg)
        launch_axis<-1, 3>(ctx, g.n1, s, d, inner, 1, 0, ctx->fft->tw1, to_dev(*mult));
    else if (mult)
        launch_axis<-1, 1>(ctx, g.n1, s, d, inner, 1, 0, ctx->fft->tw1, to_dev(*mult));
    else if (dir < 0)
        launch_axis<-1, 0>(ctx, g.n1, s, d, inner, 1, 0, ctx->fft->tw1, none);
    else
        launch_axis<+1, 0>(ctx, g.n1, s, d, inner, 1, 0, ctx->fft->tw1, none);
}
// d f / d x_axis of a real field on one GPU, one axis only: the derivative is a
// 1D spectral operator along that axis (the other axes' transforms cancel), so x1
// and x2 are one fused pass over f viewed as complex pairs and x3 is a row
// r2c -> i k3 -> c2r round trip (spec: scratch of NC complex)
void deriv_axis(vr_ctx* ctx, int axis, const double* f, double* out, double* spec) {
    const GridDims& g = ctx->g;
    const auto* s = reinterpret_cast<const double2*>(f);
    auto* d = reinterpret_cast<double2*>(out);
    const long long h3 = g.n3 / 2;
    MultDev m{};
    if (axis == 0) {
        m.beta = 1.0 / g.n1;
        launch_axis<-1, 2>(ctx, g.n1, s, d, static_cast<long long>(g.n2) * h3, 1, 0, ctx->fft->tw1, m);
    } else if (axis == 1) {
        m.beta = 1.0 / g.n2;
        launch_axis<-1, 2>(ctx, g.n2, s, d, h3, g.L, static_cast<long long>(g.n2) * h3, ctx->fft->tw2,
                           m);
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
