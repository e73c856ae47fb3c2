// fft_core.cuh -- shared by fft.cu (row passes, elementwise spectral kernels) and fft_axis.cu
// (strided x1 / x2 passes): complex helpers, the in-register radix networks and the Stockham
// stage driver, the spectral multipliers, and the TMA / mbarrier helpers of the tile pipelines.
// Everything lives in an anonymous namespace (one copy per translation unit); the two files
// are split only so that their template instantiations compile in parallel.
#pragma once
#include <cuda.h>  // CUtensorMap types; cuTensorMapEncodeTiled is resolved at run time (no -lcuda)

#include <cmath>
#include <string>
#include <type_traits>

#include "vr_common.cuh"

namespace vr {

struct FftPlan {
    double2* tw1 = nullptr;   // exp(2 pi i k / n1), k < n1 (cos, sin)
    double2* tw2 = nullptr;   // n2
    double2* tw3h = nullptr;  // n3 / 2
    double2* tw3 = nullptr;   // n3
};

// d f / d x_axis for axis 0 / 1 on one GPU: one fused strided pass (fft_axis.cu)
void deriv_axis_strided(vr_ctx* ctx, int axis, const double* f, double* out);

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

// largest in-register radix of this translation unit (elements per thread per stage)
#ifndef VR_FFT_RMAX
#define VR_FFT_RMAX 16
#endif
__host__ __device__ constexpr int rmax_of(int n) { return n < VR_FFT_RMAX ? n : VR_FFT_RMAX; }

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
        const bool last = rem <= VR_FFT_RMAX;
        const int R = rem >= VR_FFT_RMAX ? VR_FFT_RMAX : rem;
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
        if constexpr (N >= 16 && VR_FFT_RMAX >= 16) { VR_STAGE(16) }
        if constexpr (N >= 8 && VR_FFT_RMAX >= 8) { VR_STAGE(8) }
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

// MultParams -> the POD the kernels take
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

}  // namespace
}  // namespace vr
