// fft_axis.cuh -- the strided-pass kernel template and its launcher, shared by fft_axis.cu
// (plain transforms, slab variants) and fft_axis_fused.cu (fused x1 multiplier / derivative
// passes): two translation units so that their instantiations compile in parallel.
#pragma once
#ifdef VR_AXIS_RMAX  // tuning: a smaller radix for the strided passes only (more threads per column)
#define VR_FFT_RMAX VR_AXIS_RMAX
#endif
#include "fft_core.cuh"

namespace vr {

// the fused x1 passes (fft_axis_fused.cu): forward -> multiplier -> inverse
void pass_x1_mult(vr_ctx* ctx, const double* src, double* dst, const MultParams& mult);

namespace {

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

}  // namespace
}  // namespace vr
