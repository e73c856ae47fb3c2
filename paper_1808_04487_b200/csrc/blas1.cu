// blas1.cu -- fused pointwise updates and deterministic reductions.
//
// Replaces the reference's BLAS-1 layer (proj/include/veloreg/field_ops.hpp:14-111)
// and its deterministic 64-chunk CPU reductions (parallel.hpp:68-97). Here the
// reduction order is fixed by a constant grid of kRedBlocks blocks with a
// shuffle tree per block and an ordered final pass, so results are bitwise
// reproducible run to run (though not bitwise equal to the CPU chunk order).
#include <cfloat>

#include <chrono>

#include "vr_common.cuh"

namespace vr {
namespace {

__global__ void k_scale(double* __restrict__ x, long long n, double a) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        x[i] = x[i] * a;
}
__global__ void k_add_scaled(double* __restrict__ y, double a, const double* __restrict__ x,
                             long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = y[i] + a * x[i];
}
// out may alias x or y (elementwise)
__global__ void k_lin_comb(double* out, double a, const double* x, double b, const double* y,
                           long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = a * x[i] + b * y[i];
}
__global__ void k_affine(const double* __restrict__ x, double* __restrict__ out, long long n,
                         double lo, double s) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = (x[i] - lo) * s;
}

enum class RedOp { dot, sum, sumsq_diff, maxabs, maxmag2, nonfinite, minval, maxval };

template <RedOp OP>
__device__ __forceinline__ double red_term(const double* a, const double* b, long long i,
                                           long long n) {
    if constexpr (OP == RedOp::dot) return a[i] * b[i];
    if constexpr (OP == RedOp::sum) return a[i];
    if constexpr (OP == RedOp::sumsq_diff) {
        double d = a[i] - b[i];
        return d * d;
    }
    if constexpr (OP == RedOp::maxabs) return fabs(a[i]);
    if constexpr (OP == RedOp::maxmag2) {
        double x = a[i], y = a[i + n], z = a[i + 2 * n];
        return x * x + y * y + z * z;
    }
    if constexpr (OP == RedOp::nonfinite) return isfinite(a[i]) ? 0.0 : 1.0;
    if constexpr (OP == RedOp::minval) return -a[i];
    if constexpr (OP == RedOp::maxval) return a[i];
    return 0.0;
}
template <RedOp OP>
constexpr bool is_max() {
    return OP == RedOp::maxabs || OP == RedOp::maxmag2 || OP == RedOp::minval ||
           OP == RedOp::maxval;
}

template <RedOp OP>
__device__ __forceinline__ double combine(double x, double y) {
    if constexpr (is_max<OP>()) return fmax(x, y);
    return x + y;
}

// grid (kRedBlocks, ncomp): component c reduces a + c*n, b + c*n
template <RedOp OP>
__global__ void __launch_bounds__(kRedThreads) k_reduce(const double* __restrict__ a,
                                                        const double* __restrict__ b, long long n,
                                                        double* __restrict__ partials) {
    const int c = blockIdx.y;
    const double* ac = a + (OP == RedOp::maxmag2 ? 0 : c * n);
    const double* bc = b ? b + c * n : nullptr;
    double acc = is_max<OP>() ? -1e300 : 0.0;
    for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < n;
         i += (long long)gridDim.x * kRedThreads)
        acc = combine<OP>(acc, red_term<OP>(ac, bc, i, n));
    __shared__ double sh[kRedThreads / 32];
    for (int o = 16; o > 0; o >>= 1) acc = combine<OP>(acc, __shfl_down_sync(0xffffffffu, acc, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = sh[0];
        for (int w = 1; w < kRedThreads / 32; ++w) s = combine<OP>(s, sh[w]);
        partials[c * gridDim.x + blockIdx.x] = s;
    }
}

// one block per component: ordered sum of nblocks partials
template <bool MAX>
__global__ void k_finalize(const double* __restrict__ partials, int nblocks,
                           double* __restrict__ out) {
    const int c = blockIdx.x;
    double acc = MAX ? -1e300 : 0.0;
    for (int i = threadIdx.x; i < nblocks; i += blockDim.x) {
        double v = partials[c * nblocks + i];
        acc = MAX ? fmax(acc, v) : acc + v;
    }
    __shared__ double sh[32];
    for (int o = 16; o > 0; o >>= 1) {
        double v = __shfl_down_sync(0xffffffffu, acc, o);
        acc = MAX ? fmax(acc, v) : acc + v;
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = sh[0];
        for (int w = 1; w < (int)(blockDim.x / 32); ++w) s = MAX ? fmax(s, sh[w]) : s + sh[w];
        out[c] = s;
    }
}

template <RedOp OP>
void reduce(vr_ctx* ctx, const double* a, const double* b, long long n, int ncomp,
            double* host_out) {
    const int nb = static_cast<int>(std::min<long long>(kRedBlocks, (n + kRedThreads - 1) / kRedThreads));
    VR_LAUNCH(ctx, "reduce", k_reduce<OP><<<dim3(nb, ncomp), kRedThreads, 0, ctx->stream>>>(a, b, n, ctx->red_partials));
    VR_LAUNCH(ctx, "reduce", k_finalize<is_max<OP>()><<<ncomp, 256, 0, ctx->stream>>>(ctx->red_partials, nb, ctx->red_out););
    VR_CUDA(cudaMemcpyAsync(ctx->red_host, ctx->red_out, sizeof(double) * ncomp,
                            cudaMemcpyDeviceToHost, ctx->stream));
    flags_enqueue_copy(ctx);  // deferred matvec flags ride on this synchronisation
    {
        const auto t0 = std::chrono::steady_clock::now();
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        if (timing_enabled())
            slow_op("reduce sync", std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    for (int c = 0; c < ncomp; ++c) host_out[c] = ctx->red_host[c];
    if (ctx->dist) ctx->dist->allreduce(ctx, host_out, ncomp, is_max<OP>());  // rank order
    flags_after_sync(ctx);
}

unsigned ew_grid(long long n) {
    return static_cast<unsigned>(std::min<long long>((n + 255) / 256, 148LL * 16));
}

template <bool MAX>
__device__ __forceinline__ double block_reduce(double acc) {
    __shared__ double sh[kRedThreads / 32];
    for (int o = 16; o > 0; o >>= 1) {
        const double v = __shfl_down_sync(0xffffffffu, acc, o);
        acc = MAX ? fmax(acc, v) : acc + v;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        s = sh[0];
        for (int w = 1; w < kRedThreads / 32; ++w) s = MAX ? fmax(s, sh[w]) : s + sh[w];
    }
    return s;
}

// PCG residual update (solver.cpp:83-86) fused with the next norm: per
// component c (grid.y): x += kappa s; r = r + (-kappa) Hs; partial sums of r.r
// and of r (for the zero-mode projection of the regularization recurrence).
// partials layout: [(2c + q) * gridDim.x + block], q = 0: r.r, q = 1: sum r
__global__ void __launch_bounds__(kRedThreads)
    k_pcg_update(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ s,
                 const double* __restrict__ Hs, double kappa, long long n,
                 double* __restrict__ partials) {
    const long long off = blockIdx.y * n;
    double rr = 0.0, rs = 0.0;
    for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < n;
         i += (long long)gridDim.x * kRedThreads) {
        const long long k = off + i;
        x[k] = x[k] + kappa * s[k];
        const double rv = r[k] + (-kappa) * Hs[k];
        r[k] = rv;
        rr += rv * rv;
        rs += rv;
    }
    const double a = block_reduce<false>(rr);
    const double b = block_reduce<false>(rs);
    if (threadIdx.x == 0) {
        partials[(2 * blockIdx.y + 0) * gridDim.x + blockIdx.x] = a;
        partials[(2 * blockIdx.y + 1) * gridDim.x + blockIdx.x] = b;
    }
}

// PCG direction update (solver.cpp:96-97) plus the regularization recurrence:
// s = 1.0 z + mu s ;  u = 1.0 (r - mean_c(r)) + mu u  (u tracks beta_v A s)
__global__ void k_pcg_direction(double* __restrict__ s, double* __restrict__ u,
                                const double* __restrict__ z, const double* __restrict__ r,
                                double mu, double m0, double m1, double m2, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < 3 * n;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = static_cast<int>(i / n);
        const double m = c == 0 ? m0 : (c == 1 ? m1 : m2);
        if (s) s[i] = 1.0 * z[i] + mu * s[i];
        if (u) u[i] = mu == 0.0 ? r[i] - m : 1.0 * (r[i] - m) + mu * u[i];
    }
}

}  // namespace

void pcg_update(vr_ctx* ctx, double* x, double* r, const double* s, const double* Hs, double kappa,
                double* rr, double* rsum) {
    const long long n = ctx->g.N;
    const int nb = static_cast<int>(std::min<long long>(kRedBlocks, (n + kRedThreads - 1) / kRedThreads));
    VR_LAUNCH(ctx, "blas1", k_pcg_update<<<dim3(nb, 3), kRedThreads, 0, ctx->stream>>>(x, r, s, Hs, kappa, n, ctx->red_partials));
    double out[6];
    finalize_sums(ctx, nb, 6, out);
    for (int c = 0; c < 3; ++c) {
        rr[c] = out[2 * c];
        rsum[c] = out[2 * c + 1];
    }
}

void pcg_direction(vr_ctx* ctx, double* s, double* u, const double* z, const double* r, double mu,
                   const double mean[3]) {
    const long long n = ctx->g.N;
    VR_LAUNCH(ctx, "blas1", k_pcg_direction<<<ew_grid(3 * n), 256, 0, ctx->stream>>>(s, u, z, r, mu, mean[0], mean[1], mean[2], n));
}

void scale(vr_ctx* ctx, double* x, long long n, double a) {
    VR_LAUNCH(ctx, "blas1", k_scale<<<ew_grid(n), 256, 0, ctx->stream>>>(x, n, a););
}
void add_scaled(vr_ctx* ctx, double* y, double a, const double* x, long long n) {
    VR_LAUNCH(ctx, "blas1", k_add_scaled<<<ew_grid(n), 256, 0, ctx->stream>>>(y, a, x, n););
}
void lin_comb(vr_ctx* ctx, double* out, double a, const double* x, double b, const double* y,
              long long n) {
    VR_LAUNCH(ctx, "blas1", k_lin_comb<<<ew_grid(n), 256, 0, ctx->stream>>>(out, a, x, b, y, n););
}
void affine(vr_ctx* ctx, const double* x, double* out, long long n, double lo, double s) {
    VR_LAUNCH(ctx, "blas1", k_affine<<<ew_grid(n), 256, 0, ctx->stream>>>(x, out, n, lo, s););
}
void dot_components(vr_ctx* ctx, const double* a, const double* b, long long n, int ncomp,
                    double* results) {
    reduce<RedOp::dot>(ctx, a, b, n, ncomp, results);
}
void sum_components(vr_ctx* ctx, const double* a, long long n, int ncomp, double* results) {
    reduce<RedOp::sum>(ctx, a, nullptr, n, ncomp, results);
}
double max_abs(vr_ctx* ctx, const double* a, long long n) {
    if (n == 0) return 0.0;
    double r;
    reduce<RedOp::maxabs>(ctx, a, nullptr, n, 1, &r);
    return r;
}
double max_magnitude(vr_ctx* ctx, const double* v3, long long n) {
    double r;
    reduce<RedOp::maxmag2>(ctx, v3, nullptr, n, 1, &r);
    return std::sqrt(r);
}
bool all_finite(vr_ctx* ctx, const double* a, long long n) {
    double r;
    reduce<RedOp::nonfinite>(ctx, a, nullptr, n, 1, &r);
    return r == 0.0;
}
double sum_sq_diff(vr_ctx* ctx, const double* a, const double* b, long long n) {
    double r;
    reduce<RedOp::sumsq_diff>(ctx, a, b, n, 1, &r);
    return r;
}
double min_value(vr_ctx* ctx, const double* a, long long n) {
    double r;
    reduce<RedOp::minval>(ctx, a, nullptr, n, 1, &r);
    return -r;
}
double max_value(vr_ctx* ctx, const double* a, long long n) {
    double r;
    reduce<RedOp::maxval>(ctx, a, nullptr, n, 1, &r);
    return r;
}
void finalize_sums(vr_ctx* ctx, int nblocks, int ncomp, double* host_out) {
    VR_LAUNCH(ctx, "blas1", k_finalize<false><<<ncomp, 256, 0, ctx->stream>>>(ctx->red_partials, nblocks, ctx->red_out););
    VR_CUDA(cudaMemcpyAsync(ctx->red_host, ctx->red_out, sizeof(double) * ncomp,
                            cudaMemcpyDeviceToHost, ctx->stream));
    flags_enqueue_copy(ctx);
    VR_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int c = 0; c < ncomp; ++c) host_out[c] = ctx->red_host[c];
    if (ctx->dist) ctx->dist->allreduce(ctx, host_out, ncomp, false);
    flags_after_sync(ctx);
}

}  // namespace vr
