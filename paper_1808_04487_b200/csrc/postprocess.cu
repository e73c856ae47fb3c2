// postprocess.cu -- deformation measures, label transport and overlap scores
// (the reference's postprocess module, proj/src/postprocess.cpp:13-167) and the
// outer continuation loops (grid / scale continuation, beta search) that SPEC.md
// describes but the reference code does not implement.
//
// Everything here is a composition of the sm_100a transport / spectral kernels
// (sl.cu, fft.cu) plus a few pointwise and counting kernels; reductions use a
// fixed grid and an ordered host combine (run-to-run reproducible); label counts
// are integer atomics (exact).
#include <algorithm>
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "objective.cuh"
#include "twolevel.cuh"

namespace vr {
namespace {

constexpr int kT = 256;

unsigned blocks_for(long long n) { return grid_1d(n, kT); }

__global__ void k_fill(double* __restrict__ x, long long n, double v) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i < n) x[i] = v;
}

// y_c = wrap_coord(x_c + u_c) (postprocess.cpp:50-59)
__global__ void k_absolute_map(const double* __restrict__ u, long long ustride, double* __restrict__ y,
                               GridDims g) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i >= g.N) return;
    long long r = i;
    const int i3 = static_cast<int>(r % g.n3);
    r /= g.n3;
    const int i2 = static_cast<int>(r % g.n2);
    const int i1 = static_cast<int>(r / g.n2);
    const double x[3] = {g.h1 * (g.off1 + i1), g.h2 * i2, g.h3 * i3};  // off1: slab origin
#pragma unroll
    for (int c = 0; c < 3; ++c) y[c * g.N + i] = wrap_coord(x[c] + u[c * ustride + i]);
}

// det_stats partials (postprocess.cpp:62-81): per block {min, max, sum, count}
// over the foreground (fg == null: everywhere); fixed grid of kRedBlocks
__global__ void __launch_bounds__(kRedThreads)
    k_det_partials(const double* __restrict__ det, const double* __restrict__ fg, double thr,
                   long long n, double* __restrict__ partials) {
    double mn = 1e300, mx = -1e300, sum = 0.0, cnt = 0.0;
    for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < n;
         i += (long long)gridDim.x * kRedThreads) {
        if (fg && fg[i] < thr) continue;
        const double d = det[i];
        mn = fmin(mn, d);
        mx = fmax(mx, d);
        sum += d;
        cnt += 1.0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
        sum += __shfl_down_sync(0xffffffffu, sum, o);
        cnt += __shfl_down_sync(0xffffffffu, cnt, o);
    }
    __shared__ double sh[4][kRedThreads / 32];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sh[0][w] = mn, sh[1][w] = mx, sh[2][w] = sum, sh[3][w] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < kRedThreads / 32; ++q) {
            mn = fmin(mn, sh[0][q]);
            mx = fmax(mx, sh[1][q]);
            sum += sh[2][q];
            cnt += sh[3][q];
        }
        double* p = partials + 4 * blockIdx.x;
        p[0] = mn, p[1] = mx, p[2] = sum, p[3] = cnt;
    }
}

// label code of a voxel: std::lround (postprocess.cpp:89, :126)
__device__ __forceinline__ long long code_of(double x) { return llround(x); }

// per block min / max code over a (and b when given)
__global__ void __launch_bounds__(kRedThreads)
    k_code_range(const double* __restrict__ a, const double* __restrict__ b, long long n,
                 double* __restrict__ partials) {
    double mn = 1e300, mx = -1e300;
    for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < n;
         i += (long long)gridDim.x * kRedThreads) {
        double c = static_cast<double>(code_of(a[i]));
        mn = fmin(mn, c), mx = fmax(mx, c);
        if (b) {
            c = static_cast<double>(code_of(b[i]));
            mn = fmin(mn, c), mx = fmax(mx, c);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    }
    __shared__ double sh[2][kRedThreads / 32];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sh[0][w] = mn, sh[1][w] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < kRedThreads / 32; ++q) mn = fmin(mn, sh[0][q]), mx = fmax(mx, sh[1][q]);
        partials[2 * blockIdx.x] = mn;
        partials[2 * blockIdx.x + 1] = mx;
    }
}

__global__ void k_code_mark(const double* __restrict__ a, long long n, long long cmin,
                            int* __restrict__ present) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i < n) present[code_of(a[i]) - cmin] = 1;
}

// binarised label (postprocess.cpp:101-104)
__global__ void k_label_mask(const double* __restrict__ labels, long long n, long long code,
                             double* __restrict__ mask) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i < n) mask[i] = code_of(labels[i]) == code ? 1.0 : 0.0;
}

// strongest response wins, exact ties keep the lower (earlier) code (postprocess.cpp:110-116)
__global__ void k_label_update(const double* __restrict__ mask, double* __restrict__ best,
                               double* __restrict__ out, long long n, double code) {
    const long long i = blockIdx.x * (long long)kT + threadIdx.x;
    if (i >= n) return;
    const double m = mask[i];
    if (m >= 0.5 && (out[i] == 0.0 || m > best[i])) {
        best[i] = m;
        out[i] = code;
    }
}

// overlap counts (postprocess.cpp:137-150): slot(code) from a dense table over
// [cmin, cmax]; counts[3 s + {0,1,2}] = |A_s|, |B_s|, |A_s & B_s|; the union in the
// last three. Block-local shared counters when the slots fit.
constexpr int kSmemSlots = 1024;
__global__ void __launch_bounds__(kT)
    k_overlap_counts(const double* __restrict__ ref, const double* __restrict__ test,
                     const double* __restrict__ mask, long long n, long long cmin,
                     const int* __restrict__ slot, int nslots,
                     unsigned long long* __restrict__ counts) {
    __shared__ unsigned int sc[3 * (kSmemSlots + 1)];
    const bool local = nslots <= kSmemSlots;
    if (local)
        for (int q = threadIdx.x; q < 3 * (nslots + 1); q += kT) sc[q] = 0;
    __syncthreads();
    for (long long i = blockIdx.x * (long long)kT + threadIdx.x; i < n;
         i += (long long)gridDim.x * kT) {
        if (mask && mask[i] < 0.5) continue;
        const long long a = code_of(ref[i]), b = code_of(test[i]);
        const int sa = a != 0 ? slot[a - cmin] : -1, sb = b != 0 ? slot[b - cmin] : -1;
        const int u = 3 * nslots;
        if (local) {
            if (sa >= 0) atomicAdd(&sc[3 * sa], 1u);
            if (sb >= 0) atomicAdd(&sc[3 * sb + 1], 1u);
            if (sa >= 0 && a == b) atomicAdd(&sc[3 * sa + 2], 1u);
            if (sa >= 0) atomicAdd(&sc[u], 1u);
            if (sb >= 0) atomicAdd(&sc[u + 1], 1u);
            if (sa >= 0 && sb >= 0) atomicAdd(&sc[u + 2], 1u);
        } else {
            if (sa >= 0) atomicAdd(&counts[3 * sa], 1ull);
            if (sb >= 0) atomicAdd(&counts[3 * sb + 1], 1ull);
            if (sa >= 0 && a == b) atomicAdd(&counts[3 * sa + 2], 1ull);
            if (sa >= 0) atomicAdd(&counts[u], 1ull);
            if (sb >= 0) atomicAdd(&counts[u + 1], 1ull);
            if (sa >= 0 && sb >= 0) atomicAdd(&counts[u + 2], 1ull);
        }
    }
    if (!local) return;
    __syncthreads();
    for (int q = threadIdx.x; q < 3 * (nslots + 1); q += kT)
        if (sc[q]) atomicAdd(&counts[q], static_cast<unsigned long long>(sc[q]));
}

// device buffer freed at scope exit (stream-ordered)
struct DevBuf {
    vr_ctx* ctx;
    double* p;
    DevBuf(vr_ctx* c, long long n) : ctx(c), p(dev_alloc(c, n)) {}
    ~DevBuf() { dev_free(ctx, p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

void check_velocity(vr_ctx* ctx, const double* v3, int nt) {
    if (nt < 1) throw_argument("trace_characteristics: n_t must be >= 1");
    if (!all_finite(ctx, v3, 3 * ctx->g.N))
        throw_numeric("trace_characteristics: velocity has non-finite values");
}

void gaussian(vr_ctx* ctx, const double* in, double* out, double sigma_voxels) {
    MultParams mp;
    mp.kind = Mult::gaussian;
    const double h[3] = {ctx->g.h1, ctx->g.h2, ctx->g.h3};
    for (int a = 0; a < 3; ++a) mp.sig2h2[a] = sigma_voxels * sigma_voxels * h[a] * h[a];
    spectral_scalar_op(ctx, in, out, mp);
}

// sorted distinct nonzero codes of a (and b) via a presence table over [cmin, cmax]
std::vector<long long> label_codes(vr_ctx* ctx, const double* a, const double* b,
                                   long long& cmin, std::vector<int>& present) {
    const long long N = ctx->g.N;
    VR_LAUNCH(ctx, "pp_labels", k_code_range<<<kRedBlocks, kRedThreads, 0, ctx->stream>>>(a, b, N, ctx->red_partials));
    std::vector<double> part(2 * kRedBlocks);
    VR_CUDA(cudaMemcpyAsync(part.data(), ctx->red_partials, sizeof(double) * part.size(),
                            cudaMemcpyDeviceToHost, ctx->stream));
    VR_CUDA(cudaStreamSynchronize(ctx->stream));
    double mn = 1e300, mx = -1e300;
    for (int q = 0; q < kRedBlocks; ++q) mn = std::min(mn, part[2 * q]), mx = std::max(mx, part[2 * q + 1]);
    if (ctx->dist) {  // the code range of all ranks
        double mm[2] = {-mn, mx};
        ctx->dist->allreduce(ctx, mm, 2, true);
        mn = -mm[0], mx = mm[1];
        if (!(mx - mn < static_cast<double>(1 << 20)))
            throw_argument("label codes must span fewer than 2^20 values on x1 slabs");
    }
    if (!(mx - mn < static_cast<double>(1 << 24)))
        throw_argument("label codes must span fewer than 2^24 values");
    cmin = static_cast<long long>(mn);
    const long long range = static_cast<long long>(mx) - cmin + 1;
    int* dp = nullptr;
    VR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dp), sizeof(int) * range, ctx->stream));
    VR_CUDA(cudaMemsetAsync(dp, 0, sizeof(int) * range, ctx->stream));
    VR_LAUNCH(ctx, "pp_labels", k_code_mark<<<blocks_for(N), kT, 0, ctx->stream>>>(a, N, cmin, dp));
    if (b) VR_LAUNCH(ctx, "pp_labels", k_code_mark<<<blocks_for(N), kT, 0, ctx->stream>>>(b, N, cmin, dp));
    present.assign(range, 0);
    VR_CUDA(cudaMemcpyAsync(present.data(), dp, sizeof(int) * range, cudaMemcpyDeviceToHost,
                            ctx->stream));
    VR_CUDA(cudaFreeAsync(dp, ctx->stream));
    VR_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->dist) {  // a code is present if any rank holds it
        std::vector<double> pd(present.begin(), present.end());
        ctx->dist->allreduce(ctx, pd.data(), static_cast<int>(pd.size()), true);
        for (size_t q = 0; q < pd.size(); ++q) present[q] = pd[q] != 0.0;
    }
    std::vector<long long> codes;
    for (long long q = 0; q < range; ++q)
        if (present[q] && q + cmin != 0) codes.push_back(q + cmin);
    return codes;
}

vr_overlap score(unsigned long long a, unsigned long long b, unsigned long long both) {
    vr_overlap s;  // postprocess.cpp:152-158
    s.dice = (a + b) == 0 ? 1.0 : 2.0 * static_cast<double>(both) / static_cast<double>(a + b);
    s.false_positive_rate = b == 0 ? 0.0 : static_cast<double>(b - both) / static_cast<double>(b);
    s.false_negative_rate = a == 0 ? 0.0 : static_cast<double>(a - both) / static_cast<double>(a);
    return s;
}


// x1 slabs: the halo-padded gather copy of v (3 components, stride hstride) with exchanged
// halos, after the same halo check as objective_evaluate. One GPU: v itself.
struct GatherVelocity {
    std::unique_ptr<DevBuf> pad;
    const double* v = nullptr;   // component 0 (interior)
    long long stride = 0;
    GatherVelocity(vr_ctx* ctx, const double* v3, int nt, const char* what) {
        const long long N = ctx->g.N;
        if (!ctx->dist) {
            v = v3, stride = N;
            return;
        }
        const int need = halo_required(max_abs(ctx, v3, N), nt, ctx->g.n1);
        if (need > ctx->g.halo)
            throw_resource(std::string(what) + ": x1 displacement needs a halo of " + std::to_string(need) +
                           " planes, ctx has " + std::to_string(ctx->g.halo));
        pad.reset(new DevBuf(ctx, 3 * ctx->hstride));
        for (int c = 0; c < 3; ++c) {
            VR_CUDA(cudaMemcpyAsync(pslice(ctx, pad->p, c), v3 + c * N, sizeof(double) * N,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
            exchange(ctx, pslice(ctx, pad->p, c));
        }
        v = pslice(ctx, pad->p, 0), stride = ctx->hstride;
    }
};
void begin_flags(vr_ctx* ctx) {
    drain_flags(ctx);
    VR_CUDA(cudaMemsetAsync(ctx->flag_dev, 0, 2 * sizeof(int), ctx->stream));
}

}  // namespace

// det_deformation_gradient (postprocess.cpp:13-29): continuity transport of 1 along the
// backward characteristics with the factor of -div v. On x1 slabs every gather source
// (div v, the two transport buffers) is halo-padded and exchanged before its step.
void det_deformation_gradient(vr_ctx* ctx, const double* v3, int nt, double* det) {
    const long long N = ctx->g.N, H = ctx->hstride;
    check_velocity(ctx, v3, nt);
    begin_flags(ctx);
    GatherVelocity gv(ctx, v3, nt, "det_deformation_gradient");
    DevBuf xb(ctx, 3 * N), div(ctx, H), factor(ctx, N), work(ctx, 2 * H);
    sl_trace(ctx, gv.v, gv.stride, nt, VR_TRACE_BACKWARD, xb.p);
    double* divi = pslice(ctx, div.p, 0);
    op_divergence(ctx, v3, divi);
    scale(ctx, divi, N, -1.0);
    exchange(ctx, divi);
    sl_factor(ctx, divi, xb.p, 0.5 / nt, factor.p);
    double* buf[2] = {pslice(ctx, work.p, 0), pslice(ctx, work.p, 1)};
    VR_LAUNCH(ctx, "pp_pointwise", k_fill<<<blocks_for(N), kT, 0, ctx->stream>>>(buf[0], N, 1.0));
    for (int j = 0; j < nt; ++j) {
        exchange(ctx, buf[j & 1]);
        sl_continuity(ctx, buf[j & 1], xb.p, factor.p, buf[(j + 1) & 1]);
    }
    VR_CUDA(cudaMemcpyAsync(det, buf[nt & 1], sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
    if (ctx->dist) check_flags(ctx, "det_deformation_gradient");
}

// deformation_map (postprocess.cpp:31-60)
void deformation_map(vr_ctx* ctx, const double* v3, int nt, bool absolute, double* out3) {
    const long long N = ctx->g.N, H = ctx->hstride;
    check_velocity(ctx, v3, nt);
    begin_flags(ctx);
    GatherVelocity gv(ctx, v3, nt, "deformation_map");
    DevBuf xb(ctx, 3 * N), vdep(ctx, 3 * N), u(ctx, 3 * H), w(ctx, 3 * H);
    sl_trace(ctx, gv.v, gv.stride, nt, VR_TRACE_BACKWARD, xb.p);
    if (ctx->dist) {
        for (int c = 0; c < 3; ++c) sl_tricubic(ctx, gv.v + c * gv.stride, 1, xb.p, vdep.p + c * N);
    } else {
        sl_tricubic(ctx, v3, 3, xb.p, vdep.p);
    }
    VR_CUDA(cudaMemsetAsync(u.p, 0, sizeof(double) * 3 * H, ctx->stream));
    double* cur = pslice(ctx, u.p, 0);  // component c at + c * hstride
    double* nxt = pslice(ctx, w.p, 0);
    for (int j = 0; j < nt; ++j) {
        if (j > 0)  // u = 0 needs no exchange
            for (int c = 0; c < 3; ++c) exchange(ctx, cur + c * H);
        sl_defmap_step(ctx, cur, xb.p, vdep.p, v3, 0.5 / nt, nxt);
        std::swap(cur, nxt);
    }
    if (absolute) {
        VR_LAUNCH(ctx, "pp_pointwise", k_absolute_map<<<blocks_for(N), kT, 0, ctx->stream>>>(cur, H, out3, ctx->g));
    } else {
        for (int c = 0; c < 3; ++c)
            VR_CUDA(cudaMemcpyAsync(out3 + c * N, cur + c * H, sizeof(double) * N, cudaMemcpyDeviceToDevice,
                                    ctx->stream));
    }
    if (ctx->dist) check_flags(ctx, "deformation_map");
}

// det_stats (postprocess.cpp:62-81); count == 0 -> all zero like DetStats{}
vr_det_summary det_stats(vr_ctx* ctx, const double* det, const double* fg, double threshold) {
    VR_LAUNCH(ctx, "pp_reduce", k_det_partials<<<kRedBlocks, kRedThreads, 0, ctx->stream>>>(det, fg, threshold, ctx->g.N, ctx->red_partials));
    std::vector<double> part(4 * kRedBlocks);
    VR_CUDA(cudaMemcpyAsync(part.data(), ctx->red_partials, sizeof(double) * part.size(),
                            cudaMemcpyDeviceToHost, ctx->stream));
    VR_CUDA(cudaStreamSynchronize(ctx->stream));
    double mn = 1e300, mx = -1e300, sum = 0.0, cnt = 0.0;
    for (int q = 0; q < kRedBlocks; ++q) {
        mn = std::min(mn, part[4 * q]);
        mx = std::max(mx, part[4 * q + 1]);
        sum += part[4 * q + 2];
        cnt += part[4 * q + 3];
    }
    if (ctx->dist) {  // min / max and sum / count over the ranks (rank-ordered sums)
        double mm[2] = {-mn, mx}, sc[2] = {sum, cnt};
        ctx->dist->allreduce(ctx, mm, 2, true);
        ctx->dist->allreduce(ctx, sc, 2, false);
        mn = -mm[0], mx = mm[1], sum = sc[0], cnt = sc[1];
    }
    vr_det_summary st{0.0, 0.0, 0.0};
    if (cnt == 0.0) return st;
    st.min = mn;
    st.max = mx;
    st.mean = sum / cnt;
    return st;
}

// transport_labels (postprocess.cpp:83-120)
void transport_labels(vr_ctx* ctx, const double* labels, const double* v3, int nt, double* out) {
    const long long N = ctx->g.N;
    long long cmin = 0;
    std::vector<int> present;
    const std::vector<long long> codes = label_codes(ctx, labels, nullptr, cmin, present);
    if (codes.size() > 64)
        throw_resource("transport_labels: more than 64 distinct labels (" +
                       std::to_string(codes.size()) + ")");
    check_velocity(ctx, v3, nt);
    begin_flags(ctx);
    GatherVelocity gv(ctx, v3, nt, "transport_labels");
    // mask / next are gather sources: halo-padded and exchanged before each step on x1 slabs
    DevBuf xb(ctx, 3 * N), best(ctx, N), work(ctx, 2 * ctx->hstride);
    sl_trace(ctx, gv.v, gv.stride, nt, VR_TRACE_BACKWARD, xb.p);
    VR_LAUNCH(ctx, "pp_pointwise", k_fill<<<blocks_for(N), kT, 0, ctx->stream>>>(out, N, 0.0));
    VR_LAUNCH(ctx, "pp_pointwise", k_fill<<<blocks_for(N), kT, 0, ctx->stream>>>(best.p, N, 0.0));
    for (long long code : codes) {
        double* cur = pslice(ctx, work.p, 0);
        double* nxt = pslice(ctx, work.p, 1);
        VR_LAUNCH(ctx, "pp_pointwise", k_label_mask<<<blocks_for(N), kT, 0, ctx->stream>>>(labels, N, code, cur));
        gaussian(ctx, cur, cur, 1.0);
        for (int j = 0; j < nt; ++j) {
            exchange(ctx, cur);
            sl_advect(ctx, cur, xb.p, nxt);
            std::swap(cur, nxt);
        }
        VR_LAUNCH(ctx, "pp_pointwise", k_label_update<<<blocks_for(N), kT, 0, ctx->stream>>>(cur, best.p, out, N, static_cast<double>(code)));
    }
    if (ctx->dist) check_flags(ctx, "transport_labels");
}

// overlap_scores (postprocess.cpp:122-165)
int overlap_scores(vr_ctx* ctx, const double* ref, const double* test, const double* mask,
                   int max_labels, int* codes_out, vr_overlap* per_label, vr_overlap* uni) {
    const long long N = ctx->g.N;
    long long cmin = 0;
    std::vector<int> present;
    const std::vector<long long> codes = label_codes(ctx, ref, test, cmin, present);
    const int ns = static_cast<int>(codes.size());
    std::vector<int> slot(present.size(), -1);
    for (int s = 0; s < ns; ++s) slot[codes[s] - cmin] = s;
    int* dslot = nullptr;
    unsigned long long* dcnt = nullptr;
    VR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dslot), sizeof(int) * slot.size(), ctx->stream));
    VR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dcnt), sizeof(unsigned long long) * 3 * (ns + 1),
                            ctx->stream));
    VR_CUDA(cudaMemcpyAsync(dslot, slot.data(), sizeof(int) * slot.size(), cudaMemcpyHostToDevice,
                            ctx->stream));
    VR_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long) * 3 * (ns + 1), ctx->stream));
    VR_LAUNCH(ctx, "pp_overlap", k_overlap_counts<<<std::min<long long>(blocks_for(N), 4LL * ctx->sms), kT, 0, ctx->stream>>>(ref, test, mask, N, cmin, dslot, ns, dcnt));
    std::vector<unsigned long long> cnt(3 * (ns + 1));
    VR_CUDA(cudaMemcpyAsync(cnt.data(), dcnt, sizeof(unsigned long long) * cnt.size(),
                            cudaMemcpyDeviceToHost, ctx->stream));
    VR_CUDA(cudaFreeAsync(dslot, ctx->stream));
    VR_CUDA(cudaFreeAsync(dcnt, ctx->stream));
    VR_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->dist) {  // voxel counts of all ranks (integers below 2^53: exact as doubles)
        std::vector<double> cd(cnt.begin(), cnt.end());
        ctx->dist->allreduce(ctx, cd.data(), static_cast<int>(cd.size()), false);
        for (size_t q = 0; q < cd.size(); ++q) cnt[q] = static_cast<unsigned long long>(cd[q]);
    }
    for (int s = 0; s < ns && s < max_labels; ++s) {
        if (codes_out) codes_out[s] = static_cast<int>(codes[s]);
        if (per_label) per_label[s] = score(cnt[3 * s], cnt[3 * s + 1], cnt[3 * s + 2]);
    }
    if (uni) *uni = score(cnt[3 * ns], cnt[3 * ns + 1], cnt[3 * ns + 2]);
    return ns;
}

// ---------------------------------------------------------------------------
// Continuation. Levels append their SolveReports / records.

// grid continuation: n_levels grids halving every axis per level
// (coarsest >= 16 per axis); level images = spectral restriction of the originals,
// then gaussian_smooth with sigma = 1 voxel of that level; the finest level solves
// on the original images; the velocity is spectrally prolonged between levels.
std::vector<GnResult> grid_continuation(vr_ctx* ctx, const double* mR, const double* mT,
                                        const double* v0, const vr_model& model,
                                        const vr_solver_params& params, int precond,
                                        int n_levels, double* v_out) {
    if (n_levels < 1) throw_argument("grid continuation: at least one level");
    const int d[3] = {ctx->g.n1, ctx->g.n2, ctx->g.n3};
    for (int a = 0; a < 3; ++a)
        if ((d[a] >> (n_levels - 1)) < 16 || (d[a] % (1 << (n_levels - 1))) != 0)
            throw_argument("grid continuation: the coarsest level must keep >= 16 points per axis");
    const long long N = ctx->g.N;
    std::vector<vr_ctx*> lv(n_levels, nullptr);
    std::vector<GnResult> out;
    {
        lv[n_levels - 1] = ctx;
        for (int l = 0; l + 1 < n_levels; ++l) {
            const int s = n_levels - 1 - l;
            lv[l] = ctx_sibling(ctx, d[0] >> s, d[1] >> s, d[2] >> s);  // owned by ctx
        }
        // initial guess restricted to the coarsest level
        DevBuf v(lv[0], 3 * lv[0]->g.N);
        if (n_levels == 1)
            VR_CUDA(cudaMemcpyAsync(v.p, v0, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
        else
            for (int c = 0; c < 3; ++c) resample_scalar(ctx, v0 + c * N, lv[0], v.p + c * lv[0]->g.N);
        std::unique_ptr<DevBuf> vcur;
        const double* vin = v.p;
        for (int l = 0; l < n_levels; ++l) {
            vr_ctx* c = lv[l];
            const long long Nl = c->g.N;
            if (l + 1 < n_levels) {
                DevBuf R(c, Nl), T(c, Nl), vl(c, 3 * Nl);
                resample_scalar(ctx, mR, c, R.p);
                resample_scalar(ctx, mT, c, T.p);
                gaussian(c, R.p, R.p, 1.0);
                gaussian(c, T.p, T.p, 1.0);
                out.push_back(gauss_newton_solve(c, R.p, T.p, vin, model, params, precond, vl.p));
                if (out.back().report.stop == VR_STOP_LINE_SEARCH_FAILURE) {
                    // abort with partial results: this level's velocity on the finest grid
                    for (int q = 0; q < 3; ++q) resample_scalar(c, vl.p + q * Nl, ctx, v_out + q * N);
                    break;
                }
                vr_ctx* f = lv[l + 1];  // prolong to the next level
                auto nb = std::make_unique<DevBuf>(f, 3 * f->g.N);
                for (int q = 0; q < 3; ++q) resample_scalar(c, vl.p + q * Nl, f, nb->p + q * f->g.N);
                vcur = std::move(nb);
                vin = vcur->p;
            } else {
                out.push_back(gauss_newton_solve(ctx, mR, mT, vin, model, params, precond, v_out));
            }
        }
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return out;
}

// scale continuation: images re-smoothed from the originals per
// level (sigma in voxels; 0 = the originals), warm-started solves
std::vector<GnResult> scale_continuation(vr_ctx* ctx, const double* mR, const double* mT,
                                         const double* v0, const vr_model& model,
                                         const vr_solver_params& params, int precond,
                                         const double* sigmas, int n, double* v_out) {
    if (n < 1) throw_argument("scale continuation: at least one level");
    for (int l = 0; l < n; ++l) {
        if (!(sigmas[l] >= 0.0)) throw_argument("scale continuation: sigmas must be >= 0");
        if (l > 0 && !(sigmas[l] < sigmas[l - 1]))
            throw_argument("scale continuation: sigmas must be strictly decreasing");
    }
    const long long N = ctx->g.N;
    DevBuf R(ctx, N), T(ctx, N), v(ctx, 3 * N);
    VR_CUDA(cudaMemcpyAsync(v.p, v0, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
    std::vector<GnResult> out;
    for (int l = 0; l < n; ++l) {
        const double* r = mR;
        const double* t = mT;
        if (sigmas[l] > 0.0) {
            gaussian(ctx, mR, R.p, sigmas[l]);
            gaussian(ctx, mT, T.p, sigmas[l]);
            r = R.p, t = T.p;
        }
        out.push_back(gauss_newton_solve(ctx, r, t, v.p, model, params, precond, v.p));
        if (out.back().report.stop == VR_STOP_LINE_SEARCH_FAILURE) break;
    }
    VR_CUDA(cudaMemcpyAsync(v_out, v.p, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
    VR_CUDA(cudaStreamSynchronize(ctx->stream));
    return out;
}

// beta search: bisection on log10 beta_v over [lo, hi]; a trial is
// feasible iff eps_J <= min det grad y and max det grad y <= 1 / eps_J. Order: the
// upper end (must be feasible), the lower end (feasible -> done), then midpoints
// until the bracket is narrower than min_width decades or max_bisections trials;
// every trial warm-starts from the previous trial's velocity.
BetaSearch beta_search(vr_ctx* ctx, const double* mR, const double* mT, const double* v0,
                       const vr_model& model, const vr_solver_params& params, int precond,
                       const vr_beta_search_params& bp, double* v_out) {
    if (!(bp.eps_J > 0.0 && bp.eps_J < 1.0)) throw_argument("beta search: eps_J must be in (0, 1)");
    if (!(bp.beta_lo > 0.0 && bp.beta_lo < bp.beta_hi))
        throw_argument("beta search: need 0 < beta_lo < beta_hi");
    if (bp.max_bisections < 0 || !(bp.min_width_decades > 0.0))
        throw_argument("beta search: max_bisections >= 0 and min_width_decades > 0");
    const long long N = ctx->g.N;
    DevBuf vprev(ctx, 3 * N), vtrial(ctx, 3 * N), vbest(ctx, 3 * N), det(ctx, N);
    VR_CUDA(cudaMemcpyAsync(vprev.p, v0, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
    BetaSearch bs;
    auto trial = [&](double beta) {
        vr_model m = model;
        m.beta_v = beta;
        GnResult r = gauss_newton_solve(ctx, mR, mT, vprev.p, m, params, precond, vtrial.p);
        det_deformation_gradient(ctx, vtrial.p, model.nt, det.p);
        vr_beta_trial t{};
        t.beta = beta;
        t.det = det_stats(ctx, det.p, nullptr, 0.0);
        t.feasible = t.det.min >= bp.eps_J && t.det.max <= 1.0 / bp.eps_J;
        t.report = r.report;
        bs.trials.push_back(t);
        VR_CUDA(cudaMemcpyAsync(vprev.p, vtrial.p, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
        if (t.feasible) {
            VR_CUDA(cudaMemcpyAsync(vbest.p, vtrial.p, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
            bs.beta = beta;
        }
        return static_cast<bool>(t.feasible);
    };
    bs.beta = 0.0;
    if (!trial(bp.beta_hi)) {
        bs.found = false;
        return bs;
    }
    if (!trial(bp.beta_lo)) {
        double lo = std::log10(bp.beta_lo), hi = std::log10(bp.beta_hi);
        for (int k = 0; k < bp.max_bisections && hi - lo >= bp.min_width_decades; ++k) {
            const double mid = 0.5 * (lo + hi);
            if (trial(std::pow(10.0, mid)))
                hi = mid;
            else
                lo = mid;
        }
    }
    bs.found = true;
    VR_CUDA(cudaMemcpyAsync(v_out, vbest.p, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, ctx->stream));
    VR_CUDA(cudaStreamSynchronize(ctx->stream));
    return bs;
}

}  // namespace vr
