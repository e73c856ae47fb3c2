// twolevel.cu -- spectral grid transfer and the two-level preconditioner.
//
// Reference: proj/src/spectral.cpp:228-385 (alias-folding restriction /
// prolongation of half spectra, spectral_resample, frequency_filter),
// proj/src/objective.cpp:158-176 (split matvec), proj/src/precond.cpp:11-249
// (Lanczos bounds, Chebyshev semi-iteration, TwoLevelContext rebuild/apply) and
// the split branch of gauss_newton_solve (proj/src/solver.cpp:208-221).
//
// Device work: the transfer kernels below (one thread per destination bin, a
// gather form of the reference's deposit loops: every destination bin receives
// from at most one source bin when prolonging, and sums the <= 8 aliases in the
// reference's p -> q -> r order when restricting), plus the existing FFT,
// transport and BLAS-1 kernels on a coarse sibling context (n/2 per axis) that
// shares the fine context's stream. The Krylov / Lanczos / Chebyshev control
// flow is host C++ with the reference's constants. On x1 slabs the coarse sibling
// is a slab context on the same transport and the grid transfers exchange the
// coarse band between the ranks' k2 slabs (resample_scalar_slabs).
#include <algorithm>
#include <cmath>
#include <random>
#include <vector>

#include "objective.cuh"
#include "twolevel.cuh"

namespace vr {

namespace {

// grid.hpp:60: signed frequency of bin index i on an n-point axis
__device__ __forceinline__ int sfreq(int i, int n) { return 2 * i <= n ? i : i - n; }
__device__ __forceinline__ int wrap_k(int k, int n) { return k >= 0 ? k : k + n; }

struct SpecGrid {
    int n1, n2, n3, nh;
};
SpecGrid spec_grid(int n1, int n2, int n3) { return {n1, n2, n3, n3 / 2 + 1}; }

// spectrum_restrict (spectral.cpp:280-306): out(q) = scale * sum over the alias
// set of q (the Nyquist mode of an even, strictly smaller target axis folds +-m/2)
__global__ void k_spec_restrict(const double2* __restrict__ in, SpecGrid s, double2* __restrict__ out,
                                SpecGrid d, double scale) {
    const long long nb = static_cast<long long>(d.n1) * d.n2 * d.nh;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
         b += (long long)gridDim.x * blockDim.x) {
        const int j3 = static_cast<int>(b % d.nh);
        const int j2 = static_cast<int>((b / d.nh) % d.n2);
        const int j1 = static_cast<int>(b / (static_cast<long long>(d.nh) * d.n2));
        int k1[2], k2[2], k3[2], c1 = 1, c2 = 1, c3 = 1;
        const int q1 = sfreq(j1, d.n1), q2 = sfreq(j2, d.n2);
        k1[0] = q1, k2[0] = q2, k3[0] = j3;
        if (d.n1 != s.n1 && d.n1 % 2 == 0 && abs(q1) == d.n1 / 2) k1[0] = d.n1 / 2, k1[1] = -d.n1 / 2, c1 = 2;
        if (d.n2 != s.n2 && d.n2 % 2 == 0 && abs(q2) == d.n2 / 2) k2[0] = d.n2 / 2, k2[1] = -d.n2 / 2, c2 = 2;
        if (d.n3 != s.n3 && d.n3 % 2 == 0 && j3 == d.n3 / 2) k3[0] = d.n3 / 2, k3[1] = -d.n3 / 2, c3 = 2;
        double vr = 0.0, vi = 0.0;
        for (int p = 0; p < c1; ++p)
            for (int q = 0; q < c2; ++q)
                for (int r = 0; r < c3; ++r) {
                    double2 m;
                    if (k3[r] >= 0) {
                        m = in[(static_cast<long long>(wrap_k(k1[p], s.n1)) * s.n2 +
                                wrap_k(k2[q], s.n2)) * s.nh + k3[r]];
                    } else {  // Hermitian image conj(spec(-k))
                        m = in[(static_cast<long long>(wrap_k(-k1[p], s.n1)) * s.n2 +
                                wrap_k(-k2[q], s.n2)) * s.nh - k3[r]];
                        m.y = -m.y;
                    }
                    vr += m.x;
                    vi += m.y;
                }
        out[b] = make_double2(vr * scale, vi * scale);
    }
}

// spectrum_prolong (spectral.cpp:308-331) as a gather: fine bin k takes the
// coarse bin q whose alias set contains k, weighted scale / (alias counts).
__global__ void k_spec_prolong(const double2* __restrict__ in, SpecGrid s, double2* __restrict__ out,
                               SpecGrid d, double scale) {
    const long long nb = static_cast<long long>(d.n1) * d.n2 * d.nh;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
         b += (long long)gridDim.x * blockDim.x) {
        const int i3 = static_cast<int>(b % d.nh);
        const int i2 = static_cast<int>((b / d.nh) % d.n2);
        const int i1 = static_cast<int>(b / (static_cast<long long>(d.nh) * d.n2));
        const int k[3] = {sfreq(i1, d.n1), sfreq(i2, d.n2), i3};
        const int m[3] = {s.n1, s.n2, s.n3};
        const int n[3] = {d.n1, d.n2, d.n3};
        int qi[3], cnt = 1;
        bool hit = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int ak = abs(k[a]);
            const int direct = a < 2 ? wrap_k(k[a], m[a]) : k[a];
            if (m[a] == n[a]) {
                qi[a] = direct;             // axis unchanged: alias set {q}
            } else if (m[a] % 2 == 0) {
                if (ak < m[a] / 2) {
                    qi[a] = direct;
                } else if (ak == m[a] / 2) {
                    qi[a] = m[a] / 2;       // the coarse Nyquist bin (+m/2) folds onto +-m/2
                    cnt *= 2;
                } else {
                    hit = false;
                }
            } else if (ak <= m[a] / 2) {    // odd coarse axis: no fold
                qi[a] = direct;
            } else {
                hit = false;
            }
        }
        double2 v = make_double2(0.0, 0.0);
        if (hit) {
            const double w = scale / cnt;
            const double2 c = in[(static_cast<long long>(qi[0]) * s.n2 + qi[1]) * s.nh + qi[2]];
            v = make_double2(0.0 + c.x * w, 0.0 + c.y * w);
        }
        out[b] = v;
    }
}

unsigned grid_for(long long n) {
    const long long b = (n + 255) / 256;
    return static_cast<unsigned>(b < 148 * 16 ? b : 148 * 16);
}

void launch_restrict(vr_ctx* ctx, const double* in, SpecGrid s, double* out, SpecGrid d, double scale) {
    const long long nb = static_cast<long long>(d.n1) * d.n2 * d.nh;
    VR_LAUNCH(ctx, "spec_transfer", k_spec_restrict<<<grid_for(nb), 256, 0, ctx->stream>>>(
        reinterpret_cast<const double2*>(in), s, reinterpret_cast<double2*>(out), d, scale));
}
void launch_prolong(vr_ctx* ctx, const double* in, SpecGrid s, double* out, SpecGrid d, double scale) {
    const long long nb = static_cast<long long>(d.n1) * d.n2 * d.nh;
    VR_LAUNCH(ctx, "spec_transfer", k_spec_prolong<<<grid_for(nb), 256, 0, ctx->stream>>>(
        reinterpret_cast<const double2*>(in), s, reinterpret_cast<double2*>(out), d, scale));
}

SpecGrid grid_of(const vr_ctx* c) { return spec_grid(c->g.n1, c->g.n2, c->g.n3); }

// ---- x1 slabs: the spectra live in the x1 layout [n1][n2s][nh] (rank r holds the k2 rows
// [r n2s, (r+1) n2s)), and the coarse rows a rank needs sit on other ranks (coarse row j2 is
// fine row j2 or j2 + m2, i.e. on the lowest or highest quarter of the fine ranks).
struct SlabSpec {
    int n1, n2, n3, nh, n2s, k2_off;
};
SlabSpec slab_of(const vr_ctx* c) {
    return {c->g.n1, c->g.n2, c->g.n3, c->g.nh, c->g.n2s, c->g.k2_off};
}

// Restriction, sender side: for every coarse bin of every destination rank q, the partial
// alias sum over the fine bins THIS rank holds (zero when it holds none); the receiver adds
// the P blocks in rank order. Same alias sets as k_spec_restrict.
__global__ void k_slab_restrict_pack(const double2* __restrict__ in, SlabSpec s, double2* __restrict__ send,
                                     SlabSpec d, int P, double scale) {
    const long long blk = static_cast<long long>(d.n1) * d.n2s * d.nh;
    const long long nb = blk * P;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
         b += (long long)gridDim.x * blockDim.x) {
        const int q = static_cast<int>(b / blk);
        const long long l = b - q * blk;
        const int j3 = static_cast<int>(l % d.nh);
        const int j2 = static_cast<int>((l / d.nh) % d.n2s) + q * d.n2s;
        const int j1 = static_cast<int>(l / (static_cast<long long>(d.nh) * d.n2s));
        int k1[2], k2[2], k3[2], c1 = 1, c2 = 1, c3 = 1;
        const int q1 = sfreq(j1, d.n1), q2 = sfreq(j2, d.n2);
        k1[0] = q1, k2[0] = q2, k3[0] = j3;
        if (d.n1 != s.n1 && d.n1 % 2 == 0 && abs(q1) == d.n1 / 2) k1[0] = d.n1 / 2, k1[1] = -d.n1 / 2, c1 = 2;
        if (d.n2 != s.n2 && d.n2 % 2 == 0 && abs(q2) == d.n2 / 2) k2[0] = d.n2 / 2, k2[1] = -d.n2 / 2, c2 = 2;
        if (d.n3 != s.n3 && d.n3 % 2 == 0 && j3 == d.n3 / 2) k3[0] = d.n3 / 2, k3[1] = -d.n3 / 2, c3 = 2;
        double vr = 0.0, vi = 0.0;
        for (int p = 0; p < c1; ++p)
            for (int qq = 0; qq < c2; ++qq)
                for (int r = 0; r < c3; ++r) {
                    const bool img = k3[r] < 0;  // Hermitian image conj(spec(-k))
                    const int i1 = wrap_k(img ? -k1[p] : k1[p], s.n1);
                    const int i2 = wrap_k(img ? -k2[qq] : k2[qq], s.n2) - s.k2_off;
                    const int i3 = img ? -k3[r] : k3[r];
                    if (i2 < 0 || i2 >= s.n2s) continue;  // another rank's row
                    const double2 m = in[(static_cast<long long>(i1) * s.n2s + i2) * s.nh + i3];
                    vr += m.x;
                    vi += img ? -m.y : m.y;
                }
        send[b] = make_double2(vr * scale, vi * scale);
    }
}
__global__ void k_slab_sum_blocks(const double2* __restrict__ recv, long long blk, int P,
                                  double2* __restrict__ out) {
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < blk;
         b += (long long)gridDim.x * blockDim.x) {
        double2 a = recv[b];
        for (int q = 1; q < P; ++q) {
            const double2 v = recv[q * blk + b];
            a.x += v.x, a.y += v.y;
        }
        out[b] = a;
    }
}
// Prolongation, receiver side: `all` = every rank's coarse slab spectrum in rank order
// (block t = [m1][m2s][mh]); fine bin k of this rank's k2 rows takes the coarse bin whose
// alias set contains k. Same rule as k_spec_prolong.
__global__ void k_slab_prolong(const double2* __restrict__ all, SlabSpec s, double2* __restrict__ out,
                               SlabSpec d, double scale) {
    const long long nb = static_cast<long long>(d.n1) * d.n2s * d.nh;
    const long long blk = static_cast<long long>(s.n1) * s.n2s * s.nh;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
         b += (long long)gridDim.x * blockDim.x) {
        const int i3 = static_cast<int>(b % d.nh);
        const int i2 = static_cast<int>((b / d.nh) % d.n2s) + d.k2_off;
        const int i1 = static_cast<int>(b / (static_cast<long long>(d.nh) * d.n2s));
        const int k[3] = {sfreq(i1, d.n1), sfreq(i2, d.n2), i3};
        const int m[3] = {s.n1, s.n2, s.n3};
        const int n[3] = {d.n1, d.n2, d.n3};
        int qi[3], cnt = 1;
        bool hit = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int ak = abs(k[a]);
            const int direct = a < 2 ? wrap_k(k[a], m[a]) : k[a];
            if (m[a] == n[a]) {
                qi[a] = direct;
            } else if (m[a] % 2 == 0) {
                if (ak < m[a] / 2) {
                    qi[a] = direct;
                } else if (ak == m[a] / 2) {
                    qi[a] = m[a] / 2;
                    cnt *= 2;
                } else {
                    hit = false;
                }
            } else if (ak <= m[a] / 2) {
                qi[a] = direct;
            } else {
                hit = false;
            }
        }
        double2 v = make_double2(0.0, 0.0);
        if (hit) {
            const double w = scale / cnt;
            const int t = qi[1] / s.n2s, row = qi[1] - t * s.n2s;
            const double2 c = all[t * blk + (static_cast<long long>(qi[0]) * s.n2s + row) * s.nh + qi[2]];
            v = make_double2(0.0 + c.x * w, 0.0 + c.y * w);
        }
        out[b] = v;
    }
}

void need_single(const vr_ctx* c, const char* what) {
    if (c->dist) throw_argument(std::string(what) + ": one GPU only (not on x1 slabs)");
}

// make `b` wait for the work queued so far on `a` (no-op on a shared stream)
void order_after(vr_ctx* a, vr_ctx* b) {
    if (a->stream == b->stream) return;
    VR_CUDA(cudaEventRecord(a->ev_fork, a->stream));
    VR_CUDA(cudaStreamWaitEvent(b->stream, a->ev_fork, 0));
}

}  // namespace

// ---------------------------------------------------------------------------
// spectral_resample (spectral.cpp:340-356), one scalar field per call
// x1 slabs (both contexts on the same transport): r2c on the source slabs, exchange of the
// coarse band, c2r on the destination slabs. Restriction: every rank packs, per destination
// rank, the partial alias sums of the fine rows it holds; one all-to-all; the receiver adds the
// blocks in rank order. Prolongation: the coarse slab spectra are all-gathered (an all-to-all of
// P copies; the coarse spectrum is 1/8 of the fine one) and every rank fills its fine rows.
static void resample_scalar_slabs(vr_ctx* src, const double* in, vr_ctx* dst, double* out) {
    if (!src->dist || !dst->dist || src->dist != dst->dist)
        throw_argument("spectral_resample: both contexts must be slabs of one rank group");
    if (src->stream != dst->stream) throw_argument("spectral_resample: slab contexts must share a stream");
    const int P = src->dist->size;
    if (src->g.n1 == dst->g.n1 && src->g.n2 == dst->g.n2 && src->g.n3 == dst->g.n3) {
        VR_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * src->g.N, cudaMemcpyDeviceToDevice, src->stream));
        return;
    }
    const bool down = dst->g.n1 <= src->g.n1 && dst->g.n2 <= src->g.n2 && dst->g.n3 <= src->g.n3;
    const bool up = dst->g.n1 >= src->g.n1 && dst->g.n2 >= src->g.n2 && dst->g.n3 >= src->g.n3;
    if (!down && !up)
        throw_dimension("spectral_resample: target must be coarser or finer on every axis");
    double* cs = spec_buf(src, 0);
    double* cd = spec_buf(dst, 0);
    fft_r2c(src, in, cs);
    const double scale = static_cast<double>(dst->g.Ng) / static_cast<double>(src->g.Ng);
    const vr_ctx* coarse = down ? dst : src;
    const long long blk = coarse->g.NC;  // complex bins of one coarse slab spectrum
    double* send = dev_alloc(src, 2 * blk * P);
    double* recv = dev_alloc(src, 2 * blk * P);
    try {
        if (down) {
            VR_LAUNCH(src, "spec_transfer", k_slab_restrict_pack<<<grid_for(blk * P), 256, 0, src->stream>>>(
                reinterpret_cast<const double2*>(cs), slab_of(src), reinterpret_cast<double2*>(send),
                slab_of(dst), P, scale));
            src->dist->alltoall(src, send, recv, static_cast<size_t>(2 * blk));
            VR_LAUNCH(src, "spec_transfer", k_slab_sum_blocks<<<grid_for(blk), 256, 0, src->stream>>>(
                reinterpret_cast<const double2*>(recv), blk, P, reinterpret_cast<double2*>(cd)));
        } else {
            for (int q = 0; q < P; ++q)
                VR_CUDA(cudaMemcpyAsync(send + 2 * blk * q, cs, sizeof(double) * 2 * blk,
                                        cudaMemcpyDeviceToDevice, src->stream));
            src->dist->alltoall(src, send, recv, static_cast<size_t>(2 * blk));
            VR_LAUNCH(src, "spec_transfer", k_slab_prolong<<<grid_for(dst->g.NC), 256, 0, src->stream>>>(
                reinterpret_cast<const double2*>(recv), slab_of(src), reinterpret_cast<double2*>(cd),
                slab_of(dst), scale));
        }
    } catch (...) {
        dev_free(src, send);
        dev_free(src, recv);
        throw;
    }
    dev_free(src, send);
    dev_free(src, recv);
    fft_c2r(dst, cd, out, 1.0 / static_cast<double>(dst->g.Ng), nullptr);
}

void resample_scalar(vr_ctx* src, const double* in, vr_ctx* dst, double* out) {
    if (src->dist || dst->dist) {
        resample_scalar_slabs(src, in, dst, out);
        return;
    }
    if (src->device != dst->device)
        throw_argument("spectral_resample: both contexts must be on one device");
    if (src->g.n1 == dst->g.n1 && src->g.n2 == dst->g.n2 && src->g.n3 == dst->g.n3) {
        VR_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * src->g.N, cudaMemcpyDeviceToDevice,
                                src->stream));
        order_after(src, dst);
        return;
    }
    const bool down = dst->g.n1 <= src->g.n1 && dst->g.n2 <= src->g.n2 && dst->g.n3 <= src->g.n3;
    const bool up = dst->g.n1 >= src->g.n1 && dst->g.n2 >= src->g.n2 && dst->g.n3 >= src->g.n3;
    if (!down && !up)
        throw_dimension("spectral_resample: target must be coarser or finer on every axis");
    double* cs = spec_buf(src, 0);
    double* cd = spec_buf(dst, 0);
    fft_r2c(src, in, cs);
    const double scale = static_cast<double>(dst->g.Ng) / static_cast<double>(src->g.Ng);
    if (down)
        launch_restrict(src, cs, grid_of(src), cd, grid_of(dst), scale);
    else
        launch_prolong(src, cs, grid_of(src), cd, grid_of(dst), scale);
    order_after(src, dst);
    fft_c2r(dst, cd, out, 1.0 / static_cast<double>(dst->g.Ng), nullptr);
    order_after(dst, src);
}

// frequency_filter (spectral.cpp:358-385): F_L f = prolong(restrict(f)) through
// the cutoff grid; F_H f = f - F_L f
void frequency_filter(vr_ctx* ctx, const double* in, int band, const int cutoff[3], double* out) {
    need_single(ctx, "frequency_filter");
    const GridDims& g = ctx->g;
    const int gd[3] = {g.n1, g.n2, g.n3};
    for (int a = 0; a < 3; ++a)
        if (cutoff[a] > gd[a] || cutoff[a] < 1)
            throw_dimension("frequency_filter: target/cutoff axis " + std::to_string(a) +
                            " exceeds source");
    if (cutoff[0] == g.n1 && cutoff[1] == g.n2 && cutoff[2] == g.n3) {
        if (band == 0)
            VR_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * g.N, cudaMemcpyDeviceToDevice, ctx->stream));
        else
            VR_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * g.N, ctx->stream));
        return;
    }
    const SpecGrid cg = spec_grid(cutoff[0], cutoff[1], cutoff[2]);
    const long long ncut = static_cast<long long>(cg.n1) * cg.n2 * cg.nh;
    double* cs = spec_buf(ctx, 0);
    double* lo = dev_alloc(ctx, 2 * ncut);
    try {
        fft_r2c(ctx, in, cs);
        const double ncut_pts = static_cast<double>(cutoff[0]) * cutoff[1] * cutoff[2];
        launch_restrict(ctx, cs, grid_of(ctx), lo, cg, ncut_pts / static_cast<double>(g.Ng));
        launch_prolong(ctx, lo, cg, cs, grid_of(ctx), static_cast<double>(g.Ng) / ncut_pts);
        if (band == 0) {
            fft_c2r(ctx, cs, out, 1.0 / static_cast<double>(g.Ng), nullptr);
        } else {
            double* low = field_buf(ctx, 0);
            fft_c2r(ctx, cs, low, 1.0 / static_cast<double>(g.Ng), nullptr);
            lin_comb(ctx, out, 1.0, in, -1.0, low, g.N);  // high = f - low
        }
    } catch (...) {
        dev_free(ctx, lo);
        throw;
    }
    dev_free(ctx, lo);
}

// ---------------------------------------------------------------------------
// Objective::split_matvec (objective.cpp:158-176): (I + R H_data R) w, R = (beta_v A)^-1/2,
// minus the per-component mean of w when A has a zero singular value
void split_matvec(vr_objective* o, const vr_state* s, const double* w3, double* out3) {
    vr_ctx* ctx = o->ctx;
    const long long N = ctx->g.N;
    double* u = dev_alloc(ctx, 3 * N);
    double* du = dev_alloc(ctx, 3 * N);
    try {
        objective_apply_reg(o, w3, VR_REGOP_INVERSE_SQRT, u);
        objective_matvec(o, s, u, du, false);
        objective_apply_reg(o, du, VR_REGOP_INVERSE_SQRT, out3);
        add_scaled(ctx, out3, 1.0, w3, 3 * N);
        if (reg_symbol(o->model.norm, 0.0) == 0.0) {
            double sums[3];
            sum_components(ctx, w3, N, 3, sums);
            for (int c = 0; c < 3; ++c) {
                const double mean = sums[c] / static_cast<double>(ctx->g.Ng);
                affine(ctx, out3 + c * N, out3 + c * N, N, mean, 1.0);
            }
        }
    } catch (...) {
        dev_free(ctx, u);
        dev_free(ctx, du);
        throw;
    }
    dev_free(ctx, u);
    dev_free(ctx, du);
}

// ---------------------------------------------------------------------------
// Lanczos bounds (precond.cpp:73-107) and the tridiagonal extreme eigenvalues
namespace {

// number of eigenvalues of the symmetric tridiagonal (alpha, beta) below x
// (Sturm sequence of the LDL^T pivots; a zero pivot is replaced by a tiny one)
int pivots_below(const std::vector<double>& alpha, const std::vector<double>& beta, double x) {
    int below = 0;
    double piv = 1.0;
    for (size_t i = 0; i < alpha.size(); ++i) {
        const double off = i ? beta[i - 1] * beta[i - 1] : 0.0;
        piv = alpha[i] - x - (piv == 0.0 ? off / 1e-300 : off / piv);
        below += piv < 0.0;
    }
    return below;
}

// smallest (largest) eigenvalue: bisection on the Gershgorin interval
double extreme_eig(const std::vector<double>& alpha, const std::vector<double>& beta, bool top) {
    const int m = static_cast<int>(alpha.size());
    double lo = alpha[0], hi = alpha[0];
    for (int i = 0; i < m; ++i) {
        double rad = 0.0;
        if (i > 0) rad += std::abs(beta[i - 1]);
        if (i + 1 < m) rad += std::abs(beta[i]);
        lo = std::min(lo, alpha[i] - rad);
        hi = std::max(hi, alpha[i] + rad);
    }
    for (int step = 0; step < 200; ++step) {
        const double x = 0.5 * (lo + hi);
        const int below = pivots_below(alpha, beta, x);
        const bool left = top ? below >= m : below >= 1;
        (left ? hi : lo) = x;
        if (hi - lo < 1e-12 * std::max(1.0, std::abs(hi))) break;
    }
    return 0.5 * (lo + hi);
}

}  // namespace

std::pair<double, double> lanczos_bounds(vr_ctx* ctx, const DevOp& op, int iterations,
                                         unsigned long long seed) {
    const long long n3 = 3 * ctx->g.N;
    // seeded start vector, drawn on the host in the reference's order (component, point)
    // (x1 slabs: every rank draws the global sequence and keeps its planes)
    std::vector<double> h(static_cast<size_t>(n3));
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    if (!ctx->dist) {
        for (auto& x : h) x = uni(rng);
    } else {
        const long long N = ctx->g.N, Ng = ctx->g.Ng;
        const long long first = static_cast<long long>(ctx->g.off1) * ctx->g.n2 * ctx->g.n3;
        for (int c = 0; c < 3; ++c)
            for (long long i = 0; i < Ng; ++i) {
                const double x = uni(rng);
                if (i >= first && i < first + N) h[static_cast<size_t>(c * N + (i - first))] = x;
            }
    }
    double* q = dev_alloc(ctx, n3);
    double* qp = dev_alloc(ctx, n3);
    double* w = dev_alloc(ctx, n3);
    std::vector<double> alpha, beta;
    try {
        VR_CUDA(cudaMemcpyAsync(q, h.data(), sizeof(double) * n3, cudaMemcpyHostToDevice, ctx->stream));
        VR_CUDA(cudaMemsetAsync(qp, 0, sizeof(double) * n3, ctx->stream));
        scale(ctx, q, n3, 1.0 / norm_l2_vec(ctx, q));
        for (int j = 0; j < iterations; ++j) {
            op(q, w);
            const double a = dot_l2_vec(ctx, q, w);
            alpha.push_back(a);
            add_scaled(ctx, w, -a, q, n3);
            if (j > 0) add_scaled(ctx, w, -beta.back(), qp, n3);
            const double b = norm_l2_vec(ctx, w);
            if (b < 1e-12) break;  // Krylov space exhausted
            if (j + 1 < iterations) beta.push_back(b);
            std::swap(qp, q);  // q_prev = q
            std::swap(q, w);   // q = w
            scale(ctx, q, n3, 1.0 / b);
        }
    } catch (...) {
        for (double* p : {q, qp, w}) dev_free(ctx, p);
        throw;
    }
    VR_CUDA(cudaStreamSynchronize(ctx->stream));  // h is read by the async upload
    for (double* p : {q, qp, w}) dev_free(ctx, p);
    beta.resize(alpha.empty() ? 0 : alpha.size() - 1);
    return {0.95 * extreme_eig(alpha, beta, false), 1.05 * extreme_eig(alpha, beta, true)};
}

// cheb_solve (precond.cpp:113-147): k steps of the three-term Chebyshev iteration
void cheb_solve(vr_ctx* ctx, const DevOp& op, const double* rhs, int k,
                std::pair<double, double> bounds, double* x) {
    const double lo = bounds.first, hi = bounds.second;
    if (lo <= 0.0) throw_argument("cheb_solve: lower eigenvalue bound must be > 0");
    if (hi < lo) throw_argument("cheb_solve: invalid eigenvalue bounds");
    const long long n3 = 3 * ctx->g.N;
    const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo);
    VR_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n3, ctx->stream));
    if (norm_l2_vec(ctx, rhs) == 0.0) return;
    double* r = dev_alloc(ctx, n3);
    double* Ad = dev_alloc(ctx, n3);
    double* d = dev_alloc(ctx, n3);
    try {
        VR_CUDA(cudaMemcpyAsync(r, rhs, sizeof(double) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
        if (delta <= 1e-14 * theta) {  // point spectrum: Richardson is exact
            for (int j = 0; j < k; ++j) {
                add_scaled(ctx, x, 1.0 / theta, r, n3);
                op(x, Ad);
                lin_comb(ctx, r, 1.0, rhs, -1.0, Ad, n3);
                if (norm_l2_vec(ctx, r) == 0.0) break;
            }
        } else {
            const double sigma1 = theta / delta;
            double rho = 1.0 / sigma1;
            VR_CUDA(cudaMemcpyAsync(d, r, sizeof(double) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
            scale(ctx, d, n3, 1.0 / theta);
            add_scaled(ctx, x, 1.0, d, n3);
            for (int j = 1; j < k; ++j) {
                op(d, Ad);
                add_scaled(ctx, r, -1.0, Ad, n3);
                const double rho_next = 1.0 / (2.0 * sigma1 - rho);
                lin_comb(ctx, d, rho_next * rho, d, 2.0 * rho_next / delta, r, n3);
                add_scaled(ctx, x, 1.0, d, n3);
                rho = rho_next;
            }
        }
    } catch (...) {
        for (double* p : {r, Ad, d}) dev_free(ctx, p);
        throw;
    }
    for (double* p : {r, Ad, d}) dev_free(ctx, p);
}

// ---------------------------------------------------------------------------
// TwoLevelContext (precond.cpp:151-249)
TwoLevel::TwoLevel(const vr_twolevel_options& o) : opts(o) {
    if (o.inner != 0 && o.inner != 1) throw_argument("two-level: inner must be 0 (pcg) or 1 (cheb)");
    if (!(o.kappa > 0.0) || o.cheb_iterations < 1 || o.max_inner_iterations < 1 ||
        o.lanczos_iterations < 1)
        throw_argument("two-level: invalid options");
}

TwoLevel::~TwoLevel() { release(); }

void TwoLevel::release() {
    delete cstate;
    cstate = nullptr;
    if (cobj) {
        add_counters(cobj->counters);
        delete cobj;
        cobj = nullptr;
    }
    if (cctx) {
        dev_free(cctx, mRc);
        dev_free(cctx, mTc);
    }
    mRc = mTc = nullptr;
}

void TwoLevel::add_counters(const vr_counters& c) {
    done.objective_evals += c.objective_evals;
    done.gradient_evals += c.gradient_evals;
    done.hessian_matvecs += c.hessian_matvecs;
    done.pde_solves += c.pde_solves;
}

vr_counters TwoLevel::counters() const {
    vr_counters c = done;
    if (cobj) {
        c.objective_evals += cobj->counters.objective_evals;
        c.gradient_evals += cobj->counters.gradient_evals;
        c.hessian_matvecs += cobj->counters.hessian_matvecs;
        c.pde_solves += cobj->counters.pde_solves;
    }
    return c;
}

void TwoLevel::destroy_ctx() {
    release();
    cctx = nullptr;  // the fine context owns its cached siblings
}

void TwoLevel::resample_vec(vr_ctx* src, const double* in, vr_ctx* dst, double* out) {
    for (int c = 0; c < 3; ++c) resample_scalar(src, in + c * src->g.N, dst, out + c * dst->g.N);
}

void TwoLevel::rebuild(vr_objective* fine_obj, const vr_state* fine_state, double eps_H) {
    vr_ctx* f = fine_obj->ctx;
    const int d[3] = {f->g.n1, f->g.n2, f->g.n3};
    for (int a = 0; a < 3; ++a)
        if (d[a] % 2 != 0 || d[a] / 2 < 4)
            throw_dimension("two-level preconditioner: fine grid " + std::to_string(d[0]) + "x" +
                            std::to_string(d[1]) + "x" + std::to_string(d[2]) +
                            " does not halve to a valid coarse grid");
    const bool full = !fine_obj->model.gauss_newton;
    if (full && !fine_state->lamhist)
        throw_logic("two-level rebuild: full Newton needs the fine adjoint history");
    if (cctx && cctx->stream != f->stream) destroy_ctx();  // a different fine context
    if (!cctx) cctx = ctx_sibling(f, d[0] / 2, d[1] / 2, d[2] / 2);
    release();
    const long long Nc = cctx->g.N;
    const int nt = fine_state->nt;
    mRc = dev_alloc(cctx, Nc);
    mTc = dev_alloc(cctx, Nc);
    resample_scalar(f, fine_obj->mR, cctx, mRc);
    resample_scalar(f, fine_obj->mT, cctx, mTc);
    cobj = objective_create(cctx, mRc, mTc, fine_obj->model);
    // coarse evaluation context: restricted v and m history, fresh coarse characteristics
    double* vc = dev_alloc(cctx, 3 * Nc);
    double* hc = dev_alloc(cctx, (nt + 1) * Nc);
    double* lc = full ? dev_alloc(cctx, (nt + 1) * Nc) : nullptr;
    try {
        resample_vec(f, fine_state->v, cctx, vc);
        for (int j = 0; j <= nt; ++j) {
            resample_scalar(f, pslice(f, fine_state->mhist, j), cctx, hc + j * Nc);
            if (full) resample_scalar(f, pslice(f, fine_state->lamhist, j), cctx, lc + j * Nc);
        }
        cstate = state_from_history(cobj, vc, hc, nt, lc);
    } catch (...) {
        dev_free(cctx, vc);
        dev_free(cctx, hc);
        dev_free(cctx, lc);
        throw;
    }
    dev_free(cctx, vc);
    dev_free(cctx, hc);
    dev_free(cctx, lc);
    eps_M = opts.kappa * eps_H;
    inner_diverged = false;
    if (opts.inner == 1) {
        DevOp op = [this](const double* u, double* out) { split_matvec(cobj, cstate, u, out); };
        bounds = lanczos_bounds(cctx, op, opts.lanczos_iterations, opts.lanczos_seed);
        ++lanczos_runs;
    }
}

void TwoLevel::coarse_matvec(const double* u, double* out) {
    if (!cobj) throw_logic("two-level preconditioner applied before rebuild");
    split_matvec(cobj, cstate, u, out);
}

// u = Q_P u_bar + F_H s, H_bar u_bar ~ Q_R F_L s by the inner solver
void TwoLevel::apply(vr_ctx* f, const double* s, double* u) {
    if (!cobj) throw_logic("two-level preconditioner applied before rebuild");
    const long long N = f->g.N, Nc = cctx->g.N;
    double* slc = dev_alloc(cctx, 3 * Nc);   // Q_R s (= Q_R F_L s)
    double* shigh = dev_alloc(f, 3 * N);     // s - F_L s
    double* ubar = dev_alloc(cctx, 3 * Nc);
    auto cleanup = [&] {
        dev_free(cctx, slc);
        dev_free(f, shigh);
        dev_free(cctx, ubar);
    };
    try {
        resample_vec(f, s, cctx, slc);
        resample_vec(cctx, slc, f, shigh);                 // F_L s
        lin_comb(f, shigh, 1.0, s, -1.0, shigh, 3 * N);    // s_high = s - s_low
        DevOp op = [this](const double* x, double* y) { split_matvec(cobj, cstate, x, y); };
        if (norm_l2_vec(cctx, slc) <= 1e-14 * std::max(1.0, norm_l2_vec(f, s))) {
            VR_CUDA(cudaMemsetAsync(ubar, 0, sizeof(double) * 3 * Nc, cctx->stream));
        } else if (opts.inner == 1) {
            cheb_solve(cctx, op, slc, opts.cheb_iterations, bounds, ubar);
        } else {
            DevOp ident = [this](const double* r, double* z) {
                VR_CUDA(cudaMemcpyAsync(z, r, sizeof(double) * 3 * cctx->g.N,
                                        cudaMemcpyDeviceToDevice, cctx->stream));
            };
            vr_pcg_stats st = pcg_solve(cctx, op, slc, eps_M, opts.max_inner_iterations, ident, ubar);
            if (!st.converged && !st.negative_curvature) inner_diverged = true;
        }
        resample_vec(cctx, ubar, f, u);
        add_scaled(f, u, 1.0, shigh, 3 * N);
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
}

}  // namespace vr
