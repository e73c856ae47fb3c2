// capi.cu -- extern "C" boundary (include/veloreg_gpu.h). Every entry point
// catches vr::Error and maps it to the veloreg::ErrorCategory status code
// (errors.hpp:9-17) plus a thread-local message, so a C++ adapter can rethrow
// the reference's typed exception.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "objective.cuh"
#include "twolevel.cuh"

namespace {

thread_local std::string g_err;
thread_local int g_cls = VR_EXC_NONE;

template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return VR_OK;
    } catch (const vr::Error& e) {
        g_err = e.what();
        g_cls = e.cls;
        return e.status;
    } catch (const std::bad_alloc& e) {
        g_err = std::string("host allocation failed: ") + e.what();
        g_cls = VR_EXC_RESOURCE;
        return VR_ERR_RESOURCE;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_cls = VR_EXC_LOGIC;
        return VR_ERR_LOGIC;
    }
}

void need(bool ok, const char* what) {
    if (!ok) vr::throw_argument(std::string(what) + ": null argument");
}
void set_dev(vr_ctx* ctx) {
    need(ctx != nullptr, "context");
    VR_CUDA(cudaSetDevice(ctx->device));
}
void check_ncomp(int ncomp) {
    if (ncomp != 1 && ncomp != 3) vr::throw_argument("ncomp must be 1 or 3");
}
bool pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
// per-operator entry points whose arguments are whole fields in the reference
// layout: one GPU only (on x1 slabs use the objective / solver entry points)
void set_dev_single(vr_ctx* ctx, const char* what) {
    set_dev(ctx);
    if (ctx->dist) vr::throw_argument(std::string(what) + ": not available on x1 slabs");
}

}  // namespace

namespace vr {

void set_last_error(int cls, const std::string& msg) {
    g_err = msg;
    g_cls = cls;
}

double* spec_buf(vr_ctx* ctx, int i) {
    if (static_cast<int>(ctx->spec_scratch.size()) <= i) ctx->spec_scratch.resize(i + 1, nullptr);
    if (!ctx->spec_scratch[i]) {
        void* p = nullptr;
        VR_CUDA(cudaMalloc(&p, sizeof(double) * 2 * ctx->g.NC));
        mem_track_alloc(ctx, p, static_cast<long long>(sizeof(double)) * 2 * ctx->g.NC);
        ctx->spec_scratch[i] = static_cast<double*>(p);
    }
    return ctx->spec_scratch[i];
}
cudaEvent_t prof_event(vr_ctx* ctx) {
    if (ctx->ev_used == ctx->ev_pool.size()) {
        cudaEvent_t e;
        VR_CUDA(cudaEventCreate(&e));
        ctx->ev_pool.push_back(e);
    }
    return ctx->ev_pool[ctx->ev_used++];
}

double* field_buf(vr_ctx* ctx, int i) {
    if (static_cast<int>(ctx->field_scratch.size()) <= i) ctx->field_scratch.resize(i + 1, nullptr);
    if (!ctx->field_scratch[i]) {
        void* p = nullptr;
        VR_CUDA(cudaMalloc(&p, sizeof(double) * ctx->g.N));
        mem_track_alloc(ctx, p, static_cast<long long>(sizeof(double)) * ctx->g.N);
        ctx->field_scratch[i] = static_cast<double*>(p);
    }
    return ctx->field_scratch[i];
}

vr_ctx* ctx_new_sibling(vr_ctx* parent, int n1, int n2, int n3) {
    // x1 slabs: the sibling is the same ranks' slab of the other grid on the parent's
    // transport; its halo covers the parent's halo in physical units (+2 planes of slack)
    int halo = 0;
    if (parent->dist) {
        const int L = n1 / parent->dist->size;
        halo = (parent->g.halo * n1 + parent->g.n1 - 1) / parent->g.n1 + 2;
        halo = halo < 4 ? 4 : halo;
        halo = halo > L ? L : halo;
    }
    vr_ctx* c = ctx_new(n1, n2, n3, parent->device, parent->dist, halo);
    VR_CUDA(cudaStreamDestroy(c->stream));
    c->stream = parent->stream;
    c->owns_stream = false;
    // slab siblings keep every exchange on the shared stream (the side-stream communicator
    // belongs to the parent's overlapped work)
    c->overlap = parent->dist ? false : parent->overlap;
    c->fuse_acc = parent->fuse_acc;
    c->parent = parent;
    return c;
}
vr_ctx* ctx_sibling(vr_ctx* parent, int n1, int n2, int n3) {
    for (vr_ctx* c : parent->siblings)
        if (c->g.n1 == n1 && c->g.n2 == n2 && c->g.n3 == n3) return c;
    vr_ctx* c = ctx_new_sibling(parent, n1, n2, n3);
    parent->siblings.push_back(c);
    return c;
}

}  // namespace vr

extern "C" {

const char* vr_last_error(void) { return g_err.c_str(); }
int vr_last_error_class(void) { return g_cls; }
int vr_abi_version(void) { return VR_ABI_VERSION; }

void vr_model_default(vr_model* m) {
    m->norm.kind = VR_REG_H2;
    m->norm.gamma = 1.0;
    m->norm.helmholtz_squared = 1;
    m->norm.div_penalty = 0;
    m->norm.beta_w = 1e-4;
    m->projection = VR_PROJ_IDENTITY;
    m->beta_v = 1e-2;
    m->nt = 4;
    m->gauss_newton = 1;
}
void vr_twolevel_options_default(vr_twolevel_options* o) {
    o->inner = VR_INNER_PCG;  // TwoLevelOptions (precond.hpp:46-53)
    o->kappa = 0.1;
    o->cheb_iterations = 10;
    o->max_inner_iterations = 500;
    o->lanczos_iterations = 10;
    o->lanczos_seed = 1234;
}
void vr_solver_params_default(vr_solver_params* p) {
    p->eps_opt = 5e-2;
    p->abs_grad_tol = 1e-6;
    p->max_newton = 50;
    p->max_krylov = 100;
    p->armijo_c1 = 1e-4;
    p->armijo_backtrack = 0.5;
    p->armijo_max_trials = 20;
    p->squared_norm_stop = 1;
}
int vr_model_validate(const vr_model* m) {
    return guard([&] {
        need(m, "model");
        vr::validate_model(*m);
    });
}
int vr_solver_params_validate(const vr_solver_params* p) {
    return guard([&] {
        need(p, "params");
        vr::validate_params(*p);
    });
}

// ---- context -----------------------------------------------------------------
int vr_ctx_create(int n1, int n2, int n3, int device, vr_ctx** out) {
    return guard([&] {
        need(out, "out");
        *out = vr::ctx_new(n1, n2, n3, device, nullptr, 0);
    });
}

}  // extern "C"

namespace vr {

// Grid3 checks (grid.hpp:24-31) plus the GPU FFT domain; with a transport of
// size P > 1 the context owns the x1 slab of rank t->rank
// x1-slab geometry of rank `rank` of P; host only.
static void slab_geometry_ex(int n1, int n2, int n3, int P, int rank, int halo, GridDims& g,
                             bool one_rank_slab) {
    const int d[3] = {n1, n2, n3};
    for (int a = 0; a < 3; ++a)
        if (d[a] < 4)
            throw_dimension("Grid3: every dimension must be >= 4, got " + std::to_string(n1) +
                            "x" + std::to_string(n2) + "x" + std::to_string(n3));
    for (int a = 0; a < 3; ++a)
        if (!pow2(d[a]) || d[a] > 1024)
            throw_dimension("vr_ctx_create: GPU grids need power-of-two dims <= 1024, got " +
                            std::to_string(n1) + "x" + std::to_string(n2) + "x" +
                            std::to_string(n3));
    if (P < 1 || rank < 0 || rank >= P) throw_argument("x1 slabs: rank must be in [0, nranks)");
    const bool slab = P > 1 || one_rank_slab;  // one-rank slabs: VR_DIST_SINGLE_RANK (self exchanges)
    if (slab) {
        if (n1 % P != 0 || n2 % P != 0 || n1 / P < 4)
            throw_argument("x1 slabs: n1 and n2 must be divisible by the rank count, >= 4 planes each");
        if (halo < 4 || halo > n1 / P)
            throw_argument("x1 slabs: halo must be in [4, n1/P]");
    }
    g.n1 = n1;
    g.n2 = n2;
    g.n3 = n3;
    g.nh = n3 / 2 + 1;
    g.dist = slab;
    g.L = n1 / P;
    g.z0 = 0;
    g.zn = g.L;
    g.off1 = rank * g.L;
    g.halo = slab ? halo : 0;
    g.n2s = n2 / P;
    g.k2_off = rank * g.n2s;
    g.N = static_cast<long long>(g.L) * n2 * n3;
    g.NC = static_cast<long long>(g.L) * n2 * g.nh;
    g.Ng = static_cast<long long>(n1) * n2 * n3;
    g.h1 = kTwoPi / n1;
    g.h2 = kTwoPi / n2;
    g.h3 = kTwoPi / n3;
    g.flags = nullptr;
}

void slab_geometry(int n1, int n2, int n3, int P, int rank, int halo, GridDims& g) {
    slab_geometry_ex(n1, n2, n3, P, rank, halo, g, false);
}

int halo_required(double vmax_x1, int nt, int n1) {
    // RK2 departure points move at most dt max|v_1| (+10% for the midpoint
    // interpolant's overshoot) and the stencil reaches 2 planes beyond floor(u) - 1
    return static_cast<int>(std::ceil(1.1 * vmax_x1 / nt / (kTwoPi / n1))) + 4;
}

vr_ctx* ctx_new(int n1, int n2, int n3, int device, Transport* t, int halo) {
    const int P = t ? t->size : 1;
    const bool slab = t && (P > 1 || std::getenv("VR_DIST_SINGLE_RANK"));
    GridDims geo;
    slab_geometry_ex(n1, n2, n3, P, slab ? t->rank : 0, halo, geo, slab);
    int count = 0;
    VR_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
        throw_resource("vr_ctx_create: no CUDA device " + std::to_string(device));
    // host waits spin instead of yielding (VR_SYNC=yield keeps the driver default): the solver
    // drains the stream for every scalar, and a yielded waiter can be rescheduled late.
    // Only takes effect if this call creates the device's primary context.
    if (const char* e = std::getenv("VR_SYNC"); !e || std::string(e) != "yield") {
        unsigned flags = 0;
        if (cudaGetDeviceFlags(&flags) == cudaSuccess && !(flags & cudaDeviceScheduleMask))
            (void)cudaSetDeviceFlags(cudaDeviceScheduleSpin);
        (void)cudaGetLastError();
    }
    VR_CUDA(cudaSetDevice(device));
    auto* ctx = new vr_ctx();
    try {
        ctx->device = device;
        VR_CUDA(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device));
        ctx->dist = slab ? t : nullptr;
        ctx->overlap = ctx->dist != nullptr;  // slabs: reg-term transposes under the sweeps
        if (const char* e = std::getenv("VR_OVERLAP")) ctx->overlap = std::atoi(e) != 0;
        if (const char* e = std::getenv("VR_FUSE_ACC")) ctx->fuse_acc = std::atoi(e) != 0;
        GridDims& g = ctx->g;
        g = geo;
        ctx->hstride = static_cast<long long>(g.L + 2 * g.halo) * n2 * n3;
        VR_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        VR_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        VR_CUDA(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        VR_CUDA(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
        VR_CUDA(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
        VR_CUDA(cudaEventCreateWithFlags(&ctx->ev_halo_fork, cudaEventDisableTiming));
        // keep freed blocks cached in the stream-ordered pool (no OS round trips)
        cudaMemPool_t pool;
        VR_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        VR_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        fft_plan_create(ctx);
        VR_CUDA(cudaMalloc(&ctx->red_partials, sizeof(double) * kRedBlocks * 8));
        VR_CUDA(cudaMalloc(&ctx->red_out, sizeof(double) * 8));
        VR_CUDA(cudaMallocHost(&ctx->red_host, sizeof(double) * 8));
        VR_CUDA(cudaMalloc(&ctx->flag_dev, sizeof(int) * 4));
        VR_CUDA(cudaMemset(ctx->flag_dev, 0, sizeof(int) * 4));
        VR_CUDA(cudaMallocHost(&ctx->flag_host, sizeof(int) * 4));
        g.flags = ctx->flag_dev;
    } catch (...) {
        ctx->dist = nullptr;  // the transport belongs to the caller
        vr_ctx_destroy(ctx);
        throw;
    }
    return ctx;
}

}  // namespace vr

extern "C" {

int vr_slab_layout(int n1, int n2, int n3, int rank, int nranks, int halo, long long* out) {
    return guard([&] {
        need(out != nullptr, "vr_slab_layout");
        vr::GridDims g;
        vr::slab_geometry(n1, n2, n3, nranks, rank, halo, g);
        const long long v[VR_SLAB_FIELDS] = {
            g.L, g.off1, g.halo, g.n2s, g.k2_off, g.N, g.NC,
            static_cast<long long>(g.L + 2 * g.halo) * n2 * n3, g.Ng};
        for (int i = 0; i < VR_SLAB_FIELDS; ++i) out[i] = v[i];
    });
}

int vr_slab_halo_required(double vmax_x1, int nt, int n1, int* planes) {
    return guard([&] {
        need(planes != nullptr, "vr_slab_halo_required");
        if (nt < 1 || n1 < 4 || !(vmax_x1 >= 0.0) || !std::isfinite(vmax_x1))
            vr::throw_argument("vr_slab_halo_required: need nt >= 1, n1 >= 4, finite vmax >= 0");
        *planes = vr::halo_required(vmax_x1, nt, n1);
    });
}

int vr_ctx_destroy(vr_ctx* ctx) {
    if (!ctx) return VR_OK;
    return guard([&] {
        cudaSetDevice(ctx->device);
        if (ctx->stream) cudaStreamSynchronize(ctx->stream);
        for (vr_ctx* c : ctx->siblings) vr_ctx_destroy(c);  // they share this stream
        ctx->siblings.clear();
        vr::fft_plan_destroy(ctx);
        vr::release_cache(ctx);
        if (ctx->side) cudaStreamSynchronize(ctx->side);
        cudaStreamSynchronize(ctx->stream);
        for (double* p : ctx->spec_scratch) cudaFree(p);
        for (double* p : ctx->field_scratch) cudaFree(p);
        for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
        cudaFree(ctx->red_partials);
        cudaFree(ctx->red_out);
        cudaFreeHost(ctx->red_host);
        cudaFree(ctx->flag_dev);
        cudaFreeHost(ctx->flag_host);
        if (ctx->side) cudaStreamSynchronize(ctx->side);
        if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
        if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
        if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
        if (ctx->ev_halo_fork) cudaEventDestroy(ctx->ev_halo_fork);
        if (ctx->side) cudaStreamDestroy(ctx->side);
        if (ctx->stream && ctx->owns_stream) cudaStreamDestroy(ctx->stream);
        if (ctx->owns_dist) delete ctx->dist;
        delete ctx;
    });
}
int vr_ctx_synchronize(vr_ctx* ctx) {
    return guard([&] {
        set_dev(ctx);
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
void* vr_ctx_stream(vr_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
int vr_ctx_grid(const vr_ctx* ctx, int dims[3]) {
    return guard([&] {
        need(ctx && dims, "vr_ctx_grid");
        dims[0] = ctx->g.n1;
        dims[1] = ctx->g.n2;
        dims[2] = ctx->g.n3;
    });
}
long long vr_ctx_kernel_launches(const vr_ctx* ctx) { return ctx ? ctx->launches : 0; }
void vr_ctx_reset_kernel_launches(vr_ctx* ctx) {
    if (ctx) ctx->launches = 0;
}

int vr_ctx_set_profiling(vr_ctx* ctx, int on) {
    return guard([&] {
        set_dev(ctx);
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        VR_CUDA(cudaStreamSynchronize(ctx->side));
        ctx->profiling = on != 0;
        ctx->prof.clear();
        ctx->ev_used = 0;
    });
}
int vr_ctx_profile_read(vr_ctx* ctx, char* buf, size_t len) {
    return guard([&] {
        set_dev(ctx);
        need(buf && len > 0, "vr_ctx_profile_read");
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        struct Acc {
            long long n = 0;
            double ms = 0.0;
        };
        std::vector<std::pair<std::string, Acc>> acc;
        for (const auto& r : ctx->prof) {
            float ms = 0.f;
            VR_CUDA(cudaEventElapsedTime(&ms, r.start, r.stop));
            const std::string cat = (r.sibling ? "coarse_" : "") + std::string(r.cat);
            auto it = acc.begin();
            for (; it != acc.end(); ++it)
                if (it->first == cat) break;
            if (it == acc.end()) {
                acc.push_back({cat, Acc{}});
                it = acc.end() - 1;
            }
            it->second.n += 1;
            it->second.ms += ms;
        }
        std::string out;
        for (const auto& a : acc)
            out += a.first + "," + std::to_string(a.second.n) + "," + std::to_string(a.second.ms) + "\n";
        std::snprintf(buf, len, "%s", out.c_str());
        ctx->prof.clear();
        ctx->ev_used = 0;
    });
}

// ---- memory -------------------------------------------------------------------
int vr_device_alloc(vr_ctx* ctx, size_t bytes, void** out) {
    return guard([&] {
        set_dev(ctx);
        need(out, "out");
        VR_CUDA(cudaMalloc(out, bytes));
        vr::mem_track_alloc(ctx, *out, static_cast<long long>(bytes));
    });
}
int vr_device_free(vr_ctx* ctx, void* p) {
    return guard([&] {
        set_dev(ctx);
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        vr::mem_track_free(ctx, p);
        VR_CUDA(cudaFree(p));
    });
}
int vr_ctx_memory(const vr_ctx* ctx, long long* live_bytes, long long* peak_bytes,
                  long long* pool_reserved_high) {
    return guard([&] {
        need(ctx != nullptr, "vr_ctx_memory");
        if (live_bytes) *live_bytes = ctx->mem_live;
        if (peak_bytes) *peak_bytes = ctx->mem_peak;
        if (pool_reserved_high) {
            cudaMemPool_t pool;
            unsigned long long v = 0;
            VR_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
            VR_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &v));
            *pool_reserved_high = static_cast<long long>(v);
        }
    });
}
int vr_ctx_reset_memory_peak(vr_ctx* ctx) {
    return guard([&] {
        need(ctx != nullptr, "vr_ctx_reset_memory_peak");
        ctx->mem_peak = ctx->mem_live;
    });
}
int vr_host_alloc_pinned(size_t bytes, void** out) {
    return guard([&] {
        need(out, "out");
        VR_CUDA(cudaMallocHost(out, bytes));
    });
}
int vr_host_free_pinned(void* p) { return guard([&] { VR_CUDA(cudaFreeHost(p)); }); }
int vr_memcpy_h2d(vr_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guard([&] {
        set_dev(ctx);
        VR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    });
}
int vr_memcpy_d2h(vr_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guard([&] {
        set_dev(ctx);
        VR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
int vr_memcpy_d2d(vr_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guard([&] {
        set_dev(ctx);
        VR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    });
}
int vr_memset_zero(vr_ctx* ctx, void* dst, size_t bytes) {
    return guard([&] {
        set_dev(ctx);
        VR_CUDA(cudaMemsetAsync(dst, 0, bytes, ctx->stream));
    });
}

// ---- BLAS-1 ---------------------------------------------------------------------
int vr_scale(vr_ctx* ctx, double* x, int ncomp, double a) {
    return guard([&] {
        set_dev(ctx);
        check_ncomp(ncomp);
        vr::scale(ctx, x, ncomp * ctx->g.N, a);
    });
}
int vr_add_scaled(vr_ctx* ctx, double* y, double a, const double* x, int ncomp) {
    return guard([&] {
        set_dev(ctx);
        check_ncomp(ncomp);
        vr::add_scaled(ctx, y, a, x, ncomp * ctx->g.N);
    });
}
int vr_lin_comb(vr_ctx* ctx, double* out, double a, const double* x, double b, const double* y,
                int ncomp) {
    return guard([&] {
        set_dev(ctx);
        check_ncomp(ncomp);
        vr::lin_comb(ctx, out, a, x, b, y, ncomp * ctx->g.N);
    });
}
int vr_dot_l2(vr_ctx* ctx, const double* a, const double* b, int ncomp, double* out) {
    return guard([&] {
        set_dev(ctx);
        check_ncomp(ncomp);
        double r[3];
        vr::dot_components(ctx, a, b, ctx->g.N, ncomp, r);
        double s = 0.0;
        for (int c = 0; c < ncomp; ++c) s += r[c];
        *out = s;
    });
}
int vr_norm_l2(vr_ctx* ctx, const double* a, int ncomp, double* out) {
    double d = 0.0;
    int st = vr_dot_l2(ctx, a, a, ncomp, &d);
    if (st == VR_OK) *out = std::sqrt(d);
    return st;
}
int vr_max_abs(vr_ctx* ctx, const double* a, int ncomp, double* out) {
    return guard([&] {
        set_dev(ctx);
        check_ncomp(ncomp);
        *out = vr::max_abs(ctx, a, ncomp * ctx->g.N);
    });
}
int vr_max_magnitude(vr_ctx* ctx, const double* v3, double* out) {
    return guard([&] {
        set_dev(ctx);
        *out = vr::max_magnitude(ctx, v3, ctx->g.N);
    });
}
int vr_all_finite(vr_ctx* ctx, const double* a, int ncomp, int* out) {
    return guard([&] {
        set_dev(ctx);
        check_ncomp(ncomp);
        *out = vr::all_finite(ctx, a, ncomp * ctx->g.N) ? 1 : 0;
    });
}
int vr_inner_product(vr_ctx* ctx, const double* a, const double* b, int ncomp, double* out) {
    return guard([&] {
        set_dev(ctx);
        check_ncomp(ncomp);
        *out = ncomp == 3 ? vr::inner_product_vec(ctx, a, b) : vr::inner_product_scalar(ctx, a, b);
    });
}

// ---- spectral -------------------------------------------------------------------
int vr_fft_r2c(vr_ctx* ctx, const double* in, double* out_spectrum) {
    return guard([&] {
        set_dev_single(ctx, "vr_fft_r2c");
        vr::fft_r2c(ctx, in, out_spectrum);
    });
}
int vr_fft_c2r(vr_ctx* ctx, const double* spectrum, double* out) {
    return guard([&] {
        set_dev_single(ctx, "vr_fft_c2r");
        double* s = vr::spec_buf(ctx, 0);
        VR_CUDA(cudaMemcpyAsync(s, spectrum, sizeof(double) * 2 * ctx->g.NC,
                                cudaMemcpyDeviceToDevice, ctx->stream));
        vr::fft_c2r(ctx, s, out, 1.0 / static_cast<double>(ctx->g.Ng), nullptr);
    });
}
int vr_gradient(vr_ctx* ctx, const double* f, double* out3) {
    return guard([&] {
        set_dev(ctx);
        vr::op_gradient(ctx, f, out3);
    });
}
int vr_divergence(vr_ctx* ctx, const double* v3, double* out) {
    return guard([&] {
        set_dev(ctx);
        vr::op_divergence(ctx, v3, out);
    });
}
int vr_laplacian(vr_ctx* ctx, const double* f, double* out, int ncomp) {
    return guard([&] {
        set_dev(ctx);
        check_ncomp(ncomp);
        vr::MultParams mp;
        mp.kind = vr::Mult::laplacian;
        for (int c = 0; c < ncomp; ++c)
            vr::spectral_scalar_op(ctx, f + c * ctx->g.N, out + c * ctx->g.N, mp);
    });
}
int vr_helmholtz1_apply(vr_ctx* ctx, const double* f, double* out) {
    return guard([&] {
        set_dev(ctx);
        vr::MultParams mp;
        mp.kind = vr::Mult::helmholtz1;
        vr::spectral_scalar_op(ctx, f, out, mp);
    });
}
int vr_gaussian_smooth(vr_ctx* ctx, const double* f, double* out, int ncomp,
                       const double sigma[3]) {
    return guard([&] {
        set_dev(ctx);
        check_ncomp(ncomp);
        need(sigma, "sigma");
        for (int a = 0; a < 3; ++a)
            if (sigma[a] < 0.0) vr::throw_argument("gaussian_smooth: sigma must be >= 0");
        vr::MultParams mp;
        mp.kind = vr::Mult::gaussian;
        const double h[3] = {ctx->g.h1, ctx->g.h2, ctx->g.h3};
        for (int a = 0; a < 3; ++a) mp.sig2h2[a] = sigma[a] * sigma[a] * h[a] * h[a];
        for (int c = 0; c < ncomp; ++c)
            vr::spectral_scalar_op(ctx, f + c * ctx->g.N, out + c * ctx->g.N, mp);
    });
}
int vr_apply_reg_operator(vr_ctx* ctx, const double* v3, double* out3, const vr_regnorm* norm,
                          int mode, double beta) {
    return guard([&] {
        set_dev(ctx);
        need(norm, "norm");
        vr_model m;
        vr_model_default(&m);
        m.norm = *norm;
        vr::validate_model(m);
        if (beta <= 0.0) vr::throw_argument("apply_reg_operator: beta must be > 0");
        if (mode < VR_REGOP_APPLY || mode > VR_REGOP_INVERSE_SQRT)
            vr::throw_argument("apply_reg_operator: unknown mode");
        vr::op_reg(ctx, v3, out3, *norm, mode, beta);
    });
}
int vr_apply_projection(vr_ctx* ctx, const double* f3, double* out3, int kind, double beta_v,
                        double beta_w) {
    return guard([&] {
        set_dev(ctx);
        vr::op_projection(ctx, f3, out3, kind, beta_v, beta_w);
    });
}
int vr_rescale_intensity(vr_ctx* ctx, const double* f, double* out, int* degenerate) {
    return guard([&] {
        set_dev_single(ctx, "vr_rescale_intensity");
        const long long N = ctx->g.N;
        const double lo = vr::min_value(ctx, f, N), hi = vr::max_value(ctx, f, N);
        if (hi <= lo) {
            VR_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * N, ctx->stream));
            if (degenerate) *degenerate = 1;
            return;
        }
        vr::affine(ctx, f, out, N, lo, 1.0 / (hi - lo));
        if (degenerate) *degenerate = 0;
    });
}

// ---- transport -------------------------------------------------------------------
int vr_tricubic_interpolate(vr_ctx* ctx, const double* f, const double* pts3, double* out,
                            int nfields) {
    return guard([&] {
        set_dev_single(ctx, "vr_tricubic_interpolate");
        vr::sl_tricubic(ctx, f, nfields, pts3, out);
    });
}
int vr_trace_characteristics(vr_ctx* ctx, const double* v3, int nt, int direction,
                             double* dep3) {
    return guard([&] {
        set_dev_single(ctx, "vr_trace_characteristics");
        if (nt < 1) vr::throw_argument("trace_characteristics: n_t must be >= 1");
        if (!vr::all_finite(ctx, v3, 3 * ctx->g.N))
            vr::throw_numeric("trace_characteristics: velocity has non-finite values");
        vr::sl_trace(ctx, v3, ctx->g.N, nt, direction, dep3);
    });
}
int vr_continuity_factor(vr_ctx* ctx, const double* div_v, const double* dep3, double dt,
                         double* factor) {
    return guard([&] {
        set_dev_single(ctx, "vr_continuity_factor");
        vr::sl_factor(ctx, div_v, dep3, 0.5 * dt, factor);
    });
}
int vr_solve_state(vr_ctx* ctx, const double* m_T, const double* v3, int nt, double* history) {
    return guard([&] {
        set_dev_single(ctx, "vr_solve_state");
        const long long N = ctx->g.N;
        if (nt < 1) vr::throw_argument("trace_characteristics: n_t must be >= 1");
        if (!vr::all_finite(ctx, v3, 3 * N))
            vr::throw_numeric("trace_characteristics: velocity has non-finite values");
        double* xb = vr::dev_alloc(ctx, 3 * N);
        vr::sl_trace(ctx, v3, ctx->g.N, nt, VR_TRACE_BACKWARD, xb);
        VR_CUDA(cudaMemcpyAsync(history, m_T, sizeof(double) * N, cudaMemcpyDeviceToDevice,
                                ctx->stream));
        for (int j = 0; j < nt; ++j) vr::sl_advect(ctx, history + j * N, xb, history + (j + 1) * N);
        vr::dev_free(ctx, xb);
    });
}
// ---- fp32 lane ------------------------------------------------------------------
int vr_tricubic_interpolate_f32(vr_ctx* ctx, const float* f, const float* points3, float* out,
                                int nfields) {
    return guard([&] {
        set_dev_single(ctx, "vr_tricubic_interpolate_f32");
        need(f && points3 && out, "vr_tricubic_interpolate_f32");
        vr::sl_tricubic_f32(ctx, f, nfields, points3, out);
    });
}
int vr_trace_characteristics_f32(vr_ctx* ctx, const float* v3, int nt, int direction,
                                 float* departure3) {
    return guard([&] {
        set_dev_single(ctx, "vr_trace_characteristics_f32");
        need(v3 && departure3, "vr_trace_characteristics_f32");
        if (nt < 1) vr::throw_argument("trace_characteristics: n_t must be >= 1");
        if (!vr::all_finite_f32(ctx, v3, 3 * ctx->g.N))
            vr::throw_numeric("trace_characteristics: velocity has non-finite values");
        vr::sl_trace_f32(ctx, v3, nt, direction, departure3);
    });
}
int vr_solve_state_f32(vr_ctx* ctx, const float* m_T, const float* v3, int nt, float* history) {
    return guard([&] {
        set_dev_single(ctx, "vr_solve_state_f32");
        need(m_T && v3 && history, "vr_solve_state_f32");
        const long long N = ctx->g.N;
        if (nt < 1) vr::throw_argument("trace_characteristics: n_t must be >= 1");
        if (!vr::all_finite_f32(ctx, v3, 3 * N))
            vr::throw_numeric("trace_characteristics: velocity has non-finite values");
        float* xb = nullptr;
        VR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&xb), sizeof(float) * 3 * N, ctx->stream));
        vr::sl_trace_f32(ctx, v3, nt, VR_TRACE_BACKWARD, xb);
        VR_CUDA(cudaMemcpyAsync(history, m_T, sizeof(float) * N, cudaMemcpyDeviceToDevice, ctx->stream));
        for (int j = 0; j < nt; ++j) vr::sl_tricubic_f32(ctx, history + j * N, 1, xb, history + (j + 1) * N);
        VR_CUDA(cudaFreeAsync(xb, ctx->stream));
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// fp32 fields through the fp64 spectral operators: convert at the boundary like the
// reference's float lane (fft.hpp:12-17), one rounding to fp32 at the end
extern "C++" template <class Fn>
void via_f64(vr_ctx* ctx, const float* in, int nin, float* out, int nout, Fn&& fn) {
    const long long N = ctx->g.N;
    double* din = vr::dev_alloc(ctx, nin * N);
    double* dout = out ? vr::dev_alloc(ctx, nout * N) : nullptr;
    try {
        if (in) vr::convert_f2d(ctx, in, din, nin * N);
        fn(din, dout);
        if (out) vr::convert_d2f(ctx, dout, out, nout * N);
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        vr::dev_free(ctx, din);
        vr::dev_free(ctx, dout);
        throw;
    }
    vr::dev_free(ctx, din);
    vr::dev_free(ctx, dout);
}
int vr_fft_r2c_f32(vr_ctx* ctx, const float* in, double* out_spectrum) {
    return guard([&] {
        set_dev_single(ctx, "vr_fft_r2c_f32");
        need(in && out_spectrum, "vr_fft_r2c_f32");
        via_f64(ctx, in, 1, nullptr, 0, [&](double* d, double*) { vr::fft_r2c(ctx, d, out_spectrum); });
    });
}
int vr_fft_c2r_f32(vr_ctx* ctx, const double* spectrum, float* out) {
    return guard([&] {
        set_dev_single(ctx, "vr_fft_c2r_f32");
        need(spectrum && out, "vr_fft_c2r_f32");
        via_f64(ctx, nullptr, 1, out, 1, [&](double*, double* o) {
            double* s = vr::spec_buf(ctx, 0);
            VR_CUDA(cudaMemcpyAsync(s, spectrum, sizeof(double) * 2 * ctx->g.NC,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
            vr::fft_c2r(ctx, s, o, 1.0 / static_cast<double>(ctx->g.Ng), nullptr);
        });
    });
}
int vr_gradient_f32(vr_ctx* ctx, const float* f, float* out3) {
    return guard([&] {
        set_dev_single(ctx, "vr_gradient_f32");
        need(f && out3, "vr_gradient_f32");
        via_f64(ctx, f, 1, out3, 3, [&](double* d, double* o) { vr::op_gradient(ctx, d, o); });
    });
}
int vr_divergence_f32(vr_ctx* ctx, const float* v3, float* out) {
    return guard([&] {
        set_dev_single(ctx, "vr_divergence_f32");
        need(v3 && out, "vr_divergence_f32");
        via_f64(ctx, v3, 3, out, 1, [&](double* d, double* o) { vr::op_divergence(ctx, d, o); });
    });
}
int vr_gaussian_smooth_f32(vr_ctx* ctx, const float* f, float* out, int ncomp,
                           const double sigma[3]) {
    return guard([&] {
        set_dev_single(ctx, "vr_gaussian_smooth_f32");
        need(f && out && sigma, "vr_gaussian_smooth_f32");
        check_ncomp(ncomp);
        for (int a = 0; a < 3; ++a)
            if (sigma[a] < 0.0) vr::throw_argument("gaussian_smooth: sigma must be >= 0");
        vr::MultParams mp;
        mp.kind = vr::Mult::gaussian;
        const double h[3] = {ctx->g.h1, ctx->g.h2, ctx->g.h3};
        for (int a = 0; a < 3; ++a) mp.sig2h2[a] = sigma[a] * sigma[a] * h[a] * h[a];
        via_f64(ctx, f, ncomp, out, ncomp, [&](double* d, double* o) {
            for (int c = 0; c < ncomp; ++c)
                vr::spectral_scalar_op(ctx, d + c * ctx->g.N, o + c * ctx->g.N, mp);
        });
    });
}
int vr_apply_reg_operator_f32(vr_ctx* ctx, const float* v3, float* out3, const vr_regnorm* norm,
                              int mode, double beta) {
    return guard([&] {
        set_dev_single(ctx, "vr_apply_reg_operator_f32");
        need(v3 && out3 && norm, "vr_apply_reg_operator_f32");
        vr_model m;
        vr_model_default(&m);
        m.norm = *norm;
        vr::validate_model(m);
        if (beta <= 0.0) vr::throw_argument("apply_reg_operator: beta must be > 0");
        if (mode < VR_REGOP_APPLY || mode > VR_REGOP_INVERSE_SQRT)
            vr::throw_argument("apply_reg_operator: unknown mode");
        via_f64(ctx, v3, 3, out3, 3, [&](double* d, double* o) { vr::op_reg(ctx, d, o, *norm, mode, beta); });
    });
}
int vr_apply_projection_f32(vr_ctx* ctx, const float* f3, float* out3, int kind, double beta_v,
                            double beta_w) {
    return guard([&] {
        set_dev_single(ctx, "vr_apply_projection_f32");
        need(f3 && out3, "vr_apply_projection_f32");
        via_f64(ctx, f3, 3, out3, 3,
                [&](double* d, double* o) { vr::op_projection(ctx, d, o, kind, beta_v, beta_w); });
    });
}

// ---- Objective<float> --------------------------------------------------------------
static vr::ObjF32* of(vr_objective_f32* o) { return reinterpret_cast<vr::ObjF32*>(o); }
static vr::StateF32* sf(vr_state_f32* s) { return reinterpret_cast<vr::StateF32*>(s); }
static const vr::StateF32* sfc(const vr_state_f32* s) { return reinterpret_cast<const vr::StateF32*>(s); }
int vr_objective_f32_create(vr_ctx* ctx, const float* m_R, const float* m_T, const vr_model* model,
                            vr_objective_f32** out) {
    return guard([&] {
        set_dev_single(ctx, "vr_objective_f32_create");
        need(m_R && m_T && model && out, "vr_objective_f32_create");
        *out = reinterpret_cast<vr_objective_f32*>(vr::objf32_create(ctx, m_R, m_T, *model));
    });
}
int vr_objective_f32_destroy(vr_objective_f32* obj) {
    return guard([&] { vr::objf32_destroy(of(obj)); });
}
int vr_objective_f32_counters(const vr_objective_f32* obj, vr_counters* out) {
    return guard([&] {
        need(obj && out, "vr_objective_f32_counters");
        *out = vr::objf32_counters(reinterpret_cast<const vr::ObjF32*>(obj));
    });
}
int vr_evaluate_f32(vr_objective_f32* obj, const float* v3, vr_state_f32** out_state) {
    return guard([&] {
        need(obj && v3 && out_state, "vr_evaluate_f32");
        set_dev(vr::objf32_ctx(of(obj)));
        *out_state = reinterpret_cast<vr_state_f32*>(vr::objf32_evaluate(of(obj), v3));
    });
}
int vr_state_f32_destroy(vr_state_f32* s) { return guard([&] { vr::statef32_destroy(sf(s)); }); }
int vr_state_f32_scalars(const vr_state_f32* s, double* objective, double* mismatch,
                         double* mismatch_rel) {
    return guard([&] {
        need(s && objective && mismatch && mismatch_rel, "vr_state_f32_scalars");
        vr::statef32_scalars(sfc(s), objective, mismatch, mismatch_rel);
    });
}
int vr_compute_gradient_f32(vr_objective_f32* obj, vr_state_f32* s, float* g3) {
    return guard([&] {
        need(obj && s, "vr_compute_gradient_f32");
        set_dev(vr::objf32_ctx(of(obj)));
        vr::objf32_gradient(of(obj), sf(s));
        if (g3) vr::objf32_copy_gradient(of(obj), sf(s), g3);
    });
}
int vr_hessian_matvec_f32(vr_objective_f32* obj, const vr_state_f32* s, const float* vt3,
                          float* out3) {
    return guard([&] {
        need(obj && s && vt3 && out3, "vr_hessian_matvec_f32");
        set_dev(vr::objf32_ctx(of(obj)));
        vr::objf32_matvec(of(obj), sfc(s), vt3, out3);
    });
}

static void adjoint_like(vr_ctx* ctx, const double* terminal, const double* v3, int nt,
                         double* history, double* initial) {
    const long long N = ctx->g.N;
    if (nt < 1) vr::throw_argument("trace_characteristics: n_t must be >= 1");
    if (!vr::all_finite(ctx, v3, 3 * N))
        vr::throw_numeric("trace_characteristics: velocity has non-finite values");
    double* xf = vr::dev_alloc(ctx, 3 * N);
    double* factor = vr::dev_alloc(ctx, N);
    double* work = vr::dev_alloc(ctx, 2 * N);
    vr::sl_trace(ctx, v3, ctx->g.N, nt, VR_TRACE_FORWARD, xf);
    double* div = vr::field_buf(ctx, 0);
    vr::op_divergence(ctx, v3, div);
    vr::sl_factor(ctx, div, xf, 0.5 / nt, factor);
    const double* cur = terminal;
    if (history)
        VR_CUDA(cudaMemcpyAsync(history + nt * N, terminal, sizeof(double) * N,
                                cudaMemcpyDeviceToDevice, ctx->stream));
    int pp = 0;
    for (int j = nt - 1; j >= 0; --j) {
        double* dst = history ? history + j * N : work + pp * N;
        vr::sl_continuity(ctx, cur, xf, factor, dst);
        cur = dst;
        pp ^= 1;
    }
    if (initial)
        VR_CUDA(cudaMemcpyAsync(initial, cur, sizeof(double) * N, cudaMemcpyDeviceToDevice,
                                ctx->stream));
    VR_CUDA(cudaStreamSynchronize(ctx->stream));
    vr::dev_free(ctx, xf);
    vr::dev_free(ctx, factor);
    vr::dev_free(ctx, work);
}
int vr_solve_adjoint(vr_ctx* ctx, const double* terminal, const double* v3, int nt,
                     double* history, double* initial) {
    return guard([&] {
        set_dev_single(ctx, "vr_solve_adjoint");
        adjoint_like(ctx, terminal, v3, nt, history, initial);
    });
}
int vr_solve_inc_adjoint(vr_ctx* ctx, const double* terminal, const double* v3, int nt,
                         double* history, double* initial) {
    return guard([&] {
        set_dev_single(ctx, "vr_solve_inc_adjoint");
        adjoint_like(ctx, terminal, v3, nt, history, initial);
    });
}
int vr_gradient_dot(vr_ctx* ctx, const double* f, const double* w3, double* out) {
    return guard([&] {
        set_dev_single(ctx, "vr_gradient_dot");
        double* gm = vr::dev_alloc(ctx, 3 * ctx->g.N);
        vr::op_gradient(ctx, f, gm);
        vr::sl_gradient_dot(ctx, gm, w3, out);
        vr::dev_free(ctx, gm);
    });
}
int vr_solve_inc_state(vr_ctx* ctx, const double* m_history, const double* v3, const double* vt3,
                       int nt, double* mt_history) {
    // step-by-step restatement of transport.cpp:150-173 (the fused matvec path
    // lives in objective.cu; this entry point returns the whole mt history)
    return guard([&] {
        set_dev_single(ctx, "vr_solve_inc_state");
        const long long N = ctx->g.N;
        if (nt < 1) vr::throw_argument("trace_characteristics: n_t must be >= 1");
        double* xb = vr::dev_alloc(ctx, 3 * N);
        double* gm = vr::dev_alloc(ctx, 3 * N);
        double* q = vr::dev_alloc(ctx, 2 * N);
        double* tmp = vr::dev_alloc(ctx, N);
        vr::sl_trace(ctx, v3, ctx->g.N, nt, VR_TRACE_BACKWARD, xb);
        const double hdt = 0.5 / nt;
        double* qp = q;
        double* qn = q + N;
        vr::op_gradient(ctx, m_history, gm);
        vr::sl_gradient_dot(ctx, gm, vt3, qp);
        VR_CUDA(cudaMemsetAsync(mt_history, 0, sizeof(double) * N, ctx->stream));
        for (int j = 0; j < nt; ++j) {
            vr::op_gradient(ctx, m_history + (j + 1) * N, gm);
            vr::sl_gradient_dot(ctx, gm, vt3, qn);
            vr::lin_comb(ctx, tmp, 1.0, mt_history + j * N, -hdt, qp, N);
            vr::sl_advect(ctx, tmp, xb, mt_history + (j + 1) * N);
            vr::add_scaled(ctx, mt_history + (j + 1) * N, -hdt, qn, N);
            std::swap(qp, qn);
        }
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        vr::dev_free(ctx, xb);
        vr::dev_free(ctx, gm);
        vr::dev_free(ctx, q);
        vr::dev_free(ctx, tmp);
    });
}

// ---- objective -------------------------------------------------------------------
int vr_objective_create(vr_ctx* ctx, const double* m_R, const double* m_T, const vr_model* model,
                        vr_objective** out) {
    return guard([&] {
        set_dev(ctx);
        need(m_R && m_T && model && out, "vr_objective_create");
        *out = vr::objective_create(ctx, m_R, m_T, *model);
    });
}
int vr_objective_destroy(vr_objective* obj) {
    return guard([&] {
        if (obj) {
            cudaSetDevice(obj->ctx->device);
            delete obj;
        }
    });
}
int vr_objective_initial_mismatch(const vr_objective* obj, double* out) {
    return guard([&] {
        need(obj && out, "vr_objective_initial_mismatch");
        *out = obj->initial_mismatch;
    });
}
int vr_objective_counters(const vr_objective* obj, vr_counters* out) {
    return guard([&] {
        need(obj && out, "vr_objective_counters");
        *out = obj->counters;
    });
}
int vr_objective_reset_counters(vr_objective* obj) {
    return guard([&] {
        need(obj, "vr_objective_reset_counters");
        obj->counters = vr_counters{};
    });
}
int vr_objective_set_beta(vr_objective* obj, double beta_v) {
    return guard([&] {
        need(obj, "vr_objective_set_beta");
        if (beta_v <= 0.0) vr::throw_argument("RegModel: beta_v must be > 0");
        obj->model.beta_v = beta_v;
    });
}
// every objective entry point first completes pipelined host-buffer matvecs
// (vr_hessian_matvec_host_async), so their deferred non-finite check cannot be lost
static void drain_pipe(vr_objective* obj) {
    if (obj->pipe.issued) vr::objective_pipe_wait(obj);
}
int vr_evaluate(vr_objective* obj, const double* v3, vr_state** out_state) {
    return guard([&] {
        need(obj && v3 && out_state, "vr_evaluate");
        set_dev(obj->ctx);
        drain_pipe(obj);
        *out_state = vr::objective_evaluate(obj, v3);
    });
}
int vr_state_destroy(vr_state* s) {
    return guard([&] {
        if (s) {
            cudaSetDevice(s->obj->ctx->device);
            delete s;
        }
    });
}
int vr_state_scalars(const vr_state* s, double* objective, double* mismatch, double* mismatch_rel,
                     int* has_gradient, int* has_adjoint_ctx) {
    return guard([&] {
        need(s, "vr_state_scalars");
        if (objective) *objective = s->objective;
        if (mismatch) *mismatch = s->mismatch;
        if (mismatch_rel) *mismatch_rel = s->mismatch_rel;
        if (has_gradient) *has_gradient = s->has_gradient;
        if (has_adjoint_ctx) *has_adjoint_ctx = s->has_adjoint_ctx;
    });
}
int vr_state_get(const vr_state* s, int which, double* out) {
    return guard([&] {
        need(s && out, "vr_state_get");
        vr_ctx* ctx = s->obj->ctx;
        set_dev(ctx);
        const long long N = ctx->g.N;
        const double* src = nullptr;
        long long n = 0;
        switch (which) {
            case VR_STATE_V: src = s->v; n = 3 * N; break;
            case VR_STATE_X_BWD: src = s->xb; n = 3 * N; break;
            case VR_STATE_X_FWD: src = s->xf; n = 3 * N; break;
            case VR_STATE_FACTOR: src = s->factor; n = N; break;
            case VR_STATE_M_HISTORY:  // halo-padded series: copy slice by slice
                for (int j = 0; j <= s->nt; ++j)
                    VR_CUDA(cudaMemcpyAsync(out + j * N, vr::pslice(ctx, s->mhist, j),
                                            sizeof(double) * N, cudaMemcpyDeviceToDevice,
                                            ctx->stream));
                return;
            case VR_STATE_GRADIENT: src = s->has_gradient ? s->grad : nullptr; n = 3 * N; break;
            case VR_STATE_GRAD_M: src = s->gradm; n = 3LL * (s->nt + 1) * N; break;
            case VR_STATE_LAMBDA_HISTORY:
                if (!s->lamhist) vr::throw_logic("vr_state_get: field not computed yet");
                for (int j = 0; j <= s->nt; ++j)
                    VR_CUDA(cudaMemcpyAsync(out + j * N, vr::pslice(ctx, s->lamhist, j),
                                            sizeof(double) * N, cudaMemcpyDeviceToDevice,
                                            ctx->stream));
                return;
            default: vr::throw_argument("vr_state_get: unknown field");
        }
        if (!src) vr::throw_logic("vr_state_get: field not computed yet");
        VR_CUDA(cudaMemcpyAsync(out, src, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                ctx->stream));
    });
}
int vr_compute_gradient(vr_objective* obj, vr_state* s, double* g3) {
    return guard([&] {
        need(obj && s, "vr_compute_gradient");
        set_dev(obj->ctx);
        drain_pipe(obj);
        vr::objective_gradient(obj, s);
        if (g3)
            VR_CUDA(cudaMemcpyAsync(g3, s->grad, sizeof(double) * 3 * obj->ctx->g.N,
                                    cudaMemcpyDeviceToDevice, obj->ctx->stream));
    });
}
int vr_hessian_matvec(vr_objective* obj, const vr_state* s, const double* vt3, double* out3) {
    return guard([&] {
        need(obj && s && vt3 && out3, "vr_hessian_matvec");
        set_dev(obj->ctx);
        drain_pipe(obj);
        vr::objective_matvec(obj, s, vt3, out3, true);
        vr::drain_flags(obj->ctx);  // the public call reports a non-finite direction itself
    });
}
int vr_hessian_data_matvec(vr_objective* obj, const vr_state* s, const double* vt3, double* out3) {
    return guard([&] {
        need(obj && s && vt3 && out3, "vr_hessian_data_matvec");
        set_dev(obj->ctx);
        drain_pipe(obj);
        vr::objective_matvec(obj, s, vt3, out3, false);
        vr::drain_flags(obj->ctx);
    });
}
int vr_hessian_matvec_host(vr_objective* obj, const vr_state* s, const double* vt3_host,
                           double* out3_host) {
    return guard([&] {
        need(obj && s && vt3_host && out3_host, "vr_hessian_matvec_host");
        vr_ctx* ctx = obj->ctx;
        set_dev(ctx);
        drain_pipe(obj);
        const size_t bytes = sizeof(double) * 3 * ctx->g.N;
        if (!obj->host_vt) obj->host_vt = vr::dev_alloc(ctx, 3 * ctx->g.N);
        if (!obj->host_out) obj->host_out = vr::dev_alloc(ctx, 3 * ctx->g.N);
        VR_CUDA(cudaMemcpyAsync(obj->host_vt, vt3_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
        vr::objective_matvec(obj, s, obj->host_vt, obj->host_out, true);
        VR_CUDA(cudaMemcpyAsync(out3_host, obj->host_out, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        vr::flags_enqueue_copy(ctx);  // the flags ride on the download's synchronisation
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        vr::flags_after_sync(ctx);
    });
}
int vr_hessian_matvec_host_async(vr_objective* obj, const vr_state* s, const double* vt3_host,
                                 double* out3_host) {
    return guard([&] {
        need(obj && s && vt3_host && out3_host, "vr_hessian_matvec_host_async");
        set_dev(obj->ctx);
        vr::objective_matvec_host_async(obj, s, vt3_host, out3_host);
    });
}
int vr_objective_wait(vr_objective* obj) {
    return guard([&] {
        need(obj, "vr_objective_wait");
        set_dev(obj->ctx);
        vr::objective_pipe_wait(obj);
    });
}
int vr_objective_apply_reg(vr_objective* obj, const double* u3, int mode, double* out3) {
    return guard([&] {
        need(obj && u3 && out3, "vr_objective_apply_reg");
        set_dev(obj->ctx);
        drain_pipe(obj);
        vr::objective_apply_reg(obj, u3, mode, out3);
    });
}
int vr_objective_apply_K(vr_objective* obj, const double* u3, double* out3) {
    return guard([&] {
        need(obj && u3 && out3, "vr_objective_apply_K");
        set_dev(obj->ctx);
        drain_pipe(obj);
        vr::objective_apply_K(obj, u3, out3);
    });
}

// ---- solvers ----------------------------------------------------------------------
// SolveReport::write_csv (solver.cpp:29-47): optional "# comment" line, the header, one
// row per IterationRecord, precision 17 -- so GPU and CPU reports diff column by column
int vr_solve_report_csv(const vr_solve_report* report, const vr_iteration_record* records,
                        const char* comment, char* buf, size_t len, size_t* needed) {
    return guard([&] {
        need(report != nullptr && (records != nullptr || report->n_records == 0), "vr_solve_report_csv");
        std::ostringstream os;
        if (comment) os << "# " << comment << "\n";
        os << "iter,objective,mismatch_rel,grad_norm,grad_rel,step_length,forcing,"
              "inner_iterations,fine_matvecs,coarse_matvecs,pde_solves,wall_time_s\n";
        std::ostringstream row;
        row.precision(17);
        for (int i = 0; i < report->n_records; ++i) {
            const vr_iteration_record& r = records[i];
            row.str("");
            row << r.k << ',' << r.objective << ',' << r.mismatch_rel << ',' << r.grad_norm << ','
                << r.grad_rel << ',' << r.step_length << ',' << r.forcing << ',' << r.inner_iterations
                << ',' << r.fine_matvecs << ',' << r.coarse_matvecs << ',' << r.pde_solves << ','
                << r.wall_time_s;
            os << row.str() << "\n";
        }
        const std::string out = os.str();
        if (needed) *needed = out.size() + 1;
        if (buf && len > 0) {
            if (out.size() + 1 > len) vr::throw_argument("vr_solve_report_csv: buffer too small");
            std::memcpy(buf, out.c_str(), out.size() + 1);
        }
    });
}
int vr_compute_forcing(double grad_norm, double grad0_norm, double* out) {
    return guard([&] {
        if (grad0_norm <= 0.0)
            vr::throw_logic("compute_forcing: |g_0| = 0, the solver should have terminated");
        *out = std::min(0.5, std::sqrt(grad_norm / grad0_norm));
    });
}
int vr_pcg_solve(vr_objective* obj, const vr_state* s, const double* rhs3, double rel_tol,
                 int max_iter, int precond, double* x3, vr_pcg_stats* stats) {
    return guard([&] {
        need(obj && s && rhs3 && x3 && stats, "vr_pcg_solve");
        vr_ctx* ctx = obj->ctx;
        set_dev(ctx);
        drain_pipe(obj);
        const long long n3 = 3 * ctx->g.N;
        vr::DevOp op = [&](const double* u, double* out) {
            vr::objective_matvec(obj, s, u, out, true);
        };
        vr::DevOp pc = [&](const double* r, double* z) {
            if (precond == VR_PRECOND_SPECTRAL)
                vr::objective_apply_reg(obj, r, VR_REGOP_INVERSE, z);
            else
                VR_CUDA(cudaMemcpyAsync(z, r, sizeof(double) * n3, cudaMemcpyDeviceToDevice,
                                        ctx->stream));
        };
        *stats = precond == VR_PRECOND_SPECTRAL
                     ? vr::pcg_solve_gn(obj, s, rhs3, rel_tol, max_iter, x3)
                     : vr::pcg_solve(ctx, op, rhs3, rel_tol, max_iter, pc, x3);
        vr::drain_flags(ctx);
    });
}
static void copy_records(const vr::GnResult& r, vr_iteration_record* recs, int max_recs,
                         int offset) {
    if (!recs) return;
    for (size_t i = 0; i < r.records.size(); ++i) {
        const int slot = offset + static_cast<int>(i);
        if (slot >= max_recs) break;
        recs[slot] = r.records[i];
    }
}
int vr_gauss_newton_solve(vr_ctx* ctx, const double* m_R, const double* m_T, const double* v0,
                          const vr_model* model, const vr_solver_params* params, int precond,
                          double* v_out, vr_solve_report* report, vr_iteration_record* records,
                          int max_records) {
    return guard([&] {
        set_dev(ctx);
        need(m_R && m_T && v0 && model && params && v_out && report, "vr_gauss_newton_solve");
        vr::GnResult r = vr::gauss_newton_solve(ctx, m_R, m_T, v0, *model, *params, precond, v_out);
        *report = r.report;
        copy_records(r, records, max_records, 0);
    });
}
int vr_gauss_newton_solve_f32(vr_ctx* ctx, const float* m_R, const float* m_T, const float* v0,
                              const vr_model* model, const vr_solver_params* params, int precond,
                              float* v_out, vr_solve_report* report, vr_iteration_record* records,
                              int max_records) {
    return guard([&] {
        set_dev_single(ctx, "vr_gauss_newton_solve_f32");
        need(m_R && m_T && v0 && model && params && v_out && report, "vr_gauss_newton_solve_f32");
        vr::GnResult r = vr::gauss_newton_solve_f32(ctx, m_R, m_T, v0, *model, *params, precond, v_out);
        *report = r.report;
        copy_records(r, records, max_records, 0);
    });
}

int vr_gauss_newton_solve_two_level_f32(vr_ctx* ctx, const float* m_R, const float* m_T, const float* v0,
                                        const vr_model* model, const vr_solver_params* params,
                                        const vr_twolevel_options* opts, float* v_out,
                                        vr_solve_report* report, vr_iteration_record* records,
                                        int max_records) {
    return guard([&] {
        set_dev_single(ctx, "vr_gauss_newton_solve_two_level_f32");
        need(m_R && m_T && v0 && model && params && v_out && report, "vr_gauss_newton_solve_two_level_f32");
        vr::GnResult r = vr::gauss_newton_solve_f32(ctx, m_R, m_T, v0, *model, *params, VR_PRECOND_TWO_LEVEL,
                                                    v_out, opts);
        *report = r.report;
        copy_records(r, records, max_records, 0);
    });
}

int vr_parameter_continuation_f32(vr_ctx* ctx, const float* m_R, const float* m_T, const float* v0,
                                  const vr_model* model, const vr_solver_params* params,
                                  int precond, float* v_out, vr_solve_report* reports,
                                  int max_levels, int* n_levels, vr_iteration_record* records,
                                  int max_records) {
    return guard([&] {
        set_dev_single(ctx, "vr_parameter_continuation_f32");
        need(m_R && m_T && v0 && model && params && v_out && n_levels, "vr_parameter_continuation_f32");
        auto rs = vr::parameter_continuation_f32(ctx, m_R, m_T, v0, *model, *params, precond, v_out);
        int off = 0;
        for (size_t l = 0; l < rs.size(); ++l) {
            if (reports && static_cast<int>(l) < max_levels) reports[l] = rs[l].report;
            copy_records(rs[l], records, max_records, off);
            off += static_cast<int>(rs[l].records.size());
        }
        *n_levels = static_cast<int>(rs.size());
    });
}
int vr_parameter_continuation(vr_ctx* ctx, const double* m_R, const double* m_T, const double* v0,
                              const vr_model* model, const vr_solver_params* params, int precond,
                              double* v_out, vr_solve_report* reports, int max_levels,
                              int* n_levels, vr_iteration_record* records, int max_records) {
    return guard([&] {
        set_dev(ctx);
        need(m_R && m_T && v0 && model && params && v_out && n_levels, "vr_parameter_continuation");
        if (!(model->beta_v <= 1.0))
            vr::throw_argument("parameter continuation: target beta_v > 1");
        std::vector<double> levels;
        for (int i = 0;; ++i) {
            const double b = std::pow(10.0, -i);
            if (b <= model->beta_v * (1.0 + 1e-9)) break;
            levels.push_back(b);
        }
        levels.push_back(model->beta_v);
        const long long n3 = 3 * ctx->g.N;
        double* v = vr::dev_alloc(ctx, n3);
        VR_CUDA(cudaMemcpyAsync(v, v0, sizeof(double) * n3, cudaMemcpyDeviceToDevice, ctx->stream));
        int off = 0;
        *n_levels = 0;
        try {
            for (size_t l = 0; l < levels.size(); ++l) {
                vr_model m = *model;
                m.beta_v = levels[l];
                vr::GnResult r = vr::gauss_newton_solve(ctx, m_R, m_T, v, m, *params, precond, v);
                if (reports && static_cast<int>(l) < max_levels) reports[l] = r.report;
                copy_records(r, records, max_records, off);
                off += static_cast<int>(r.records.size());
                *n_levels = static_cast<int>(l) + 1;
                if (r.report.stop == VR_STOP_LINE_SEARCH_FAILURE) break;
            }
            VR_CUDA(cudaMemcpyAsync(v_out, v, sizeof(double) * n3, cudaMemcpyDeviceToDevice,
                                    ctx->stream));
            VR_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            vr::dev_free(ctx, v);
            throw;
        }
        vr::dev_free(ctx, v);
    });
}

// ---- continuation / beta search / postprocess (postprocess.cu) ------------------
static void copy_levels(const std::vector<vr::GnResult>& rs, vr_solve_report* reports, int max_levels,
                        int* n_levels, vr_iteration_record* records, int max_records) {
    int off = 0;
    for (size_t l = 0; l < rs.size(); ++l) {
        if (reports && static_cast<int>(l) < max_levels) reports[l] = rs[l].report;
        copy_records(rs[l], records, max_records, off);
        off += static_cast<int>(rs[l].records.size());
    }
    *n_levels = static_cast<int>(rs.size());
}
int vr_grid_continuation(vr_ctx* ctx, const double* m_R, const double* m_T, const double* v0,
                         const vr_model* model, const vr_solver_params* params, int precond,
                         int n_grid_levels, double* v_out, vr_solve_report* reports,
                         int max_levels, int* n_levels, vr_iteration_record* records,
                         int max_records) {
    return guard([&] {
        set_dev(ctx);  // one GPU or x1 slabs
        need(m_R && m_T && v0 && model && params && v_out && n_levels, "vr_grid_continuation");
        copy_levels(vr::grid_continuation(ctx, m_R, m_T, v0, *model, *params, precond, n_grid_levels, v_out),
                    reports, max_levels, n_levels, records, max_records);
    });
}
int vr_scale_continuation(vr_ctx* ctx, const double* m_R, const double* m_T, const double* v0,
                          const vr_model* model, const vr_solver_params* params, int precond,
                          const double* sigmas, int n_sigmas, double* v_out,
                          vr_solve_report* reports, int max_levels, int* n_levels,
                          vr_iteration_record* records, int max_records) {
    return guard([&] {
        set_dev(ctx);
        need(m_R && m_T && v0 && model && params && sigmas && v_out && n_levels, "vr_scale_continuation");
        copy_levels(vr::scale_continuation(ctx, m_R, m_T, v0, *model, *params, precond, sigmas, n_sigmas, v_out),
                    reports, max_levels, n_levels, records, max_records);
    });
}
void vr_beta_search_params_default(vr_beta_search_params* p) {
    p->eps_J = 0.1;  // H2 (Table 2); 0.25 for H1-div
    p->beta_lo = 1e-5;
    p->beta_hi = 1.0;
    p->max_bisections = 10;
    p->min_width_decades = 0.25;
}
int vr_beta_search(vr_ctx* ctx, const double* m_R, const double* m_T, const double* v0,
                   const vr_model* model, const vr_solver_params* params, int precond,
                   const vr_beta_search_params* bp, double* beta_out, double* v_out,
                   vr_beta_trial* trials, int max_trials, int* n_trials) {
    return guard([&] {
        set_dev(ctx);  // one GPU or x1 slabs
        need(m_R && m_T && v0 && model && params && bp && beta_out && v_out && n_trials, "vr_beta_search");
        vr::BetaSearch r = vr::beta_search(ctx, m_R, m_T, v0, *model, *params, precond, *bp, v_out);
        *n_trials = static_cast<int>(r.trials.size());
        for (int t = 0; t < *n_trials && t < max_trials; ++t) trials[t] = r.trials[t];
        *beta_out = r.beta;
        if (!r.found)
            vr::throw_numeric("beta search: no feasible beta_v in [" + std::to_string(bp->beta_lo) + ", " +
                              std::to_string(bp->beta_hi) + "] (det grad y bound " + std::to_string(bp->eps_J) + ")");
    });
}
int vr_det_deformation_gradient(vr_ctx* ctx, const double* v3, int nt, double* det) {
    return guard([&] {
        set_dev(ctx);  // one GPU or x1 slabs
        need(v3 && det, "vr_det_deformation_gradient");
        vr::det_deformation_gradient(ctx, v3, nt, det);
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
int vr_deformation_map(vr_ctx* ctx, const double* v3, int nt, int absolute, double* out3) {
    return guard([&] {
        set_dev(ctx);  // one GPU or x1 slabs
        need(v3 && out3, "vr_deformation_map");
        vr::deformation_map(ctx, v3, nt, absolute != 0, out3);
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
int vr_det_stats(vr_ctx* ctx, const double* det, const double* foreground, double threshold,
                 vr_det_summary* out) {
    return guard([&] {
        set_dev(ctx);  // one GPU or x1 slabs
        need(det && out, "vr_det_stats");
        *out = vr::det_stats(ctx, det, foreground, threshold);
    });
}
int vr_transport_labels(vr_ctx* ctx, const double* labels, const double* v3, int nt,
                        double* out) {
    return guard([&] {
        set_dev(ctx);  // one GPU or x1 slabs
        need(labels && v3 && out, "vr_transport_labels");
        vr::transport_labels(ctx, labels, v3, nt, out);
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
int vr_overlap_scores(vr_ctx* ctx, const double* reference, const double* test,
                      const double* mask, int max_labels, int* n_labels, int* codes,
                      vr_overlap* per_label, vr_overlap* union_scores) {
    return guard([&] {
        set_dev(ctx);  // one GPU or x1 slabs
        need(reference && test && n_labels, "vr_overlap_scores");
        *n_labels = vr::overlap_scores(ctx, reference, test, mask, max_labels, codes, per_label,
                                       union_scores);
    });
}

// ---- two-level preconditioner / grid transfer ----------------------------------
struct vr_twolevel {
    explicit vr_twolevel(const vr_twolevel_options& o) : tl(o) {}
    vr::TwoLevel tl;
};
int vr_spectral_resample(vr_ctx* src, const double* in, int ncomp, vr_ctx* dst, double* out) {
    return guard([&] {
        set_dev(src);
        need(dst && in && out, "vr_spectral_resample");
        check_ncomp(ncomp);
        for (int c = 0; c < ncomp; ++c)
            vr::resample_scalar(src, in + c * src->g.N, dst, out + c * dst->g.N);
    });
}
int vr_frequency_filter(vr_ctx* ctx, const double* in, int ncomp, int band, const int cutoff[3],
                        double* out) {
    return guard([&] {
        set_dev(ctx);
        need(in && out && cutoff, "vr_frequency_filter");
        check_ncomp(ncomp);
        if (band != 0 && band != 1) vr::throw_argument("frequency_filter: band must be 0 or 1");
        for (int c = 0; c < ncomp; ++c)
            vr::frequency_filter(ctx, in + c * ctx->g.N, band, cutoff, out + c * ctx->g.N);
    });
}
int vr_split_matvec(vr_objective* obj, const vr_state* state, const double* w3, double* out3) {
    return guard([&] {
        need(obj && state && w3 && out3, "vr_split_matvec");
        set_dev(obj->ctx);
        drain_pipe(obj);
        if (!state->has_adjoint_ctx)
            vr::throw_logic("split_matvec: evaluation context is missing the adjoint sweep data "
                            "(compute the gradient first)");
        vr::split_matvec(obj, state, w3, out3);
        vr::drain_flags(obj->ctx);
    });
}
int vr_twolevel_create(const vr_twolevel_options* opts, vr_twolevel** out) {
    return guard([&] {
        need(out != nullptr, "vr_twolevel_create");
        vr_twolevel_options d;
        vr_twolevel_options_default(&d);
        *out = new vr_twolevel(opts ? *opts : d);
    });
}
int vr_twolevel_destroy(vr_twolevel* tl) {
    return guard([&] { delete tl; });
}
int vr_twolevel_rebuild(vr_twolevel* tl, vr_objective* obj, const vr_state* state, double eps_H) {
    return guard([&] {
        need(tl && obj && state, "vr_twolevel_rebuild");
        set_dev(obj->ctx);
        drain_pipe(obj);
        tl->tl.rebuild(obj, state, eps_H);
    });
}
int vr_twolevel_apply(vr_twolevel* tl, vr_ctx* ctx, const double* r3, double* z3) {
    return guard([&] {
        need(tl && r3 && z3, "vr_twolevel_apply");
        set_dev(ctx);
        tl->tl.apply(ctx, r3, z3);
        vr::drain_flags(ctx);
        if (tl->tl.cctx) vr::drain_flags(tl->tl.cctx);
    });
}
int vr_twolevel_coarse_matvec(vr_twolevel* tl, const double* u3, double* out3) {
    return guard([&] {
        need(tl && u3 && out3, "vr_twolevel_coarse_matvec");
        tl->tl.coarse_matvec(u3, out3);
        if (tl->tl.cctx) vr::drain_flags(tl->tl.cctx);
    });
}
int vr_twolevel_info(const vr_twolevel* tl, int dims[3], int* lanczos_runs, int* inner_diverged,
                     double bounds[2], vr_counters* coarse) {
    return guard([&] {
        need(tl != nullptr, "vr_twolevel_info");
        const vr::TwoLevel& t = tl->tl;
        if (dims) {
            dims[0] = t.cctx ? t.cctx->g.n1 : 0;
            dims[1] = t.cctx ? t.cctx->g.n2 : 0;
            dims[2] = t.cctx ? t.cctx->g.n3 : 0;
        }
        if (lanczos_runs) *lanczos_runs = t.lanczos_runs;
        if (inner_diverged) *inner_diverged = t.inner_diverged;
        if (bounds) bounds[0] = t.bounds.first, bounds[1] = t.bounds.second;
        if (coarse) *coarse = t.counters();
    });
}
int vr_gauss_newton_solve_two_level(vr_ctx* ctx, const double* m_R, const double* m_T,
                                    const double* v0, const vr_model* model,
                                    const vr_solver_params* params,
                                    const vr_twolevel_options* opts, double* v_out,
                                    vr_solve_report* report, vr_iteration_record* records,
                                    int max_records) {
    return guard([&] {
        set_dev(ctx);
        need(m_R && m_T && v0 && model && params && v_out && report,
             "vr_gauss_newton_solve_two_level");
        vr::GnResult r = vr::gauss_newton_solve(ctx, m_R, m_T, v0, *model, *params,
                                                VR_PRECOND_TWO_LEVEL, v_out, opts);
        *report = r.report;
        copy_records(r, records, max_records, 0);
    });
}

int vr_generate_synthetic(vr_ctx* ctx, int nt, double amplitude, double* m_R, double* m_T,
                          double* v_star) {
    return guard([&] {
        set_dev_single(ctx, "vr_generate_synthetic");
        need(m_R && m_T && v_star, "vr_generate_synthetic");
        const long long N = ctx->g.N;
        vr::synth_fill(ctx, amplitude, m_T, v_star);
        double* xb = vr::dev_alloc(ctx, 3 * N);
        double* a = vr::dev_alloc(ctx, N);
        double* b = vr::dev_alloc(ctx, N);
        vr::sl_trace(ctx, v_star, ctx->g.N, nt, VR_TRACE_BACKWARD, xb);
        const double* cur = m_T;
        double* bufs[2] = {a, b};
        for (int j = 0; j < nt; ++j) {
            double* dst = (j + 1 == nt) ? m_R : bufs[j & 1];
            vr::sl_advect(ctx, cur, xb, dst);
            cur = dst;
        }
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        vr::dev_free(ctx, xb);
        vr::dev_free(ctx, a);
        vr::dev_free(ctx, b);
    });
}

}  // extern "C"
