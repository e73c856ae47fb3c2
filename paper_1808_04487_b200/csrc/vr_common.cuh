// vr_common.cuh -- shared types for the sm_100a operator layer.
//
// Layout contract (reference proj/include/veloreg/grid.hpp:17-19, field.hpp:101-151):
// fp64 scalar fields are N = n1*n2*n3 doubles, row-major, axis 0 slowest; vector
// fields are 3 scalar fields back to back; half spectra are (n1, n2, n3/2+1)
// complex128 (fft.hpp:12-23).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <map>
#include <unordered_map>
#include <vector>

#include "veloreg_gpu.h"

namespace vr {

constexpr double kTwoPi = 6.283185307179586476925286766559;

// VR_TIMING diagnostics: host operations (allocations, synchronisations) that take longer
// than VR_SLOW_MS (default 20 ms) are reported on stderr with their name
bool timing_enabled();
void slow_op(const char* what, double ms);

// NVTX range per operator / solver phase (visible in nsys / ncu --nvtx timelines; a
// no-op unless a tool injects the NVTX handler)
struct Range {
    explicit Range(const char* name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
    Range(const Range&) = delete;
    Range& operator=(const Range&) = delete;
};

// ---------------------------------------------------------------------------
// Errors: mirror veloreg::Error categories (errors.hpp:9-67)
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    int status;
    int cls;
    Error(int s, int c, const std::string& m) : std::runtime_error(m), status(s), cls(c) {}
};
[[noreturn]] inline void throw_argument(const std::string& m) {
    throw Error(VR_ERR_ARGUMENT, VR_EXC_ARGUMENT, m);
}
[[noreturn]] inline void throw_dimension(const std::string& m) {
    throw Error(VR_ERR_ARGUMENT, VR_EXC_DIMENSION, m);
}
[[noreturn]] inline void throw_numeric(const std::string& m) {
    throw Error(VR_ERR_NUMERICS, VR_EXC_NUMERIC, m);
}
[[noreturn]] inline void throw_logic(const std::string& m) {
    throw Error(VR_ERR_LOGIC, VR_EXC_LOGIC, m);
}
[[noreturn]] inline void throw_resource(const std::string& m) {
    throw Error(VR_ERR_RESOURCE, VR_EXC_RESOURCE, m);
}

#define VR_CUDA(call)                                                                          \
    do {                                                                                       \
        cudaError_t vr_e_ = (call);                                                            \
        if (vr_e_ != cudaSuccess)                                                              \
            ::vr::throw_resource(std::string(#call) + ": " + cudaGetErrorString(vr_e_));       \
    } while (0)

// ---------------------------------------------------------------------------
// Grid (Grid3, grid.hpp:20-56) as passed to kernels by value
// ---------------------------------------------------------------------------
// On one GPU L = n1, off1 = 0, halo = 0, n2s = n2, k2_off = 0, dist = 0. With P
// x1 slabs rank r owns planes [off1, off1 + L), L = n1/P;
// gathered fields carry `halo` planes on each side; the x1 FFT pass runs on the
// k2-slab [n1][n2s][nh] (n2s = n2/P, first column k2_off).
struct GridDims {
    int n1, n2, n3;     // global grid (Grid3)
    int nh;             // n3/2 + 1
    int L;              // x1 planes owned here
    int off1;           // global index of the first owned plane
    int halo;           // halo planes on each side of gathered fields
    int n2s;            // k2 extent of the x1-pass spectrum layout
    int k2_off;         // global k2 of its first column
    int dist;           // 1 when x1-slab decomposed across ranks
    long long N;        // local points L*n2*n3
    long long NC;       // local spectral bins L*n2*nh (== n1*n2s*nh)
    long long Ng;       // global points n1*n2*n3 (FFT normalisation)
    double h1, h2, h3;  // two_pi / n_a, exactly as Grid3::spacing
    int* flags;         // device flags: [0] non-finite input, [1] departure beyond halo
    int z0, zn;         // x1 plane window of the tiled (semi-Lagrangian) kernels: local planes
                        // [z0, z0 + zn), normally [0, L); narrowed to run a slab's interior
                        // planes while its halo is in flight
};

// Signed FFT frequency / odd-derivative frequency (grid.hpp:58-64)
__host__ __device__ inline int fft_freq(int i, int n) { return (2 * i <= n) ? i : i - n; }
__host__ __device__ inline int deriv_freq(int i, int n) {
    return (n % 2 == 0 && 2 * i == n) ? 0 : fft_freq(i, n);
}
// wrap_coord (grid.hpp:66-71)
__device__ __forceinline__ double wrap_coord(double x) {
    double y = x - kTwoPi * floor(x / kTwoPi);
    if (y >= kTwoPi) y -= kTwoPi;
    return y >= 0.0 ? y : 0.0;
}

// ---------------------------------------------------------------------------
// Context
// ---------------------------------------------------------------------------
struct FftPlan;

// Exchange layer of the x1-slab decomposition (dist.cu): NCCL between processes,
// or an in-process group of virtual ranks (host threads, one GPU) for tests.
// Every rank calls the same sequence of operations.
struct Transport {
    int rank = 0, size = 1;
    virtual ~Transport() = default;
    // equal blocks: send + q*count -> rank q ; recv + q*count <- rank q (doubles)
    virtual void alltoall(vr_ctx* ctx, const double* send, double* recv, size_t count) = 0;
    // field interior at `interior` (L planes of `plane` doubles, halo H planes each
    // side): lower halo <- previous rank's top H planes, upper <- next's bottom H
    virtual void halo(vr_ctx* ctx, double* interior, size_t plane, int L, int H) = 0;
    // combine k host doubles over ranks in rank order (sum, or max when `max`)
    virtual void allreduce(vr_ctx* ctx, double* vals, int k, bool max) = 0;
    // exchanges may be issued on the context's side stream concurrently with main-stream
    // exchanges (every rank issues the same host-ordered sequence either way)
    virtual bool side_stream_ok() const { return true; }
};

}  // namespace vr

struct vr_ctx {
    int device = 0;
    int sms = 0;                     // streaming multiprocessors of `device` (persistent grids)
    cudaStream_t stream = nullptr;   // all public calls are ordered on this stream
    bool owns_stream = true;         // false for siblings running on a parent's stream
    cudaStream_t side = nullptr;     // internal: overlaps independent spectral work
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_halo = nullptr, ev_halo_fork = nullptr;  // interior / halo overlap on slabs
    vr::GridDims g{};
    vr::FftPlan* fft = nullptr;
    vr::Transport* dist = nullptr;  // null on one GPU
    bool owns_dist = false;         // NCCL contexts own their transport
    long long hstride = 0;          // doubles per halo-padded field ((L + 2 halo) n2 n3)
    // lazily allocated scratch: spectra (NC complex) and real fields (N doubles)
    std::vector<double*> spec_scratch;
    std::vector<double*> field_scratch;
    // deterministic reductions
    double* red_partials = nullptr;  // device, kRedBlocks * 4 doubles
    double* red_out = nullptr;       // device, 8 doubles
    double* red_host = nullptr;      // pinned host, 8 doubles
    int* flag_dev = nullptr;         // device int flags (non-finite detection)
    int* flag_host = nullptr;        // pinned
    // deferred flag check: the operation that raised flags last (e.g. "hessian_matvec"),
    // read back by the next host synchronisation (a reduction) instead of its own sync
    const char* flags_pending = nullptr;
    long long launches = 0;
    // device-memory accounting (FieldAllocStats analogue, field.hpp:16-33): bytes live in
    // allocations made by the library for this context, and their peak since the last reset
    long long mem_live = 0, mem_peak = 0;
    std::unordered_map<const void*, long long> mem_sizes;
    // freed library buffers kept for reuse by size (and the stream they were freed on, so a
    // reuse is ordered after every kernel that used the buffer): the solver's per-iterate
    // states and trial velocities then cost no cudaMallocAsync in steady state, where the
    // stream-ordered pool's growth stalls the host for 20-800 ms (VR_TIMING)
    std::multimap<long long, std::pair<double*, cudaStream_t>> free_cache;
    // optional per-launch CUDA-event timing (bench / roofline evidence)
    bool profiling = false;
    // side-stream overlap of independent spectral work (VR_OVERLAP=1 / 0 forces it).
    // Off by default on one GPU: the FFT kernels' shared memory shrinks the L1 that the
    // concurrent gather kernels live on (measured 7.7 vs 6.9 ms per matvec). On by default
    // on x1 slabs, where the beta_v A vt transposes (all-to-all over NVLink) hide under
    // the semi-Lagrangian sweeps (SURVEY 8(e) "Overlap").
    bool overlap = false;
    // GN matvec: accumulate b inside the adjoint steps (HBM slack of the
    // L1-bound gathers) instead of a separate pass over all lam_j (VR_FUSE_ACC)
    // (measured slower at 256^3: 0.90 vs 0.63 + 0.11 ms per step, the extra
    // streams compete with the gather for the LSU; off by default)
    bool fuse_acc = false;
    struct ProfRec {
        const char* cat;
        cudaEvent_t start, stop;
        bool sibling;  // launched by a sibling context (reported as coarse_<cat>)
    };
    vr_ctx* parent = nullptr;  // sibling contexts: launches are profiled by the parent
    std::vector<vr_ctx*> siblings;  // cached siblings (other grids on this stream), owned
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
};

namespace vr {

constexpr int kRedBlocks = 592;  // 4 x 148 SMs; fixed => deterministic partial order
constexpr int kRedThreads = 256;

// create a context for grid (n1, n2, n3) on `device`; with a transport of size
// P > 1 it owns that rank's x1 slab with `halo` planes (capi.cu)
vr_ctx* ctx_new(int n1, int n2, int n3, int device, Transport* t, int halo);
// a one-GPU context of another grid on parent's device that runs on parent's stream
vr_ctx* ctx_new_sibling(vr_ctx* parent, int n1, int n2, int n3);
// the parent's cached sibling of that grid (created on first use, destroyed with the
// parent): repeated solves do not pay for context / plan / scratch setup again
vr_ctx* ctx_sibling(vr_ctx* parent, int n1, int n2, int n3);
void slab_geometry(int n1, int n2, int n3, int P, int rank, int halo, GridDims& g);
int halo_required(double vmax_x1, int nt, int n1);
void set_last_error(int cls, const std::string& msg);  // the C ABI's vr_last_error slot
double* spec_buf(vr_ctx* ctx, int i);   // NC complex (2*NC doubles)
double* field_buf(vr_ctx* ctx, int i);  // N doubles
inline void count_launch(vr_ctx* ctx, int n = 1) { ctx->launches += n; }
inline void mem_track_alloc(vr_ctx* ctx, const void* p, long long bytes) {
    if (!p) return;
    ctx->mem_sizes[p] = bytes;
    ctx->mem_live += bytes;
    if (ctx->mem_live > ctx->mem_peak) ctx->mem_peak = ctx->mem_live;
}
inline void mem_track_free(vr_ctx* ctx, const void* p) {
    auto it = ctx->mem_sizes.find(p);
    if (it == ctx->mem_sizes.end()) return;
    ctx->mem_live -= it->second;
    ctx->mem_sizes.erase(it);
}
inline void check_launch() { VR_CUDA(cudaGetLastError()); }
cudaEvent_t prof_event(vr_ctx* ctx);
// the context that owns the profile (a sibling shares its parent's stream)
inline vr_ctx* prof_owner(vr_ctx* ctx) { return ctx->parent ? ctx->parent : ctx; }
inline cudaEvent_t prof_begin(vr_ctx* ctx) {
    vr_ctx* p = prof_owner(ctx);
    if (!p->profiling) return nullptr;
    cudaEvent_t e = prof_event(p);
    VR_CUDA(cudaEventRecord(e, ctx->stream));
    return e;
}
inline void prof_end(vr_ctx* ctx, const char* cat, cudaEvent_t start) {
    ctx->launches += 1;
    if (!start) return;
    vr_ctx* p = prof_owner(ctx);
    cudaEvent_t e = prof_event(p);
    VR_CUDA(cudaEventRecord(e, ctx->stream));
    p->prof.push_back({cat, start, e, p != ctx});
}
// Launch a kernel on ctx's stream, check it, count it, and (when profiling)
// bracket it with CUDA events under category CAT.
#define VR_LAUNCH(ctx, cat, ...)                                   \
    do {                                                           \
        cudaEvent_t vr_ev_ = ::vr::prof_begin(ctx);                \
        __VA_ARGS__;                                               \
        ::vr::check_launch();                                      \
        ::vr::prof_end(ctx, cat, vr_ev_);                          \
    } while (0)

inline unsigned grid_1d(long long n, int threads) {
    return static_cast<unsigned>((n + threads - 1) / threads);
}

// ---- BLAS-1 / reductions (blas1.cu) ----
void scale(vr_ctx* ctx, double* x, long long n, double a);
void add_scaled(vr_ctx* ctx, double* y, double a, const double* x, long long n);
void lin_comb(vr_ctx* ctx, double* out, double a, const double* x, double b, const double* y,
              long long n);
// sums over `ncomp` consecutive blocks of length n; results[c] per component (host)
void dot_components(vr_ctx* ctx, const double* a, const double* b, long long n, int ncomp,
                    double* results);
void sum_components(vr_ctx* ctx, const double* a, long long n, int ncomp, double* results);
double max_abs(vr_ctx* ctx, const double* a, long long n);
double max_magnitude(vr_ctx* ctx, const double* v3, long long n);
bool all_finite(vr_ctx* ctx, const double* a, long long n);
double sum_sq_diff(vr_ctx* ctx, const double* a, const double* b, long long n);
double min_value(vr_ctx* ctx, const double* a, long long n);
double max_value(vr_ctx* ctx, const double* a, long long n);
void affine(vr_ctx* ctx, const double* x, double* out, long long n, double lo, double s);
// deferred device-flag checks (objective.cu): `defer_flags` marks the flags raised by an
// enqueued operation; the next reduction copies them back with its result (no extra
// synchronisation) and `flags_after_sync` raises them; `drain_flags` checks now
void defer_flags(vr_ctx* ctx, const char* what);
void drain_flags(vr_ctx* ctx);
void flags_enqueue_copy(vr_ctx* ctx);
void flags_after_sync(vr_ctx* ctx);
// device-side partial reduction helper: finalize `nblocks` partial sums (ncomp
// interleaved per block) into red_out[0..ncomp) and copy to host
void finalize_sums(vr_ctx* ctx, int nblocks, int ncomp, double* host_out);
// fused PCG kernels on 3-component fields: x += kappa s; r -= kappa Hs, returning
// per-component r.r and sum(r); and s = z + mu s with u = (r - mean) + mu u (u may be null)
void pcg_update(vr_ctx* ctx, double* x, double* r, const double* s, const double* Hs, double kappa,
                double* rr, double* rsum);
void pcg_direction(vr_ctx* ctx, double* s, double* u, const double* z, const double* r, double mu,
                   const double mean[3]);

// ---- FFT / spectral (fft.cu) ----
enum class Mult : int {
    none = 0,
    deriv0,
    deriv1,
    deriv2,
    laplacian,
    helmholtz1,
    reg,
    gaussian,
};
struct MultParams {
    Mult kind = Mult::none;
    int reg_kind = VR_REG_H2;
    int reg_mode = VR_REGOP_APPLY;
    double gamma = 1.0;
    int helm_sq = 1;
    double beta = 1.0;
    double sig2h2[3] = {0, 0, 0};  // sigma_d^2 * h_d^2 for the gaussian
};
void fft_plan_create(vr_ctx* ctx);
void fft_plan_destroy(vr_ctx* ctx);
// pass primitives (fft.cu): x3 rows on the local slab, x2 on the local slab,
// x1 on the x1-pass layout [n1][n2s][nh] (mult: fused forward-multiply-inverse)
void pass_rows_forward(vr_ctx* ctx, const double* in, double* spec);
void pass_rows_inverse(vr_ctx* ctx, const double* spec, double* out, double scale,
                       const double* add);
void pass_x2(vr_ctx* ctx, double* spec, int dir);
// x1 slabs: the x2 passes with the all-to-all pack / unpack fused into their stores / loads
void pass_x2_to_blocks(vr_ctx* ctx, const double* slab, double* send);
void pass_x2_from_blocks(vr_ctx* ctx, const double* recv, double* slab);
// fp32 lane: r2c rows reading fp32; c2r rows writing out = float(add + scale x) (add: fp32 or null)
void pass_rows_forward_f32(vr_ctx* ctx, const float* in, double* spec);
void pass_rows_inverse_f32(vr_ctx* ctx, const double* spec, float* out, double scale,
                           const float* add);
void pass_x1(vr_ctx* ctx, const double* src, double* dst, int dir, const MultParams* mult);
void pass_spec_div(vr_ctx* ctx, const double* s0, const double* s1, const double* s2, double* acc);
// <A v, v>_h at beta = 1 by Parseval (one GPU)
double reg_energy(vr_ctx* ctx, const double* v3, const vr_regnorm& norm);
// one-GPU spectral derivative along one axis (1D transforms only); spec: NC-complex scratch
void deriv_axis(vr_ctx* ctx, int axis, const double* f, double* out, double* spec);
void pass_spec_project(vr_ctx* ctx, double* s0, double* s1, double* s2, int kind, double beta_v,
                       double beta_w);
void fft_r2c(vr_ctx* ctx, const double* in, double* spec);
// c2r of spec (destroyed) -> out = add + scale*x (add may be null)
void fft_c2r(vr_ctx* ctx, double* spec, double* out, double scale, const double* add);
// out = c2r(mult * r2c(in)) / N (+ add), fused x1 pass; in may equal out
void spectral_scalar_op(vr_ctx* ctx, const double* in, double* out, const MultParams& m,
                        const double* add = nullptr);
void op_gradient(vr_ctx* ctx, const double* f, double* out3);
void op_divergence(vr_ctx* ctx, const double* v3, double* out);
void op_projection(vr_ctx* ctx, const double* in3, double* out3, int kind, double beta_v,
                   double beta_w);
void op_reg(vr_ctx* ctx, const double* in3, double* out3, const vr_regnorm& norm, int mode,
            double beta, const double* add3 = nullptr);
// split form of op_reg for overlap: begin leaves the three x2-inverse-transformed
// spectra in spec_buf(ctx, 4..6); finish runs the c2r passes with out = add + x/N
void op_reg_begin(vr_ctx* ctx, const double* in3, const vr_regnorm& norm, int mode, double beta);
void op_reg_finish(vr_ctx* ctx, double* out3, const double* add3);
void op_reg_finish_f32(vr_ctx* ctx, float* out3, const float* add3);  // out = float(add + x/N)
void op_reg_begin_f32(vr_ctx* ctx, const float* in3, const vr_regnorm& norm, int mode, double beta);
// run `fn` (which launches on ctx->stream) on the side stream, forked from the
// current point of ctx->stream; join_side() makes ctx->stream wait for it
// (on x1 slabs the side-stream exchanges use their own communicator, and every rank
// issues them in the same host order; while profiling the work stays on the main
// stream, so per-kernel event intervals do not include time shared with a concurrent
// kernel)
template <class Fn>
void on_side_stream(vr_ctx* ctx, Fn&& fn) {
    if ((ctx->dist && !ctx->dist->side_stream_ok()) || ctx->profiling || !ctx->overlap) {
        fn();
        return;
    }
    VR_CUDA(cudaEventRecord(ctx->ev_fork, ctx->stream));
    VR_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    cudaStream_t main = ctx->stream;
    ctx->stream = ctx->side;
    try {
        fn();
    } catch (...) {
        ctx->stream = main;
        throw;
    }
    ctx->stream = main;
    VR_CUDA(cudaEventRecord(ctx->ev_join, ctx->side));
}
inline void join_side(vr_ctx* ctx) {
    if (!(ctx->dist && !ctx->dist->side_stream_ok()) && !ctx->profiling && ctx->overlap)
        VR_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
}
double reg_symbol(const vr_regnorm& n, double k2);

// ---- semi-Lagrangian (sl.cu) ----
void sl_tricubic(vr_ctx* ctx, const double* f, int nfields, const double* pts3, double* out);
// v3: component c at v3 + c*vstride (N, or the halo-padded stride on x1 slabs)
void sl_trace(vr_ctx* ctx, const double* v3, long long vstride, int nt, int direction,
              double* dep3);
void sl_factor(vr_ctx* ctx, const double* div_v, const double* dep3, double half_dt,
               double* factor);
void sl_advect(vr_ctx* ctx, const double* f, const double* dep3, double* out);
void sl_continuity(vr_ctx* ctx, const double* f, const double* dep3, const double* factor,
                   double* out);
// incremental state fused step: g = I[src](X); m = g - hdt*q(gm, vt);
// mode 0: dst = m - hdt*q (next tmp); mode 1: dst = -m (terminal);
// mode 2: mode 1 and b3 = 0 + (wb * dst) * gm (first observer of the adjoint sweep)
void sl_incstate_first(vr_ctx* ctx, const double* gm0, const double* vt3, double hdt,
                       double* tmp0);
void sl_incstate_step(vr_ctx* ctx, const double* src, const double* dep3, const double* gm,
                      const double* vt3, double hdt, double* dst, int mode, double* b3 = nullptr,
                      double wb = 0.0, double* mt_out = nullptr);
// adjoint step with optional gradient accumulation bout_a = (b_a + (w*lam) * gm_a) [+ add_a]
// (bout defaults to b3)
void sl_adjoint_step(vr_ctx* ctx, const double* src, const double* dep3, const double* factor,
                     double* dst, const double* gm, double w, double* b3,
                     const double* add3 = nullptr, double* bout3 = nullptr);
void sl_grad_terminal(vr_ctx* ctx, const double* mR, const double* mfinal, const double* gm,
                      double w, double* lam, double* b3);
// b_a = sum_{j=nt..0} (w_j lam_j) d_a m_j [+ (w_j lam2_j) d_a mt_j]  (+ add_a when add3 is given)
void sl_accumulate(vr_ctx* ctx, const double* lam_hist, const double* gm_hist, int nt, double dt,
                   double* b3, const double* add3 = nullptr, const double* lam2_hist = nullptr,
                   const double* gm2_hist = nullptr);
// full-Newton inc-adjoint step: dst = I[src](X) * factor + hdt * (rcur + I[rnext](X))
void sl_adjoint_fn_step(vr_ctx* ctx, const double* src, const double* rnext, const double* dep3,
                        const double* factor, const double* rcur, double hdt, double* dst);
// deformation_map step: out_c = I[u_c](X) - half_dt (vdep_c + v_c) (out must not alias u)
void sl_defmap_step(vr_ctx* ctx, const double* u3, const double* dep3, const double* vdep3,
                    const double* v3, double half_dt, double* out3);
// fp32 lane (one GPU): fields / points in fp32, stencil arithmetic in fp64
void sl_tricubic_f32(vr_ctx* ctx, const float* f, int nfields, const float* pts3, float* out);
void sl_trace_f32(vr_ctx* ctx, const float* v3, int nt, int direction, float* dep3);
bool all_finite_f32(vr_ctx* ctx, const float* a, long long n);
void sl_incstate_first_f32(vr_ctx* ctx, const float* gm0, const float* vt3, double hdt, float* tmp0);
void sl_incstate_step_f32(vr_ctx* ctx, const float* src, const float* dep3, const float* gm,
                          const float* vt3, double hdt, float* dst, bool last);
void sl_continuity_f32(vr_ctx* ctx, const float* src, const float* dep3, const float* factor, float* dst);
void sl_accumulate_f32(vr_ctx* ctx, const float* lam_hist, const float* gm_hist, int nt, double dt,
                       float* b3);
void convert_f2d(vr_ctx* ctx, const float* a, double* b, long long n);
void convert_d2f(vr_ctx* ctx, const double* a, float* b, long long n);
// out_c = lam * vt_c
void sl_scale_vec(vr_ctx* ctx, const double* lam, const double* vt3, double* out3);
void sl_gradient_dot(vr_ctx* ctx, const double* gm3, const double* w3, double* out);
void synth_fill(vr_ctx* ctx, double amplitude, double* m_T, double* v3);

}  // namespace vr
