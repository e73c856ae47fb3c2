// dist.cu -- x1-slab decomposition across ranks (DESIGN.md
// section 7). The reference is single-process (no MPI/NCCL); the paper's CLAIRE
// used MPI pencils, AccFFT transposes and ghost layers.
//
// Two exchange layers implement vr::Transport:
//  * NcclTransport: one process per GPU; grouped ncclSend/ncclRecv for the FFT
//    all-to-all and the halo planes, ncclAllGather of reduction partials summed
//    in rank order (deterministic). libnccl is dlopen'ed on first use so the
//    library has no link-time NCCL dependency (torch may bring its own copy).
//  * LocalGroup: P virtual ranks as host threads of one process on one GPU.
//    Exchanges are host-barrier-separated device copies, so no kernel ever
//    waits on another rank's kernel; used to validate the slab path on a
//    single B200 (vr_dist_selftest*).
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "objective.cuh"

namespace vr {
namespace {

// ---------------------------------------------------------------------------
// NCCL (dlopen)
// ---------------------------------------------------------------------------
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names)
            if ((api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!api.h) return;
        api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
        api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(api.h, "ncclCommInitRank"));
        api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(api.h, "ncclCommDestroy"));
        api.commSplit = reinterpret_cast<decltype(api.commSplit)>(dlsym(api.h, "ncclCommSplit"));
        api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(api.h, "ncclGroupStart"));
        api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(api.h, "ncclGroupEnd"));
        api.send = reinterpret_cast<decltype(api.send)>(dlsym(api.h, "ncclSend"));
        api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(api.h, "ncclRecv"));
        api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(api.h, "ncclAllGather"));
        api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(api.h, "ncclGetErrorString"));
    });
    if (!api.h || !api.commInitRank || !api.send || !api.allGather)
        throw_resource("NCCL: libnccl.so.2 not loadable");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw_resource(std::string("NCCL ") + what + ": " +
                       (nccl().errorString ? nccl().errorString(r) : "error"));
}

struct NcclTransport final : Transport {
    ncclComm_t comm = nullptr;
    // a second communicator for the exchanges issued on the context's side stream (the
    // beta_v A vt transposes running under the sweeps): two concurrent NCCL operations
    // must not share a communicator. Null when ncclCommSplit is unavailable (then the
    // side-stream work stays on the main stream)
    ncclComm_t comm_side = nullptr;
    double* buf = nullptr;  // device: 8 doubles in, size*8 gathered

    NcclTransport(int r, int p, const unsigned char uid[NCCL_UNIQUE_ID_BYTES]) {
        rank = r;
        size = p;
        ncclUniqueId id;
        std::memcpy(id.internal, uid, NCCL_UNIQUE_ID_BYTES);
        nccl_check(nccl().commInitRank(&comm, p, id, r), "commInitRank");
        if (nccl().commSplit) nccl_check(nccl().commSplit(comm, 0, r, &comm_side, nullptr), "commSplit");
        VR_CUDA(cudaMalloc(&buf, sizeof(double) * 8 * (p + 1)));
    }
    ~NcclTransport() override {
        if (buf) cudaFree(buf);
        if (comm_side) nccl().commDestroy(comm_side);
        if (comm) nccl().commDestroy(comm);
    }
    bool side_stream_ok() const override { return comm_side != nullptr; }
    ncclComm_t comm_of(const vr_ctx* ctx) const {
        return (comm_side && ctx->stream == ctx->side) ? comm_side : comm;
    }
    // exchange time as a profile category (library kernels: not counted as our launches);
    // the exchanges run on the context stream, so their time is also the exposed time
    static void comm_end(vr_ctx* ctx, const char* cat, cudaEvent_t start) {
        if (!start) return;
        vr_ctx* p = prof_owner(ctx);
        cudaEvent_t e = prof_event(p);
        VR_CUDA(cudaEventRecord(e, ctx->stream));
        p->prof.push_back({cat, start, e, false});
    }
    void alltoall(vr_ctx* ctx, const double* send, double* recv, size_t count) override {
        auto& api = nccl();
        ncclComm_t cm = comm_of(ctx);
        cudaEvent_t ev = prof_begin(ctx);
        nccl_check(api.groupStart(), "groupStart");
        for (int q = 0; q < size; ++q) {
            nccl_check(api.send(send + q * count, count, ncclDouble, q, cm, ctx->stream), "send");
            nccl_check(api.recv(recv + q * count, count, ncclDouble, q, cm, ctx->stream), "recv");
        }
        nccl_check(api.groupEnd(), "groupEnd");
        comm_end(ctx, "comm_alltoall", ev);
    }
    void halo(vr_ctx* ctx, double* interior, size_t plane, int L, int H) override {
        auto& api = nccl();
        ncclComm_t cm = comm_of(ctx);
        const int prev = (rank + size - 1) % size, next = (rank + 1) % size;
        const size_t n = static_cast<size_t>(H) * plane;
        cudaEvent_t ev = prof_begin(ctx);
        nccl_check(api.groupStart(), "groupStart");
        nccl_check(api.send(interior, n, ncclDouble, prev, cm, ctx->stream), "send");
        nccl_check(api.recv(interior + L * plane, n, ncclDouble, next, cm, ctx->stream), "recv");
        nccl_check(api.send(interior + (L - H) * plane, n, ncclDouble, next, cm, ctx->stream), "send");
        nccl_check(api.recv(interior - n, n, ncclDouble, prev, cm, ctx->stream), "recv");
        nccl_check(api.groupEnd(), "groupEnd");
        comm_end(ctx, "comm_halo", ev);
    }
    void allreduce(vr_ctx* ctx, double* vals, int k, bool max) override {
        double* b = buf;  // 8 in, 8 * size gathered; larger tables (label codes) get a temporary
        const size_t in = k <= 8 ? 8 : static_cast<size_t>(k);
        if (k > 8) VR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&b), sizeof(double) * in * (size + 1), ctx->stream));
        VR_CUDA(cudaMemcpyAsync(b, vals, sizeof(double) * k, cudaMemcpyHostToDevice, ctx->stream));
        nccl_check(nccl().allGather(b, b + in, k, ncclDouble, comm, ctx->stream), "allGather");
        std::vector<double> all(static_cast<size_t>(k) * size);
        VR_CUDA(cudaMemcpyAsync(all.data(), b + in, sizeof(double) * k * size,
                                cudaMemcpyDeviceToHost, ctx->stream));
        if (k > 8) VR_CUDA(cudaFreeAsync(b, ctx->stream));
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int i = 0; i < k; ++i) {
            double acc = all[i];
            for (int q = 1; q < size; ++q)
                acc = max ? std::max(acc, all[q * k + i]) : acc + all[q * k + i];
            vals[i] = acc;
        }
    }
};

// ---------------------------------------------------------------------------
// LocalGroup: virtual ranks = host threads sharing one device
// ---------------------------------------------------------------------------
struct LocalShared {
    int P;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    bool aborted = false;
    std::vector<const double*> ptr;
    std::vector<std::vector<double>> host;
    explicit LocalShared(int p) : P(p), ptr(p, nullptr), host(p) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        if (aborted) throw_logic("local group aborted by another rank");
        const long gen = generation;
        if (++arrived == P) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen || aborted; });
            if (aborted) throw_logic("local group aborted by another rank");
        }
    }
    void abort() {
        std::lock_guard<std::mutex> lk(m);
        aborted = true;
        cv.notify_all();
    }
};

struct LocalTransport final : Transport {
    std::shared_ptr<LocalShared> sh;
    LocalTransport(int r, std::shared_ptr<LocalShared> s) : sh(std::move(s)) {
        rank = r;
        size = sh->P;
    }
    void publish(vr_ctx* ctx, const double* p) {
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        sh->ptr[rank] = p;
        sh->barrier();
    }
    void finish(vr_ctx* ctx) {
        VR_CUDA(cudaStreamSynchronize(ctx->stream));
        sh->barrier();
    }
    void alltoall(vr_ctx* ctx, const double* send, double* recv, size_t count) override {
        publish(ctx, send);
        for (int q = 0; q < size; ++q)
            VR_CUDA(cudaMemcpyAsync(recv + q * count, sh->ptr[q] + rank * count,
                                    sizeof(double) * count, cudaMemcpyDeviceToDevice, ctx->stream));
        finish(ctx);
    }
    void halo(vr_ctx* ctx, double* interior, size_t plane, int L, int H) override {
        publish(ctx, interior);
        const int prev = (rank + size - 1) % size, next = (rank + 1) % size;
        const size_t n = static_cast<size_t>(H) * plane;
        VR_CUDA(cudaMemcpyAsync(interior - n, sh->ptr[prev] + (L - H) * plane, sizeof(double) * n,
                                cudaMemcpyDeviceToDevice, ctx->stream));
        VR_CUDA(cudaMemcpyAsync(interior + L * plane, sh->ptr[next], sizeof(double) * n,
                                cudaMemcpyDeviceToDevice, ctx->stream));
        finish(ctx);
    }
    void allreduce(vr_ctx*, double* vals, int k, bool max) override {
        sh->host[rank].assign(vals, vals + k);
        sh->barrier();
        for (int i = 0; i < k; ++i) {
            double acc = sh->host[0][i];
            for (int q = 1; q < size; ++q) acc = max ? std::max(acc, sh->host[q][i]) : acc + sh->host[q][i];
            vals[i] = acc;
        }
        sh->barrier();
    }
};

// Run fn(rank, ctx) on P virtual ranks (threads) on one device; the first
// failure aborts the group and is rethrown.
template <class Fn>
void run_local_group(int P, int n1, int n2, int n3, int device, int halo, Fn&& fn) {
    auto sh = std::make_shared<LocalShared>(P);
    std::vector<std::unique_ptr<LocalTransport>> tr;
    for (int r = 0; r < P; ++r) tr.emplace_back(new LocalTransport(r, sh));
    std::mutex em;
    std::unique_ptr<Error> first;
    std::vector<std::thread> th;
    for (int r = 0; r < P; ++r)
        th.emplace_back([&, r] {
            vr_ctx* ctx = nullptr;
            try {
                VR_CUDA(cudaSetDevice(device));
                ctx = ctx_new(n1, n2, n3, device, tr[r].get(), halo);
                fn(r, ctx);
            } catch (const Error& e) {
                std::lock_guard<std::mutex> lk(em);
                if (!first && std::string(e.what()).find("aborted by another rank") == std::string::npos)
                    first.reset(new Error(e));
                sh->abort();
            } catch (const std::exception& e) {
                std::lock_guard<std::mutex> lk(em);
                if (!first) first.reset(new Error(VR_ERR_LOGIC, VR_EXC_LOGIC, e.what()));
                sh->abort();
            }
            if (ctx) {
                ctx->dist = nullptr;
                vr_ctx_destroy(ctx);
            }
        });
    for (auto& t : th) t.join();
    if (first) throw *first;
}

vr_model model_or_default(const vr_model* m) {
    vr_model out;
    if (m) {
        out = *m;
    } else {
        vr_model_default(&out);
    }
    return out;
}

}  // namespace
}  // namespace vr

namespace {
template <typename Fn>
int dguard(Fn&& fn) {
    try {
        fn();
        return VR_OK;
    } catch (const vr::Error& e) {
        // surface through the common last-error slot of capi.cu
        vr::set_last_error(e.cls, e.what());
        return e.status;
    } catch (const std::exception& e) {
        vr::set_last_error(VR_EXC_LOGIC, e.what());
        return VR_ERR_LOGIC;
    }
}
}  // namespace

extern "C" {

int vr_nccl_unique_id(unsigned char out[128]) {
    return dguard([&] {
        ncclUniqueId id;
        vr::nccl_check(vr::nccl().getUniqueId(&id), "getUniqueId");
        static_assert(NCCL_UNIQUE_ID_BYTES == 128, "ncclUniqueId size");
        std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

int vr_ctx_create_dist(int n1, int n2, int n3, int device, int rank, int nranks,
                       const unsigned char uid[128], int halo, vr_ctx** out) {
    return dguard([&] {
        if (!out || !uid) vr::throw_argument("vr_ctx_create_dist: null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) vr::throw_argument("vr_ctx_create_dist: bad rank");
        // one rank: a plain context, unless VR_DIST_SINGLE_RANK asks for the slab code over a
        // one-rank NCCL communicator (self send/recv: a one-GPU check of the multi-GPU plumbing)
        if (nranks == 1 && !std::getenv("VR_DIST_SINGLE_RANK")) {
            *out = vr::ctx_new(n1, n2, n3, device, nullptr, 0);
            return;
        }
        VR_CUDA(cudaSetDevice(device));
        auto* t = new vr::NcclTransport(rank, nranks, uid);
        try {
            *out = vr::ctx_new(n1, n2, n3, device, t, halo);
        } catch (...) {
            delete t;
            throw;
        }
        (*out)->owns_dist = true;
    });
}

int vr_ctx_slab(const vr_ctx* ctx, int* rank, int* nranks, int* planes, int* first_plane,
                int* halo) {
    return dguard([&] {
        if (!ctx) vr::throw_argument("vr_ctx_slab: null context");
        if (rank) *rank = ctx->dist ? ctx->dist->rank : 0;
        if (nranks) *nranks = ctx->dist ? ctx->dist->size : 1;
        if (planes) *planes = ctx->g.L;
        if (first_plane) *first_plane = ctx->g.off1;
        if (halo) *halo = ctx->g.halo;
    });
}

// Self test of the slab path: P virtual ranks on one GPU run evaluate, gradient,
// Hessian matvec and apply_reg on their slabs of the global host inputs; the
// slab outputs are assembled into the global host outputs.
// scalars: J, mismatch, mismatch_rel, ||g||_2 (unweighted), <H vt, vt>
int vr_dist_selftest_objective(int P, int n1, int n2, int n3, int device, int halo,
                               const vr_model* model, const double* mR, const double* mT,
                               const double* v, const double* vt, double* grad_out,
                               double* matvec_out, double* reg_out, double* scalars) {
    return dguard([&] {
        const vr_model m = vr::model_or_default(model);
        const long long Ng = static_cast<long long>(n1) * n2 * n3;
        vr::run_local_group(P, n1, n2, n3, device, halo, [&](int, vr_ctx* ctx) {
            const long long N = ctx->g.N, off = static_cast<long long>(ctx->g.off1) * n2 * n3;
            auto up = [&](const double* host, int nf) {
                double* d = vr::dev_alloc(ctx, nf * N);
                for (int c = 0; c < nf; ++c)
                    VR_CUDA(cudaMemcpyAsync(d + c * N, host + c * Ng + off, sizeof(double) * N,
                                            cudaMemcpyHostToDevice, ctx->stream));
                return d;
            };
            auto down = [&](const double* d, int nf, double* host) {
                for (int c = 0; c < nf; ++c)
                    VR_CUDA(cudaMemcpyAsync(host + c * Ng + off, d + c * N, sizeof(double) * N,
                                            cudaMemcpyDeviceToHost, ctx->stream));
                VR_CUDA(cudaStreamSynchronize(ctx->stream));
            };
            double* dR = up(mR, 1);
            double* dT = up(mT, 1);
            double* dv = up(v, 3);
            double* dvt = up(vt, 3);
            double* out = vr::dev_alloc(ctx, 3 * N);
            vr_objective* o = vr::objective_create(ctx, dR, dT, m);
            vr_state* s = nullptr;
            try {
                s = vr::objective_evaluate(o, dv);
                vr::objective_gradient(o, s);
                const double gn = vr::norm_l2_vec(ctx, s->grad);
                if (grad_out) down(s->grad, 3, grad_out);
                vr::objective_matvec(o, s, dvt, out, true);
                const double q = vr::dot_l2_vec(ctx, out, dvt);
                if (matvec_out) down(out, 3, matvec_out);
                vr::objective_apply_reg(o, dvt, VR_REGOP_APPLY, out);
                if (reg_out) down(out, 3, reg_out);
                if (scalars && ctx->dist->rank == 0) {
                    scalars[0] = s->objective;
                    scalars[1] = s->mismatch;
                    scalars[2] = s->mismatch_rel;
                    scalars[3] = gn;
                    scalars[4] = q;
                }
            } catch (...) {
                delete s;
                delete o;
                throw;
            }
            delete s;
            delete o;
            for (double* p : {dR, dT, dv, dvt, out}) vr::dev_free(ctx, p);
            VR_CUDA(cudaStreamSynchronize(ctx->stream));
        });
    });
}

// Self test: a whole Gauss-Newton solve on P virtual ranks (same host driver).
int vr_dist_selftest_solve(int P, int n1, int n2, int n3, int device, int halo,
                           const vr_model* model, const vr_solver_params* params,
                           const double* mR, const double* mT, const double* v0, double* v_out,
                           vr_solve_report* report) {
    return vr_dist_selftest_solve_precond(P, n1, n2, n3, device, halo, model, params, VR_PRECOND_SPECTRAL,
                                          nullptr, mR, mT, v0, v_out, report);
}

int vr_dist_selftest_solve_precond(int P, int n1, int n2, int n3, int device, int halo,
                                   const vr_model* model, const vr_solver_params* params, int precond,
                                   const vr_twolevel_options* tl_opts, const double* mR,
                                   const double* mT, const double* v0, double* v_out,
                                   vr_solve_report* report) {
    return dguard([&] {
        const vr_model m = vr::model_or_default(model);
        vr_solver_params p;
        if (params)
            p = *params;
        else
            vr_solver_params_default(&p);
        const long long Ng = static_cast<long long>(n1) * n2 * n3;
        vr::run_local_group(P, n1, n2, n3, device, halo, [&](int, vr_ctx* ctx) {
            const long long N = ctx->g.N, off = static_cast<long long>(ctx->g.off1) * n2 * n3;
            double* dR = vr::dev_alloc(ctx, N);
            double* dT = vr::dev_alloc(ctx, N);
            double* dv = vr::dev_alloc(ctx, 3 * N);
            double* dout = vr::dev_alloc(ctx, 3 * N);
            VR_CUDA(cudaMemcpyAsync(dR, mR + off, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->stream));
            VR_CUDA(cudaMemcpyAsync(dT, mT + off, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->stream));
            for (int c = 0; c < 3; ++c)
                VR_CUDA(cudaMemcpyAsync(dv + c * N, v0 + c * Ng + off, sizeof(double) * N,
                                        cudaMemcpyHostToDevice, ctx->stream));
            vr::GnResult r = vr::gauss_newton_solve(ctx, dR, dT, dv, m, p, precond, dout, tl_opts);
            for (int c = 0; c < 3; ++c)
                VR_CUDA(cudaMemcpyAsync(v_out + c * Ng + off, dout + c * N, sizeof(double) * N,
                                        cudaMemcpyDeviceToHost, ctx->stream));
            VR_CUDA(cudaStreamSynchronize(ctx->stream));
            if (report && ctx->dist->rank == 0) *report = r.report;
            for (double* q : {dR, dT, dv, dout}) vr::dev_free(ctx, q);
            VR_CUDA(cudaStreamSynchronize(ctx->stream));
        });
    });
}

int vr_dist_selftest_postprocess(int P, int n1, int n2, int n3, int device, int halo, const double* v,
                                 int nt, double* det_out, double* map_out, double* stats3) {
    return dguard([&] {
        const long long Ng = static_cast<long long>(n1) * n2 * n3;
        vr::run_local_group(P, n1, n2, n3, device, halo, [&](int, vr_ctx* ctx) {
            const long long N = ctx->g.N, off = static_cast<long long>(ctx->g.off1) * n2 * n3;
            double* dv = vr::dev_alloc(ctx, 3 * N);
            double* det = vr::dev_alloc(ctx, N);
            double* map = vr::dev_alloc(ctx, 3 * N);
            for (int c = 0; c < 3; ++c)
                VR_CUDA(cudaMemcpyAsync(dv + c * N, v + c * Ng + off, sizeof(double) * N,
                                        cudaMemcpyHostToDevice, ctx->stream));
            vr::det_deformation_gradient(ctx, dv, nt, det);
            vr::deformation_map(ctx, dv, nt, true, map);
            const vr_det_summary st = vr::det_stats(ctx, det, nullptr, 0.0);
            VR_CUDA(cudaMemcpyAsync(det_out + off, det, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
            for (int c = 0; c < 3; ++c)
                VR_CUDA(cudaMemcpyAsync(map_out + c * Ng + off, map + c * N, sizeof(double) * N,
                                        cudaMemcpyDeviceToHost, ctx->stream));
            VR_CUDA(cudaStreamSynchronize(ctx->stream));
            if (stats3 && ctx->dist->rank == 0) stats3[0] = st.min, stats3[1] = st.max, stats3[2] = st.mean;
            for (double* q : {dv, det, map}) vr::dev_free(ctx, q);
            VR_CUDA(cudaStreamSynchronize(ctx->stream));
        });
    });
}

int vr_dist_selftest_labels(int P, int n1, int n2, int n3, int device, int halo, const double* labels,
                            const double* v, int nt, double* warped_out, int max_labels, int* n_labels,
                            int* codes, vr_overlap* per_label, vr_overlap* union_scores) {
    return dguard([&] {
        const long long Ng = static_cast<long long>(n1) * n2 * n3;
        vr::run_local_group(P, n1, n2, n3, device, halo, [&](int, vr_ctx* ctx) {
            const long long N = ctx->g.N, off = static_cast<long long>(ctx->g.off1) * n2 * n3;
            double* dv = vr::dev_alloc(ctx, 3 * N);
            double* dl = vr::dev_alloc(ctx, N);
            double* dw = vr::dev_alloc(ctx, N);
            VR_CUDA(cudaMemcpyAsync(dl, labels + off, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->stream));
            for (int c = 0; c < 3; ++c)
                VR_CUDA(cudaMemcpyAsync(dv + c * N, v + c * Ng + off, sizeof(double) * N,
                                        cudaMemcpyHostToDevice, ctx->stream));
            vr::transport_labels(ctx, dl, dv, nt, dw);
            VR_CUDA(cudaMemcpyAsync(warped_out + off, dw, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
            const bool r0 = ctx->dist->rank == 0;
            std::vector<int> cd(max_labels > 0 ? max_labels : 1);
            std::vector<vr_overlap> pl(max_labels > 0 ? max_labels : 1);
            vr_overlap un{};
            const int ns = vr::overlap_scores(ctx, dl, dw, nullptr, max_labels, cd.data(), pl.data(), &un);
            VR_CUDA(cudaStreamSynchronize(ctx->stream));
            if (r0) {
                if (n_labels) *n_labels = ns;
                for (int s = 0; s < ns && s < max_labels; ++s) {
                    if (codes) codes[s] = cd[s];
                    if (per_label) per_label[s] = pl[s];
                }
                if (union_scores) *union_scores = un;
            }
            for (double* q : {dv, dl, dw}) vr::dev_free(ctx, q);
            VR_CUDA(cudaStreamSynchronize(ctx->stream));
        });
    });
}

}  // extern "C"
