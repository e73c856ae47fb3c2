// objective.cuh -- device-resident Objective / EvalState (objective.hpp:11-122)
// and the host-side Gauss-Newton-Krylov driver (solver.hpp:78-164).
#pragma once

#include <functional>

#include "vr_common.cuh"

struct vr_objective;

// EvalState<T> (objective.hpp:37-54), device resident. Beyond the reference's
// fields it caches grad m_j (3 (n_t+1) fields), built once per iterate in the
// gradient: it makes every Hessian matvec FFT-free except the beta_v A term.
struct vr_state {
    vr_objective* obj = nullptr;
    int nt = 0;
    double* v = nullptr;       // 3N
    double* xb = nullptr;      // 3N backward departure points
    double* mhist = nullptr;   // (nt+1)N
    double* xf = nullptr;      // 3N forward departure points (adjoint ctx)
    double* factor = nullptr;  // N continuity factor (adjoint ctx)
    double* gradm = nullptr;   // 3(nt+1)N, [j*3 + a]
    double* grad = nullptr;    // 3N
    double* vpad = nullptr;    // x1 slabs: halo-padded copy of v (gather source of the trace)
    double* lamhist = nullptr; // full Newton: adjoint history lambda_j, (nt+1) halo-padded fields
    double objective = 0.0, mismatch = 0.0, mismatch_rel = 0.0;
    bool has_gradient = false, has_adjoint_ctx = false;
    ~vr_state();
};

struct vr_objective {
    vr_ctx* ctx = nullptr;
    const double* mR = nullptr;  // non-owning (objective.hpp:97-98)
    const double* mT = nullptr;
    vr_model model{};
    vr_counters counters{};
    double initial_mismatch = 0.0;
    // workspace reused by every call
    double* ws_lam = nullptr;  // (nt+1) halo-padded fields
    double* ws_tmp = nullptr;  // 2 halo-padded fields
    double* ws_div = nullptr;  // 1 halo-padded field (div v, gathered by the factor)
    double* ws_b = nullptr;    // 3N
    // device staging of the synchronous host-buffer matvec (vr_hessian_matvec_host),
    // allocated on first use and kept: no per-call allocation on the e2e path
    double* host_vt = nullptr;   // 3N
    double* host_out = nullptr;  // 3N
    // pipelined host-buffer matvecs (vr_hessian_matvec_host_async): two device slots;
    // H2D and D2H on their own streams so step k+1's upload and step k's download
    // overlap step k / k+1 compute on the context's stream
    struct Pipe {
        double* vt[2] = {nullptr, nullptr};
        double* out[2] = {nullptr, nullptr};
        cudaStream_t h2d = nullptr, d2h = nullptr;
        cudaEvent_t up[2] = {}, done[2] = {}, down[2] = {};
        long long issued = 0;  // calls since the last wait
    } pipe;
    ~vr_objective();
};

namespace vr {

double* dev_alloc(vr_ctx* ctx, long long ndoubles);
void dev_free(vr_ctx* ctx, double* p);
void release_cache(vr_ctx* ctx);  // return the context's cached device buffers to the pool
// halo-padded field helpers (objective.cu)
long long hoff(const vr_ctx* ctx);
double* pslice(const vr_ctx* ctx, double* base, int j);
void exchange(vr_ctx* ctx, double* interior);
// read the device flags now (non-finite input, departure beyond the x1 halo) and raise
void check_flags(vr_ctx* ctx, const char* what);

void validate_model(const vr_model& m);
void validate_params(const vr_solver_params& p);

vr_objective* objective_create(vr_ctx* ctx, const double* mR, const double* mT,
                               const vr_model& model);
vr_state* objective_evaluate(vr_objective* o, const double* v3);
void objective_gradient(vr_objective* o, vr_state* s);
// H vt (add_reg) or H_data vt; reg_given (may be null, add_reg false): a field
// equal to beta_v A vt computed elsewhere, added instead of the spectral term
void objective_matvec(vr_objective* o, const vr_state* s, const double* vt3, double* out3,
                      bool add_reg, const double* reg_given = nullptr, bool check = true);
// pipelined H vt with host buffers (see vr_objective::Pipe); errors of the batch
// (non-finite directions) surface in objective_pipe_wait
void objective_matvec_host_async(vr_objective* o, const vr_state* s, const double* vt3_host,
                                 double* out3_host);
void objective_pipe_wait(vr_objective* o);
// PCG on the GN Hessian with the spectral preconditioner (solver.cpp:51-100),
// carrying u = beta_v A s through the recurrence (see objective.cu)
vr_pcg_stats pcg_solve_gn(vr_objective* o, const vr_state* s, const double* rhs, double rel_tol,
                          int max_iter, double* x);
void objective_apply_reg(vr_objective* o, const double* u3, int mode, double* out3);
void objective_apply_K(vr_objective* o, const double* u3, double* out3);

// weighted / unweighted reductions on vector fields (component order as the reference)
double dot_l2_vec(vr_ctx* ctx, const double* a, const double* b);
double norm_l2_vec(vr_ctx* ctx, const double* a);
double inner_product_vec(vr_ctx* ctx, const double* a, const double* b);
double inner_product_scalar(vr_ctx* ctx, const double* a, const double* b);

using DevOp = std::function<void(const double*, double*)>;
vr_pcg_stats pcg_solve(vr_ctx* ctx, const DevOp& apply, const double* rhs, double rel_tol,
                       int max_iter, const DevOp& precond, double* x);

struct GnResult {
    vr_solve_report report{};
    std::vector<vr_iteration_record> records;
};
GnResult gauss_newton_solve(vr_ctx* ctx, const double* mR, const double* mT, const double* v0,
                            const vr_model& model, const vr_solver_params& params, int precond,
                            double* v_out, const vr_twolevel_options* tl_opts = nullptr);
// evaluation context from given v and m history (coarse state of the two-level preconditioner)
// (lamhist: optional adjoint history, (nt+1) fields, for the full-Newton matvec)
vr_state* state_from_history(vr_objective* o, const double* v3, const double* mhist, int nt,
                             const double* lamhist = nullptr);

// ---- fp32 lane objective (objective_f32.cu) ----
struct ObjF32;
struct StateF32;
ObjF32* objf32_create(vr_ctx* ctx, const float* mR, const float* mT, const vr_model& model);
void objf32_destroy(ObjF32* o);
StateF32* objf32_evaluate(ObjF32* o, const float* v3);
void statef32_destroy(StateF32* s);
void statef32_scalars(const StateF32* s, double* J, double* mis, double* rel);
const float* statef32_gradient(const StateF32* s);
void objf32_gradient(ObjF32* o, StateF32* s);
void objf32_matvec(ObjF32* o, const StateF32* s, const float* vt3, float* out3);
vr_counters objf32_counters(const ObjF32* o);
vr_ctx* objf32_ctx(ObjF32* o);
void objf32_copy_gradient(ObjF32* o, const StateF32* s, float* g3);  // synchronises
GnResult gauss_newton_solve_f32(vr_ctx* ctx, const float* mR, const float* mT, const float* v0,
                                const vr_model& model, const vr_solver_params& params, int precond,
                                float* v_out, const vr_twolevel_options* tl_opts = nullptr);
std::vector<GnResult> parameter_continuation_f32(vr_ctx* ctx, const float* mR, const float* mT,
                                                 const float* v0, const vr_model& model,
                                                 const vr_solver_params& params, int precond,
                                                 float* v_out);

// ---- postprocess / continuation (postprocess.cu) ----
void det_deformation_gradient(vr_ctx* ctx, const double* v3, int nt, double* det);
void deformation_map(vr_ctx* ctx, const double* v3, int nt, bool absolute, double* out3);
vr_det_summary det_stats(vr_ctx* ctx, const double* det, const double* fg, double threshold);
void transport_labels(vr_ctx* ctx, const double* labels, const double* v3, int nt, double* out);
// returns the number of distinct nonzero codes; fills the first max_labels
int overlap_scores(vr_ctx* ctx, const double* ref, const double* test, const double* mask,
                   int max_labels, int* codes_out, vr_overlap* per_label, vr_overlap* uni);
std::vector<GnResult> grid_continuation(vr_ctx* ctx, const double* mR, const double* mT,
                                        const double* v0, const vr_model& model,
                                        const vr_solver_params& params, int precond,
                                        int n_levels, double* v_out);
std::vector<GnResult> scale_continuation(vr_ctx* ctx, const double* mR, const double* mT,
                                         const double* v0, const vr_model& model,
                                         const vr_solver_params& params, int precond,
                                         const double* sigmas, int n, double* v_out);
struct BetaSearch {
    bool found = false;
    double beta = 0.0;
    std::vector<vr_beta_trial> trials;
};
BetaSearch beta_search(vr_ctx* ctx, const double* mR, const double* mT, const double* v0,
                       const vr_model& model, const vr_solver_params& params, int precond,
                       const vr_beta_search_params& bp, double* v_out);

}  // namespace vr
