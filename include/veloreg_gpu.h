/*
 * veloreg_gpu.h -- C ABI of the B200-native (sm_100a) operator layer for the
 * CLAIRE / veloreg Gauss-Newton-Krylov registration hot path.
 *
 * The reference (/root/reference/proj, "veloreg") has no FFI: its operator
 * boundary is the C++ template API Objective<T> (include/veloreg/objective.hpp:56-102),
 * the free functions of transport.hpp / spectral.hpp / interp.hpp / field_ops.hpp,
 * and the solver entry points of solver.hpp:100-164. Every function below names
 * the reference interface it replaces. A C++ adapter rethrows
 * status codes as the matching veloreg::Error subclasses.
 *
 * Conventions
 *  - All arithmetic is IEEE fp64 (the reference precision for parity).
 *  - Field arguments are DEVICE pointers (double*), laid out exactly like the
 *    reference: scalar field = N = n1*n2*n3 doubles, row-major, axis 0 slowest,
 *    linear index (i1*n2+i2)*n3+i3 (grid.hpp:17-19); vector field = 3 scalar
 *    fields back to back (component c at ptr + c*N; VectorField SoA, field.hpp:101-126);
 *    time series = (n_t+1) scalar fields back to back (field.hpp:129-151).
 *    Spectra are complex128 interleaved (re,im), dims (n1, n2, n3/2+1) row-major
 *    (fft.hpp:12-23).
 *  - Functions ending in _host take HOST pointers and include the H2D/D2H copies.
 *  - Every call is ordered on the context's CUDA stream; calls that return host
 *    scalars synchronize that stream.
 *  - Return value: 0 on success, else a veloreg::ErrorCategory value
 *    (errors.hpp:9-17); vr_last_error() gives the thread-local message and
 *    vr_last_error_class() the exception subclass to rethrow.
 *  - Grids: every axis a power of two in [4, 1024] (the GPU FFT's domain).
 */
#ifndef VELOREG_GPU_H
#define VELOREG_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VR_ABI_VERSION 1

/* ---- status codes: veloreg::ErrorCategory (errors.hpp:9-17) ---------------- */
enum {
    VR_OK = 0,
    VR_ERR_IO = 2,
    VR_ERR_FORMAT = 3,
    VR_ERR_ARGUMENT = 4,
    VR_ERR_NUMERICS = 5,
    VR_ERR_CONVERGENCE = 6,
    VR_ERR_RESOURCE = 7,
    VR_ERR_LOGIC = 8
};
/* exception subclass of the last error (errors.hpp:32-67) */
enum {
    VR_EXC_NONE = 0,
    VR_EXC_IO = 1,
    VR_EXC_FORMAT = 2,
    VR_EXC_ARGUMENT = 3,
    VR_EXC_DIMENSION = 4, /* DimensionError : ArgumentError */
    VR_EXC_NUMERIC = 5,
    VR_EXC_CONVERGENCE = 6,
    VR_EXC_RESOURCE = 7,
    VR_EXC_LOGIC = 8
};
const char* vr_last_error(void);
int vr_last_error_class(void);
int vr_abi_version(void);

/* ---- model / solver parameter PODs ---------------------------------------- */
/* RegKind, spectral.hpp:71 */
enum { VR_REG_H1 = 0, VR_REG_H2 = 1, VR_REG_H3 = 2, VR_REG_HELMHOLTZ = 3 };
/* RegOpMode, spectral.hpp:104 */
enum { VR_REGOP_APPLY = 0, VR_REGOP_INVERSE = 1, VR_REGOP_INVERSE_SQRT = 2 };
/* ProjectionKind, spectral.hpp:115 */
enum { VR_PROJ_IDENTITY = 0, VR_PROJ_INCOMPRESSIBLE = 1, VR_PROJ_NEAR_INCOMPRESSIBLE = 2 };
/* TraceDirection, transport.hpp:17 */
enum { VR_TRACE_BACKWARD = 0, VR_TRACE_FORWARD = 1 };
/* StopReason, solver.hpp:35-41 */
enum {
    VR_STOP_ZERO_GRADIENT = 0,
    VR_STOP_CONVERGED_REL = 1,
    VR_STOP_CONVERGED_ABS = 2,
    VR_STOP_MAX_ITERATIONS = 3,
    VR_STOP_LINE_SEARCH_FAILURE = 4
};
/* Krylov preconditioner choice (solver.hpp:130-150, precond.hpp:93-110) */
enum { VR_PRECOND_NONE = 0, VR_PRECOND_SPECTRAL = 1, VR_PRECOND_TWO_LEVEL = 2 };

/* TwoLevelOptions (precond.hpp:46-53; defaults: PCG(0.1) inner, CHEB(10), 500 inner
 * iterations, 10 Lanczos steps, seed 1234) */
enum { VR_INNER_PCG = 0, VR_INNER_CHEB = 1 };
typedef struct {
    int inner;
    double kappa;
    int cheb_iterations;
    int max_inner_iterations;
    int lanczos_iterations;
    unsigned long long lanczos_seed;
} vr_twolevel_options;

/* RegNorm, spectral.hpp:75-102 (defaults: H2, gamma 1, squared, no penalty, beta_w 1e-4) */
typedef struct {
    int kind;
    double gamma;
    int helmholtz_squared;
    int div_penalty;
    double beta_w;
} vr_regnorm;

/* RegModel, objective.hpp:11-23 (defaults: K = identity, beta_v 1e-2, n_t 4, GN) */
typedef struct {
    vr_regnorm norm;
    int projection;
    double beta_v;
    int nt;
    int gauss_newton;
} vr_model;

/* SolverParams, solver.hpp:13-33 */
typedef struct {
    double eps_opt;
    double abs_grad_tol;
    int max_newton;
    int max_krylov;
    double armijo_c1;
    double armijo_backtrack;
    int armijo_max_trials;
    int squared_norm_stop;
} vr_solver_params;

/* SolveCounters, objective.hpp:26-31 */
typedef struct {
    long objective_evals;
    long gradient_evals;
    long hessian_matvecs;
    long pde_solves;
} vr_counters;

/* IterationRecord, solver.hpp:45-58 */
typedef struct {
    int k;
    double objective;
    double mismatch_rel;
    double grad_norm;
    double grad_rel;
    double step_length;
    double forcing;
    int inner_iterations;
    long fine_matvecs;
    long coarse_matvecs;
    long pde_solves;
    double wall_time_s;
} vr_iteration_record;

/* SolveReport, solver.hpp:60-75 (records returned separately) */
typedef struct {
    int stop;
    int success;
    int outer_iterations;
    double grad0;
    double final_grad_rel;
    double final_mismatch_rel;
    double final_objective;
    double wall_time_s;
    vr_counters fine;
    vr_counters coarse;
    int n_records; /* number of IterationRecords produced */
} vr_solve_report;

/* PcgStats, solver.hpp:87-93 */
typedef struct {
    int iterations;
    double rel_residual;
    int converged;
    int negative_curvature;
    int hit_max_iterations;
} vr_pcg_stats;

void vr_model_default(vr_model* m);
void vr_twolevel_options_default(vr_twolevel_options* o);
void vr_solver_params_default(vr_solver_params* p);
/* RegModel::validate / RegNorm::validate / SolverParams::validate */
int vr_model_validate(const vr_model* m);
int vr_solver_params_validate(const vr_solver_params* p);

/* ---- context: one grid, one device, one stream ---------------------------- */
typedef struct vr_ctx vr_ctx;
/* Grid3 ctor (grid.hpp:24-31): DimensionError for dims < 4 or not a power of two <= 1024 */
int vr_ctx_create(int n1, int n2, int n3, int device, vr_ctx** out);
int vr_ctx_destroy(vr_ctx* ctx);
int vr_ctx_synchronize(vr_ctx* ctx);
void* vr_ctx_stream(vr_ctx* ctx); /* cudaStream_t */
int vr_ctx_grid(const vr_ctx* ctx, int dims[3]);
/* kernels launched on this ctx since creation / last reset (evidence counter) */
long long vr_ctx_kernel_launches(const vr_ctx* ctx);
/* device-memory accounting of this context's library allocations (the reference's
 * FieldAllocStats live / peak, proj/include/veloreg/field.hpp:16-33, in bytes), and the
 * device's stream-ordered pool high-water mark (may be NULL) */
int vr_ctx_memory(const vr_ctx* ctx, long long* live_bytes, long long* peak_bytes,
                  long long* pool_reserved_high);
int vr_ctx_reset_memory_peak(vr_ctx* ctx); /* FieldAllocStats::reset_peak */
void vr_ctx_reset_kernel_launches(vr_ctx* ctx);

/* Optional per-launch CUDA-event timing on the ctx stream (bench / roofline
 * evidence). While on, work that normally overlaps on the side stream runs
 * in order on the ctx stream, so each event pair brackets one kernel running
 * alone. vr_ctx_profile_read writes "category,launches,total_ms" lines
 * for the launches since profiling was enabled (or last read) and resets. */
int vr_ctx_set_profiling(vr_ctx* ctx, int on);
int vr_ctx_profile_read(vr_ctx* ctx, char* buf, size_t len);

/* device / pinned memory plumbing */
int vr_device_alloc(vr_ctx* ctx, size_t bytes, void** out);
int vr_device_free(vr_ctx* ctx, void* p);
int vr_host_alloc_pinned(size_t bytes, void** out);
int vr_host_free_pinned(void* p);
int vr_memcpy_h2d(vr_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes); /* async */
int vr_memcpy_d2h(vr_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes); /* syncs */
int vr_memcpy_d2d(vr_ctx* ctx, void* dst_dev, const void* src_dev, size_t bytes); /* async */
int vr_memset_zero(vr_ctx* ctx, void* dst_dev, size_t bytes);                     /* async */

/* ---- BLAS-1 with deterministic reductions (field_ops.hpp:14-111) --------- */
/* ncomp = 1 (ScalarField) or 3 (VectorField); 'n' fields of the grid */
int vr_scale(vr_ctx* ctx, double* x, int ncomp, double a);                               /* scale */
int vr_add_scaled(vr_ctx* ctx, double* y, double a, const double* x, int ncomp);          /* add_scaled */
int vr_lin_comb(vr_ctx* ctx, double* out, double a, const double* x, double b, const double* y,
                int ncomp);                                                              /* lin_comb */
int vr_dot_l2(vr_ctx* ctx, const double* a, const double* b, int ncomp, double* out);    /* dot_l2 */
int vr_norm_l2(vr_ctx* ctx, const double* a, int ncomp, double* out);                    /* norm_l2 */
int vr_max_abs(vr_ctx* ctx, const double* a, int ncomp, double* out);                    /* max_abs */
int vr_max_magnitude(vr_ctx* ctx, const double* v3, double* out);                        /* max_magnitude */
int vr_all_finite(vr_ctx* ctx, const double* a, int ncomp, int* out);                    /* all_finite */
/* weighted h1*h2*h3 * sum a*b (spectral.cpp:47-62) */
int vr_inner_product(vr_ctx* ctx, const double* a, const double* b, int ncomp, double* out);

/* ---- spectral operators (fft.hpp, spectral.hpp) ---------------------------- */
/* fft_forward_raw (fft.cpp:66-73): unnormalized r2c */
int vr_fft_r2c(vr_ctx* ctx, const double* in, double* out_spectrum);
/* fft_inverse_raw (fft.cpp:75-83): c2r including the 1/N scale */
int vr_fft_c2r(vr_ctx* ctx, const double* spectrum, double* out);
int vr_gradient(vr_ctx* ctx, const double* f, double* out3);              /* spectral.cpp:108-122 */
int vr_divergence(vr_ctx* ctx, const double* v3, double* out);            /* spectral.cpp:124-140 */
int vr_laplacian(vr_ctx* ctx, const double* f, double* out, int ncomp);   /* spectral.cpp:142-153 */
int vr_helmholtz1_apply(vr_ctx* ctx, const double* f, double* out);       /* spectral.cpp:155-160 */
int vr_gaussian_smooth(vr_ctx* ctx, const double* f, double* out, int ncomp,
                       const double sigma_voxels[3]);                     /* spectral.cpp:84-106 */
int vr_apply_reg_operator(vr_ctx* ctx, const double* v3, double* out3, const vr_regnorm* norm,
                          int mode, double beta);                         /* spectral.cpp:166-184 */
int vr_apply_projection(vr_ctx* ctx, const double* f3, double* out3, int kind, double beta_v,
                        double beta_w);                                   /* spectral.cpp:190-222 */
int vr_rescale_intensity(vr_ctx* ctx, const double* f, double* out, int* degenerate); /* spectral.cpp:64-78 */

/* ---- semi-Lagrangian transport (interp.hpp, transport.hpp) ------------------ */
int vr_tricubic_interpolate(vr_ctx* ctx, const double* f, const double* points3, double* out,
                            int nfields /* 1..3: f holds nfields fields */); /* interp.hpp:80-126 */
int vr_trace_characteristics(vr_ctx* ctx, const double* v3, int nt, int direction,
                             double* departure3);                              /* transport.cpp:11-42 */
int vr_continuity_factor(vr_ctx* ctx, const double* div_v, const double* departure3, double dt,
                         double* factor);                                      /* transport.cpp:44-55 */
int vr_solve_state(vr_ctx* ctx, const double* m_T, const double* v3, int nt,
                   double* history);                                           /* transport.cpp:72-86 */
/* solve_adjoint (transport.cpp:115-124); history (nt+1 fields) may be NULL, initial may be NULL */
int vr_solve_adjoint(vr_ctx* ctx, const double* terminal, const double* v3, int nt,
                     double* history, double* initial);
int vr_gradient_dot(vr_ctx* ctx, const double* f, const double* w3, double* out); /* transport.cpp:126-148 */
int vr_solve_inc_state(vr_ctx* ctx, const double* m_history, const double* v3, const double* vt3,
                       int nt, double* mt_history);                            /* transport.cpp:150-180 */
/* Gauss-Newton branch of solve_inc_adjoint (transport.cpp:182-191, :228-237) */
int vr_solve_inc_adjoint(vr_ctx* ctx, const double* terminal, const double* v3, int nt,
                         double* history, double* initial);

/* ---- fp32 lane (one GPU): the float instantiations of the
 * semi-Lagrangian operators (T = float in interp.hpp:80-126, transport.cpp:11-42, :72-86).
 * Fields and departure points are fp32 device arrays; stencils and sums run in fp64 and
 * results are rounded to fp32, as in the reference. */
int vr_tricubic_interpolate_f32(vr_ctx* ctx, const float* f, const float* points3, float* out,
                                int nfields);
int vr_trace_characteristics_f32(vr_ctx* ctx, const float* v3, int nt, int direction,
                                 float* departure3);
int vr_solve_state_f32(vr_ctx* ctx, const float* m_T, const float* v3, int nt, float* history);
/* spectral operators with fp32 fields; the transforms run in fp64 and the half spectrum
 * stays complex128 (fft.hpp:12-23: "f32 fields are converted at the boundary") */
int vr_fft_r2c_f32(vr_ctx* ctx, const float* in, double* out_spectrum);
int vr_fft_c2r_f32(vr_ctx* ctx, const double* spectrum, float* out);
int vr_gradient_f32(vr_ctx* ctx, const float* f, float* out3);
int vr_divergence_f32(vr_ctx* ctx, const float* v3, float* out);
int vr_gaussian_smooth_f32(vr_ctx* ctx, const float* f, float* out, int ncomp,
                           const double sigma_voxels[3]);
int vr_apply_reg_operator_f32(vr_ctx* ctx, const float* v3, float* out3, const vr_regnorm* norm,
                              int mode, double beta);
int vr_apply_projection_f32(vr_ctx* ctx, const float* f3, float* out3, int kind, double beta_v,
                            double beta_w);

/* Objective<float> (objective.cpp:35-156 with T = float; Gauss-Newton, one GPU): fp32
 * images, velocities, directions and gradients (device pointers); fields stored in fp32
 * where the reference stores them, stencils / transforms / reductions in fp64. */
typedef struct vr_objective_f32 vr_objective_f32;
typedef struct vr_state_f32 vr_state_f32;
int vr_objective_f32_create(vr_ctx* ctx, const float* m_R, const float* m_T, const vr_model* model,
                            vr_objective_f32** out);
int vr_objective_f32_destroy(vr_objective_f32* obj);
int vr_objective_f32_counters(const vr_objective_f32* obj, vr_counters* out);
int vr_evaluate_f32(vr_objective_f32* obj, const float* v3, vr_state_f32** out_state);
int vr_state_f32_destroy(vr_state_f32* s);
int vr_state_f32_scalars(const vr_state_f32* s, double* objective, double* mismatch,
                         double* mismatch_rel);
int vr_compute_gradient_f32(vr_objective_f32* obj, vr_state_f32* s, float* g3);
int vr_hessian_matvec_f32(vr_objective_f32* obj, const vr_state_f32* s, const float* vt3,
                          float* out3);
/* gauss_newton_solve<float> (solver.cpp:154-269; PCG and Armijo on fp32 vectors with fp64
 * scalars); precond VR_PRECOND_NONE, VR_PRECOND_SPECTRAL or VR_PRECOND_TWO_LEVEL (default
 * options); gauss_newton = 0 selects the full-Newton Hessian; fp32 device pointers */
int vr_gauss_newton_solve_f32(vr_ctx* ctx, const float* m_R, const float* m_T, const float* v0,
                              const vr_model* model, const vr_solver_params* params, int precond,
                              float* v_out, vr_solve_report* report, vr_iteration_record* records,
                              int max_records);
/* the same with TwoLevelPreconditioner<float> (precond.cpp:153-249; opts may be NULL): the
 * Newton / split-system PCG iterates are fp32, the coarse-grid machinery behind M^-1 runs in fp64 */
int vr_gauss_newton_solve_two_level_f32(vr_ctx* ctx, const float* m_R, const float* m_T, const float* v0,
                                        const vr_model* model, const vr_solver_params* params,
                                        const vr_twolevel_options* opts, float* v_out,
                                        vr_solve_report* report, vr_iteration_record* records,
                                        int max_records);
/* parameter continuation over vr_gauss_newton_solve_f32 */
int vr_parameter_continuation_f32(vr_ctx* ctx, const float* m_R, const float* m_T, const float* v0,
                                  const vr_model* model, const vr_solver_params* params,
                                  int precond, float* v_out, vr_solve_report* reports,
                                  int max_levels, int* n_levels, vr_iteration_record* records,
                                  int max_records);

/* ---- Objective (objective.hpp:56-102) -------------------------------------- */
typedef struct vr_objective vr_objective;
typedef struct vr_state vr_state;
/* Objective ctor (objective.cpp:35-45); m_R, m_T are device pointers that must
 * outlive the objective (the reference holds non-owning pointers, objective.hpp:97-98).
 * counters may be NULL (then the objective keeps none, like counters_ == nullptr). */
int vr_objective_create(vr_ctx* ctx, const double* m_R, const double* m_T, const vr_model* model,
                        vr_objective** out);
int vr_objective_destroy(vr_objective* obj);
int vr_objective_initial_mismatch(const vr_objective* obj, double* out);
int vr_objective_counters(const vr_objective* obj, vr_counters* out);
int vr_objective_reset_counters(vr_objective* obj);
int vr_objective_set_beta(vr_objective* obj, double beta_v); /* continuation levels */

/* evaluate (objective.cpp:47-75): state solve + J. 1 PDE solve. */
int vr_evaluate(vr_objective* obj, const double* v3, vr_state** out_state);
int vr_state_destroy(vr_state* s);
/* EvalState scalars (objective.hpp:37-54) */
int vr_state_scalars(const vr_state* s, double* objective, double* mismatch, double* mismatch_rel,
                     int* has_gradient, int* has_adjoint_ctx);
/* copies of the frozen EvalState fields for parity checks */
enum {
    VR_STATE_V = 0,          /* 3 fields */
    VR_STATE_X_BWD = 1,      /* 3 fields */
    VR_STATE_X_FWD = 2,      /* 3 fields (after the gradient) */
    VR_STATE_FACTOR = 3,     /* 1 field  (after the gradient) */
    VR_STATE_M_HISTORY = 4,  /* nt+1 fields */
    VR_STATE_GRADIENT = 5,   /* 3 fields (after the gradient) */
    VR_STATE_GRAD_M = 6,     /* 3*(nt+1) fields: d_a m_j at [j*3 + a] (after the gradient) */
    VR_STATE_LAMBDA_HISTORY = 7 /* nt+1 fields: adjoint lambda_j (full Newton, after the gradient) */
};
int vr_state_get(const vr_state* s, int which, double* out_dev);
/* compute_gradient (objective.cpp:77-112): adjoint sweep with fused accumulation. 1 PDE solve.
 * g3 (device, may be NULL) receives a copy of the gradient. */
int vr_compute_gradient(vr_objective* obj, vr_state* s, double* g3);
/* hessian_matvec (objective.cpp:114-121): H vt = H_data vt + beta_v A vt. 2 PDE solves. */
int vr_hessian_matvec(vr_objective* obj, const vr_state* s, const double* vt3, double* out3);
/* same, HOST buffers in and out (H2D + matvec + D2H): the end-to-end entry */
int vr_hessian_matvec_host(vr_objective* obj, const vr_state* s, const double* vt3_host,
                           double* out3_host);
/* pipelined form of vr_hessian_matvec_host for a stream of independent directions:
 * returns once the work is queued; uploads (own stream), the matvec (ctx stream) and
 * downloads (own stream) of consecutive calls overlap through two device slots. Host
 * buffers (pinned for real overlap) must stay valid and vt3_host unmodified until
 * vr_objective_wait returns; non-finite directions surface there as NumericError. */
int vr_hessian_matvec_host_async(vr_objective* obj, const vr_state* s, const double* vt3_host,
                                 double* out3_host);
int vr_objective_wait(vr_objective* obj);
/* hessian_data_matvec (objective.cpp:123-156) */
int vr_hessian_data_matvec(vr_objective* obj, const vr_state* s, const double* vt3, double* out3);
/* apply_reg / apply_K (objective.cpp:178-186) */
int vr_objective_apply_reg(vr_objective* obj, const double* u3, int mode, double* out3);
int vr_objective_apply_K(vr_objective* obj, const double* u3, double* out3);

/* ---- solvers (solver.hpp:78-164; host driver over the device operators) ---- */
int vr_compute_forcing(double grad_norm, double grad0_norm, double* out); /* solver.cpp:23-27 */
/* SolveReport::write_csv (solver.cpp:29-47): the reference's CSV of a report and its
 * records into buf (NUL-terminated; *needed = bytes required, may be NULL; buf NULL to size) */
int vr_solve_report_csv(const vr_solve_report* report, const vr_iteration_record* records,
                        const char* comment, char* buf, size_t len, size_t* needed);
/* pcg_solve on the GN Hessian of (obj, s) with the chosen preconditioner (solver.cpp:51-100) */
int vr_pcg_solve(vr_objective* obj, const vr_state* s, const double* rhs3, double rel_tol,
                 int max_iter, int precond, double* x3, vr_pcg_stats* stats);
/* gauss_newton_solve (solver.cpp:154-269): all pointers device; v_out may alias nothing.
 * records (host, may be NULL) receives up to max_records IterationRecords. */
int vr_gauss_newton_solve(vr_ctx* ctx, const double* m_R, const double* m_T, const double* v0,
                          const vr_model* model, const vr_solver_params* params, int precond,
                          double* v_out, vr_solve_report* report, vr_iteration_record* records,
                          int max_records);
/* Parameter continuation in beta_v: levels 1, 1e-1, ... down to
 * model->beta_v (last level snapped to the target), each warm-started from the
 * previous velocity. reports[level] / records (concatenated) are filled for
 * up to max_levels levels; *n_levels receives the number of levels run. */
int vr_parameter_continuation(vr_ctx* ctx, const double* m_R, const double* m_T, const double* v0,
                              const vr_model* model, const vr_solver_params* params, int precond,
                              double* v_out, vr_solve_report* reports, int max_levels,
                              int* n_levels, vr_iteration_record* records, int max_records);

/* Grid continuation (not in the reference code): n_grid_levels grids,
 * each axis halved per level (coarsest >= 16 points per axis). A coarse level solves on
 * the spectrally restricted images smoothed with sigma = 1 voxel of that level, starting
 * from the previous level's velocity prolonged spectrally (the coarsest starts from v0
 * restricted); the finest level solves on the original images. One GPU. */
int vr_grid_continuation(vr_ctx* ctx, const double* m_R, const double* m_T, const double* v0,
                         const vr_model* model, const vr_solver_params* params, int precond,
                         int n_grid_levels, double* v_out, vr_solve_report* reports,
                         int max_levels, int* n_levels, vr_iteration_record* records,
                         int max_records);
/* Scale continuation: sigmas (voxels, strictly decreasing, >= 0; 0 =
 * the unsmoothed images), images re-smoothed from the originals per level, warm starts */
int vr_scale_continuation(vr_ctx* ctx, const double* m_R, const double* m_T, const double* v0,
                          const vr_model* model, const vr_solver_params* params, int precond,
                          const double* sigmas, int n_sigmas, double* v_out,
                          vr_solve_report* reports, int max_levels, int* n_levels,
                          vr_iteration_record* records, int max_records);
/* BetaSearchParams: eps_J, bracket [beta_lo, beta_hi] (defaults
 * 0.1 (H2, Table 2), [1e-5, 1]), at most max_bisections midpoints (10), stop below
 * min_width_decades (0.25) */
typedef struct {
    double eps_J;
    double beta_lo, beta_hi;
    int max_bisections;
    double min_width_decades;
} vr_beta_search_params;
void vr_beta_search_params_default(vr_beta_search_params* p);
/* det grad y summary (DetStats, postprocess.hpp:23-27) */
typedef struct {
    double min, mean, max;
} vr_det_summary;
/* one trial of the search: beta_v, feasibility, det grad y of its velocity, its solve */
typedef struct {
    double beta;
    int feasible;
    vr_det_summary det;
    vr_solve_report report;
} vr_beta_trial;
/* Beta search: trials at beta_hi, then beta_lo, then bisection on
 * log10 beta_v; each warm-started from the previous trial's velocity. Returns the
 * smallest feasible beta (*beta_out) and its velocity. No feasible beta in the bracket
 * (beta_hi infeasible): VR_ERR_NUMERICS / NumericError with the trials filled in. */
int vr_beta_search(vr_ctx* ctx, const double* m_R, const double* m_T, const double* v0,
                   const vr_model* model, const vr_solver_params* params, int precond,
                   const vr_beta_search_params* bp, double* beta_out, double* v_out,
                   vr_beta_trial* trials, int max_trials, int* n_trials);

/* ---- postprocess (postprocess.hpp:9-56; one GPU) ------------ */
/* det_deformation_gradient (postprocess.cpp:13-29) */
int vr_det_deformation_gradient(vr_ctx* ctx, const double* v3, int nt, double* det);
/* deformation_map (postprocess.cpp:31-60): displacement u, or y = wrap(x + u) */
int vr_deformation_map(vr_ctx* ctx, const double* v3, int nt, int absolute, double* out3);
/* det_stats (postprocess.cpp:62-81): foreground may be NULL (else voxels with
 * foreground < threshold are skipped); all zero when nothing is counted */
int vr_det_stats(vr_ctx* ctx, const double* det, const double* foreground, double threshold,
                 vr_det_summary* out);
/* transport_labels (postprocess.cpp:83-120): ResourceError above 64 distinct codes */
int vr_transport_labels(vr_ctx* ctx, const double* labels, const double* v3, int nt,
                        double* out);
/* OverlapScores (postprocess.hpp:41-45) */
typedef struct {
    double dice;
    double false_positive_rate;
    double false_negative_rate;
} vr_overlap;
/* overlap_scores (postprocess.cpp:122-165): *n_labels = distinct nonzero codes of both
 * maps (ascending); the first max_labels go to codes / per_label; mask may be NULL
 * (else voxels with mask < 0.5 are skipped). Codes must span < 2^24 values. */
int vr_overlap_scores(vr_ctx* ctx, const double* reference, const double* test,
                      const double* mask, int max_labels, int* n_labels, int* codes,
                      vr_overlap* per_label, vr_overlap* union_scores);

/* ---- two-level preconditioner and grid transfer (one GPU) ---- */
/* spectral_resample (spectral.cpp:340-356): field on src's grid -> dst's grid (coarser or
 * finer on every axis, same device); ncomp 1 or 3 */
int vr_spectral_resample(vr_ctx* src, const double* in, int ncomp, vr_ctx* dst, double* out);
/* frequency_filter (spectral.cpp:358-385): band 0 = low (F_L), 1 = high (F_H) w.r.t. cutoff */
int vr_frequency_filter(vr_ctx* ctx, const double* in, int ncomp, int band, const int cutoff[3],
                        double* out);
/* Objective::split_matvec (objective.cpp:158-176): (I + R H_data R) w, R = (beta_v A)^-1/2 */
int vr_split_matvec(vr_objective* obj, const vr_state* state, const double* w3, double* out3);
/* TwoLevelPreconditioner (precond.hpp:55-110): rebuild per outer iteration, apply = the
 * approximate inverse of the split system; counters = the coarse SolveCounters */
typedef struct vr_twolevel vr_twolevel;
int vr_twolevel_create(const vr_twolevel_options* opts, vr_twolevel** out);
int vr_twolevel_destroy(vr_twolevel* tl);
int vr_twolevel_rebuild(vr_twolevel* tl, vr_objective* obj, const vr_state* state, double eps_H);
int vr_twolevel_apply(vr_twolevel* tl, vr_ctx* ctx, const double* r3, double* z3);
/* coarse split matvec on the coarse grid (dims via vr_twolevel_info) */
int vr_twolevel_coarse_matvec(vr_twolevel* tl, const double* u3, double* out3);
/* coarse dims[3], lanczos_runs, inner_diverged, eigenvalue bounds, coarse counters */
int vr_twolevel_info(const vr_twolevel* tl, int dims[3], int* lanczos_runs, int* inner_diverged,
                     double bounds[2], vr_counters* coarse);
/* gauss_newton_solve with the two-level preconditioner (opts NULL = defaults): the
 * outer PCG runs on the split system (solver.cpp:208-221); report->coarse and
 * records[k].coarse_matvecs carry the coarse counters */
int vr_gauss_newton_solve_two_level(vr_ctx* ctx, const double* m_R, const double* m_T,
                                    const double* v0, const vr_model* model,
                                    const vr_solver_params* params,
                                    const vr_twolevel_options* opts, double* v_out,
                                    vr_solve_report* report, vr_iteration_record* records,
                                    int max_records);

/* ---- x1-slab decomposition across GPUs (no reference counterpart:
 * the reference is single-process, the paper's CLAIRE used MPI pencils,
 * PAPER.md:475-479). Rank r of P owns planes [r n1/P, (r+1) n1/P); n1 and n2 must
 * be divisible by P. Field arguments of the objective / solver entry points are
 * then this rank's slab (n1/P x n2 x n3, same row-major layout); reductions
 * return global values on every rank. Per-operator entry points (FFT, tricubic,
 * transport solves) stay one-GPU only and raise ArgumentError on a slab ctx.
 * `halo` = x1 planes exchanged on each side of every gathered field; it must
 * cover the largest per-step x1 displacement + 4 (checked per velocity). */
/* Host-only slab geometry (no GPU, no context): validates (n1,n2,n3,nranks,halo)
 * as vr_ctx_create_dist does and fills out[VR_SLAB_FIELDS] =
 * {planes L, first_plane off1, halo H, x2 rows per rank of the transposed
 *  spectrum n2s, first x2 row k2_off, local points L n2 n3, local spectrum
 *  L n2 (n3/2+1), halo-padded field stride (L+2H) n2 n3, global points}. */
#define VR_SLAB_FIELDS 9
int vr_slab_layout(int n1, int n2, int n3, int rank, int nranks, int halo, long long* out);
/* Halo planes a velocity with max |v_1| = vmax_x1 needs at n_t steps on an n1
 * grid (the check vr_evaluate applies on a slab context). */
int vr_slab_halo_required(double vmax_x1, int nt, int n1, int* planes);
/* NCCL unique id (128 bytes) created on one rank and broadcast by the caller */
int vr_nccl_unique_id(unsigned char out[128]);
/* one process per GPU: NCCL communicator over nranks, this process = rank */
int vr_ctx_create_dist(int n1, int n2, int n3, int device, int rank, int nranks,
                       const unsigned char uid[128], int halo, vr_ctx** out);
int vr_ctx_slab(const vr_ctx* ctx, int* rank, int* nranks, int* planes, int* first_plane,
                int* halo);
/* Self tests of the slab path on ONE GPU: P virtual ranks (host threads, device
 * copies between host barriers, no cross-rank kernel waits) run on slabs of the
 * global HOST inputs; outputs are assembled into global HOST arrays.
 * scalars[5] = J, mismatch, mismatch_rel, ||g||_2, <H vt, vt> (unweighted). */
int vr_dist_selftest_objective(int P, int n1, int n2, int n3, int device, int halo,
                               const vr_model* model, const double* m_R, const double* m_T,
                               const double* v, const double* vt, double* grad_out,
                               double* matvec_out, double* reg_out, double* scalars);
int vr_dist_selftest_solve(int P, int n1, int n2, int n3, int device, int halo,
                           const vr_model* model, const vr_solver_params* params,
                           const double* m_R, const double* m_T, const double* v0, double* v_out,
                           vr_solve_report* report);
/* det grad y, the absolute deformation map and det_stats of a velocity on P virtual slab ranks
 * (postprocess.cpp:13-81); stats3 = min, max, mean */
int vr_dist_selftest_postprocess(int P, int n1, int n2, int n3, int device, int halo, const double* v,
                                 int nt, double* det_out, double* map_out, double* stats3);
/* transport_labels of `labels` by v and overlap_scores(labels, warped) on P virtual slab ranks
 * (postprocess.cpp:83-165) */
int vr_dist_selftest_labels(int P, int n1, int n2, int n3, int device, int halo, const double* labels,
                            const double* v, int nt, double* warped_out, int max_labels, int* n_labels,
                            int* codes, vr_overlap* per_label, vr_overlap* union_scores);
/* The same with a preconditioner choice (VR_PRECOND_*; tl_opts may be NULL): the two-level
 * preconditioner on slabs (precond.cpp:153-249 with the coarse grid on a sibling slab context
 * and the coarse band exchanged between the ranks' k2 slabs) */
int vr_dist_selftest_solve_precond(int P, int n1, int n2, int n3, int device, int halo,
                                   const vr_model* model, const vr_solver_params* params, int precond,
                                   const vr_twolevel_options* tl_opts, const double* m_R,
                                   const double* m_T, const double* v0, double* v_out,
                                   vr_solve_report* report);

/* ---- synthetic inputs (synthetic.cpp:10-34) -------------------------------- */
/* m_T, v* analytic on the grid; m_R = solve_state(m_T, v*, nt).final() on the GPU */
int vr_generate_synthetic(vr_ctx* ctx, int nt, double amplitude, double* m_R, double* m_T,
                          double* v_star);

#ifdef __cplusplus
}
#endif

#endif /* VELOREG_GPU_H */
