// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// extern "C" harness over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see Makefile). It mirrors the product C ABI
// (include/veloreg_gpu.h) on HOST arrays with a `vref_` prefix so parity tests
// can call both sides with identical inputs. Only tests/, __graft_entry__.smoke()
// and bench.py's CPU-baseline legs load the resulting oracle/_ref/libveloreg_ref.so.
//
// It also exposes the reference test-suite input generators
// (proj/tests/test_support.hpp:46-114, used as-is) so GPU tests can reproduce
// the reference tests' seeded fields bit-for-bit.

#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "test_support.hpp"
#include "veloreg/field_ops.hpp"
#include "veloreg/fft.hpp"
#include "veloreg/objective.hpp"
#include "veloreg/parallel.hpp"
#include "veloreg/postprocess.hpp"
#include "veloreg/precond.hpp"
#include "veloreg/solver.hpp"
#include "veloreg/spectral.hpp"
#include "veloreg/synthetic.hpp"
#include "veloreg/transport.hpp"
#include "veloreg_gpu.h"

using namespace veloreg;

namespace {

thread_local std::string g_err;
thread_local int g_err_class = VR_EXC_NONE;

template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return VR_OK;
    } catch (const DimensionError& e) {
        g_err = e.what();
        g_err_class = VR_EXC_DIMENSION;
        return VR_ERR_ARGUMENT;
    } catch (const Error& e) {
        g_err = e.what();
        switch (e.category()) {
            case ErrorCategory::io: g_err_class = VR_EXC_IO; break;
            case ErrorCategory::format: g_err_class = VR_EXC_FORMAT; break;
            case ErrorCategory::argument: g_err_class = VR_EXC_ARGUMENT; break;
            case ErrorCategory::numerics: g_err_class = VR_EXC_NUMERIC; break;
            case ErrorCategory::convergence: g_err_class = VR_EXC_CONVERGENCE; break;
            case ErrorCategory::resource: g_err_class = VR_EXC_RESOURCE; break;
            case ErrorCategory::logic: g_err_class = VR_EXC_LOGIC; break;
        }
        return static_cast<int>(e.category());
    } catch (const std::exception& e) {
        g_err = e.what();
        g_err_class = VR_EXC_LOGIC;
        return VR_ERR_LOGIC;
    }
}

Grid3 grid_of(const int* d) { return Grid3(d[0], d[1], d[2]); }

ScalarField<double> load_scalar(const Grid3& g, const double* p) {
    ScalarField<double> f(g);
    std::memcpy(f.data(), p, sizeof(double) * g.size());
    return f;
}
VectorField<double> load_vector(const Grid3& g, const double* p) {
    VectorField<double> v(g);
    for (int c = 0; c < 3; ++c) std::memcpy(v[c].data(), p + c * g.size(), sizeof(double) * g.size());
    return v;
}
void store(const ScalarField<double>& f, double* p) {
    std::memcpy(p, f.data(), sizeof(double) * f.size());
}
void store(const VectorField<double>& v, double* p) {
    for (int c = 0; c < 3; ++c) std::memcpy(p + c * v.size(), v[c].data(), sizeof(double) * v.size());
}
void store(const TimeSeries<double>& t, double* p) {
    for (int j = 0; j < t.slice_count(); ++j) store(t.slice(j), p + j * t.slice(0).size());
}

// fp32 lane: the reference's float instantiations (ScalarField<float>, ...)
ScalarField<float> load_scalar_f(const Grid3& g, const float* p) {
    ScalarField<float> f(g);
    std::memcpy(f.data(), p, sizeof(float) * g.size());
    return f;
}
VectorField<float> load_vector_f(const Grid3& g, const float* p) {
    VectorField<float> v(g);
    for (int c = 0; c < 3; ++c) std::memcpy(v[c].data(), p + c * g.size(), sizeof(float) * g.size());
    return v;
}
void store_f(const ScalarField<float>& f, float* p) { std::memcpy(p, f.data(), sizeof(float) * f.size()); }
void store_f(const VectorField<float>& v, float* p) {
    for (int c = 0; c < 3; ++c) std::memcpy(p + c * v.size(), v[c].data(), sizeof(float) * v.size());
}

RegNorm to_norm(const vr_regnorm& n) {
    RegNorm r;
    r.kind = static_cast<RegKind>(n.kind);
    r.gamma = n.gamma;
    r.helmholtz_squared = n.helmholtz_squared != 0;
    r.div_penalty = n.div_penalty != 0;
    r.beta_w = n.beta_w;
    return r;
}
RegModel to_model(const vr_model& m) {
    RegModel r;
    r.norm = to_norm(m.norm);
    r.projection = static_cast<ProjectionKind>(m.projection);
    r.beta_v = m.beta_v;
    r.nt = m.nt;
    r.gauss_newton = m.gauss_newton != 0;
    return r;
}
SolverParams to_params(const vr_solver_params& p) {
    SolverParams s;
    s.eps_opt = p.eps_opt;
    s.abs_grad_tol = p.abs_grad_tol;
    s.max_newton = p.max_newton;
    s.max_krylov = p.max_krylov;
    s.armijo_c1 = p.armijo_c1;
    s.armijo_backtrack = p.armijo_backtrack;
    s.armijo_max_trials = p.armijo_max_trials;
    s.squared_norm_stop = p.squared_norm_stop != 0;
    return s;
}
void fill_counters(const SolveCounters& c, vr_counters* o) {
    o->objective_evals = c.objective_evals;
    o->gradient_evals = c.gradient_evals;
    o->hessian_matvecs = c.hessian_matvecs;
    o->pde_solves = c.pde_solves;
}
void fill_report(const SolveReport& r, vr_solve_report* o, vr_iteration_record* recs, int max_recs,
                 int rec_offset) {
    o->stop = static_cast<int>(r.stop);
    o->success = r.success;
    o->outer_iterations = r.outer_iterations;
    o->grad0 = r.grad0;
    o->final_grad_rel = r.final_grad_rel;
    o->final_mismatch_rel = r.final_mismatch_rel;
    o->final_objective = r.final_objective;
    o->wall_time_s = r.wall_time_s;
    fill_counters(r.fine, &o->fine);
    fill_counters(r.coarse, &o->coarse);
    o->n_records = static_cast<int>(r.iterations.size());
    if (!recs) return;
    for (std::size_t i = 0; i < r.iterations.size(); ++i) {
        const int slot = rec_offset + static_cast<int>(i);
        if (slot >= max_recs) break;
        const auto& a = r.iterations[i];
        vr_iteration_record& b = recs[slot];
        b.k = a.k;
        b.objective = a.objective;
        b.mismatch_rel = a.mismatch_rel;
        b.grad_norm = a.grad_norm;
        b.grad_rel = a.grad_rel;
        b.step_length = a.step_length;
        b.forcing = a.forcing;
        b.inner_iterations = a.inner_iterations;
        b.fine_matvecs = a.fine_matvecs;
        b.coarse_matvecs = a.coarse_matvecs;
        b.pde_solves = a.pde_solves;
        b.wall_time_s = a.wall_time_s;
    }
}

} // namespace

struct vref_objective {
    Grid3 g;
    ScalarField<double> m_R, m_T;
    SolveCounters counters;
    std::unique_ptr<Objective<double>> obj;
};
struct vref_state {
    EvalState<double> s;
};
// fp32 lane: Objective<float>
struct vref_objective_f32 {
    Grid3 g;
    ScalarField<float> m_R, m_T;
    SolveCounters counters;
    std::unique_ptr<Objective<float>> obj;
};
struct vref_state_f32 {
    EvalState<float> s;
};
struct vref_twolevel {
    explicit vref_twolevel(const TwoLevelOptions& o) : pre(o) {}
    TwoLevelPreconditioner<double> pre;
    Grid3 fine;
};
static TwoLevelOptions to_tl(const vr_twolevel_options* o) {
    TwoLevelOptions t;
    if (!o) return t;
    t.inner = o->inner == VR_INNER_CHEB ? TwoLevelOptions::Inner::cheb : TwoLevelOptions::Inner::pcg;
    t.kappa = o->kappa;
    t.cheb_iterations = o->cheb_iterations;
    t.max_inner_iterations = o->max_inner_iterations;
    t.lanczos_iterations = o->lanczos_iterations;
    t.lanczos_seed = o->lanczos_seed;
    return t;
}

extern "C" {

const char* vref_last_error(void) { return g_err.c_str(); }
int vref_last_error_class(void) { return g_err_class; }
void vref_set_workers(int n) { par::set_workers(n); }
int vref_workers(void) { return par::workers(); }

// ---- FFT / spectral ---------------------------------------------------------
int vref_fft_r2c(const int* d, const double* in, double* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        fft_forward_raw(g, in, reinterpret_cast<std::complex<double>*>(out));
    });
}
int vref_fft_c2r(const int* d, const double* in, double* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        fft_inverse_raw(g, reinterpret_cast<const std::complex<double>*>(in), out);
    });
}
int vref_gradient(const int* d, const double* f, double* out3) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(gradient(load_scalar(g, f)), out3);
    });
}
int vref_divergence(const int* d, const double* v3, double* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(divergence(load_vector(g, v3)), out);
    });
}
int vref_laplacian(const int* d, const double* f, double* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(laplacian(load_scalar(g, f)), out);
    });
}
int vref_helmholtz1_apply(const int* d, const double* f, double* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(helmholtz1_apply(load_scalar(g, f)), out);
    });
}
int vref_gaussian_smooth(const int* d, const double* f, double* out, const double* sigma) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(gaussian_smooth(load_scalar(g, f), {sigma[0], sigma[1], sigma[2]}), out);
    });
}
int vref_apply_reg_operator(const int* d, const double* v3, double* out3, const vr_regnorm* n,
                            int mode, double beta) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(apply_reg_operator(load_vector(g, v3), to_norm(*n), static_cast<RegOpMode>(mode),
                                 beta),
              out3);
    });
}
int vref_apply_projection(const int* d, const double* v3, double* out3, int kind, double bv,
                          double bw) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(apply_projection(load_vector(g, v3), static_cast<ProjectionKind>(kind), bv, bw),
              out3);
    });
}
int vref_rescale_intensity(const int* d, const double* f, double* out, int* degenerate) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto r = rescale_intensity(load_scalar(g, f));
        store(r.field, out);
        *degenerate = r.degenerate;
    });
}
int vref_inner_product(const int* d, const double* a, const double* b, int ncomp, double* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        if (ncomp == 3)
            *out = inner_product(load_vector(g, a), load_vector(g, b));
        else
            *out = inner_product(load_scalar(g, a), load_scalar(g, b));
    });
}
int vref_dot_l2(const int* d, const double* a, const double* b, int ncomp, double* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        if (ncomp == 3)
            *out = dot_l2(load_vector(g, a), load_vector(g, b));
        else
            *out = dot_l2(load_scalar(g, a), load_scalar(g, b));
    });
}
int vref_max_magnitude(const int* d, const double* v3, double* out) {
    return guard([&] { *out = max_magnitude(load_vector(grid_of(d), v3)); });
}

// ---- interpolation / transport -----------------------------------------------
int vref_tricubic_interpolate(const int* d, const double* f, const double* pts3, double* out,
                              int nfields) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto pts = load_vector(g, pts3);
        const std::int64_t n = g.size();
        if (nfields == 1) {
            store(tricubic_interpolate(load_scalar(g, f), pts), out);
        } else if (nfields == 2) {
            ScalarField<double> o1, o2;
            tricubic_interpolate2(load_scalar(g, f), load_scalar(g, f + n), pts, o1, o2);
            store(o1, out);
            store(o2, out + n);
        } else {
            VectorField<double> o;
            tricubic_interpolate3(load_vector(g, f), pts, o);
            store(o, out);
        }
    });
}
int vref_trace_characteristics(const int* d, const double* v3, int nt, int dir, double* dep3) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto ch = trace_characteristics(load_vector(g, v3), nt,
                                        dir == VR_TRACE_FORWARD ? TraceDirection::forward
                                                                : TraceDirection::backward);
        store(ch.departure, dep3);
    });
}
int vref_tricubic_interpolate_f32(const int* d, const float* f, const float* pts3, float* out,
                                  int nfields) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto pts = load_vector_f(g, pts3);
        const std::int64_t n = g.size();
        if (nfields == 1) {
            store_f(tricubic_interpolate(load_scalar_f(g, f), pts), out);
        } else if (nfields == 2) {
            ScalarField<float> o1, o2;
            tricubic_interpolate2(load_scalar_f(g, f), load_scalar_f(g, f + n), pts, o1, o2);
            store_f(o1, out);
            store_f(o2, out + n);
        } else {
            VectorField<float> o;
            tricubic_interpolate3(load_vector_f(g, f), pts, o);
            store_f(o, out);
        }
    });
}
int vref_trace_characteristics_f32(const int* d, const float* v3, int nt, int dir, float* dep3) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto ch = trace_characteristics(load_vector_f(g, v3), nt,
                                        dir == VR_TRACE_FORWARD ? TraceDirection::forward
                                                                : TraceDirection::backward);
        store_f(ch.departure, dep3);
    });
}
int vref_solve_state_f32(const int* d, const float* mT, const float* v3, int nt, float* hist) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto h = solve_state(load_scalar_f(g, mT), load_vector_f(g, v3), nt);
        for (int j = 0; j < h.slice_count(); ++j) store_f(h.slice(j), hist + j * g.size());
    });
}
int vref_fft_r2c_f32(const int* d, const float* in, double* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        Spectrum sp;
        fft_forward(load_scalar_f(g, in), sp);
        std::memcpy(out, sp.data(), sizeof(std::complex<double>) * sp.size());
    });
}
int vref_fft_c2r_f32(const int* d, const double* in, float* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        Spectrum sp(spectrum_size(g));
        std::memcpy(sp.data(), in, sizeof(std::complex<double>) * sp.size());
        ScalarField<float> f(g);
        fft_inverse(g, sp, f);
        store_f(f, out);
    });
}
int vref_gradient_f32(const int* d, const float* f, float* out3) {
    return guard([&] { store_f(gradient(load_scalar_f(grid_of(d), f)), out3); });
}
int vref_divergence_f32(const int* d, const float* v3, float* out) {
    return guard([&] { store_f(divergence(load_vector_f(grid_of(d), v3)), out); });
}
int vref_gaussian_smooth_f32(const int* d, const float* f, float* out, const double* sigma) {
    return guard([&] {
        store_f(gaussian_smooth(load_scalar_f(grid_of(d), f), {sigma[0], sigma[1], sigma[2]}), out);
    });
}
int vref_apply_reg_operator_f32(const int* d, const float* v3, float* out3, const vr_regnorm* n,
                                int mode, double beta) {
    return guard([&] {
        store_f(apply_reg_operator(load_vector_f(grid_of(d), v3), to_norm(*n),
                                   static_cast<RegOpMode>(mode), beta),
                out3);
    });
}
int vref_apply_projection_f32(const int* d, const float* v3, float* out3, int kind, double bv,
                              double bw) {
    return guard([&] {
        store_f(apply_projection(load_vector_f(grid_of(d), v3), static_cast<ProjectionKind>(kind), bv, bw),
                out3);
    });
}
int vref_continuity_factor(const int* d, const double* div_v, const double* dep3, double dt,
                           double* factor) {
    return guard([&] {
        Grid3 g = grid_of(d);
        Characteristics<double> ch;
        ch.departure = load_vector(g, dep3);
        ch.dt = dt;
        ch.direction = TraceDirection::forward;
        store(continuity_factor(load_scalar(g, div_v), ch), factor);
    });
}
int vref_solve_state(const int* d, const double* mT, const double* v3, int nt, double* hist) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(solve_state(load_scalar(g, mT), load_vector(g, v3), nt), hist);
    });
}
int vref_solve_adjoint(const int* d, const double* term, const double* v3, int nt, double* hist,
                       double* initial) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto sol = solve_adjoint(load_scalar(g, term), load_vector(g, v3), nt, hist != nullptr);
        if (hist) store(*sol.history, hist);
        if (initial) store(sol.initial, initial);
    });
}
int vref_gradient_dot(const int* d, const double* f, const double* w3, double* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(gradient_dot(load_scalar(g, f), load_vector(g, w3)), out);
    });
}
int vref_solve_inc_state(const int* d, const double* mhist, const double* v3, const double* vt3,
                         int nt, int hist_slices, double* mt_hist) {
    return guard([&] {
        Grid3 g = grid_of(d);
        TimeSeries<double> h(g, hist_slices - 1);
        for (int j = 0; j < hist_slices; ++j) h.slice(j) = load_scalar(g, mhist + j * g.size());
        store(solve_inc_state(h, load_vector(g, v3), load_vector(g, vt3), nt), mt_hist);
    });
}
int vref_solve_inc_adjoint(const int* d, const double* term, const double* v3, int nt,
                           double* hist, double* initial) {
    return guard([&] {
        Grid3 g = grid_of(d);
        std::vector<ScalarField<double>> slices(nt + 1);
        SliceObserver<double> obs = [&](int j, const ScalarField<double>& f) { slices[j] = f; };
        auto v = load_vector(g, v3);
        auto sol = solve_inc_adjoint<double>(load_scalar(g, term), nullptr, v, v, nt, true, obs);
        if (hist)
            for (int j = 0; j <= nt; ++j) store(slices[j], hist + j * g.size());
        if (initial) store(sol.initial, initial);
    });
}

// ---- objective ------------------------------------------------------------------
int vref_objective_create(const int* d, const double* mR, const double* mT, const vr_model* m,
                          vref_objective** out) {
    return guard([&] {
        auto o = std::make_unique<vref_objective>();
        o->g = grid_of(d);
        o->m_R = load_scalar(o->g, mR);
        o->m_T = load_scalar(o->g, mT);
        o->obj = std::make_unique<Objective<double>>(o->m_R, o->m_T, to_model(*m), &o->counters);
        *out = o.release();
    });
}
void vref_objective_destroy(vref_objective* o) { delete o; }
int vref_objective_initial_mismatch(vref_objective* o, double* out) {
    return guard([&] { *out = o->obj->initial_mismatch(); });
}
int vref_objective_counters(vref_objective* o, vr_counters* out) {
    return guard([&] { fill_counters(o->counters, out); });
}
int vref_evaluate(vref_objective* o, const double* v3, vref_state** out) {
    return guard([&] {
        auto s = std::make_unique<vref_state>();
        s->s = o->obj->evaluate(load_vector(o->g, v3));
        *out = s.release();
    });
}
void vref_state_destroy(vref_state* s) { delete s; }
int vref_state_scalars(vref_state* s, double* J, double* mis, double* mis_rel, int* has_g,
                       int* has_ctx) {
    return guard([&] {
        *J = s->s.objective;
        *mis = s->s.mismatch;
        *mis_rel = s->s.mismatch_rel;
        *has_g = s->s.has_gradient;
        *has_ctx = s->s.has_adjoint_ctx;
    });
}
int vref_state_get(vref_state* st, int which, double* out) {
    return guard([&] {
        const auto& s = st->s;
        switch (which) {
            case VR_STATE_V: store(s.v, out); break;
            case VR_STATE_X_BWD: store(s.bwd.departure, out); break;
            case VR_STATE_X_FWD: store(s.fwd.departure, out); break;
            case VR_STATE_FACTOR: store(s.factor_fwd, out); break;
            case VR_STATE_M_HISTORY: store(s.m_history, out); break;
            case VR_STATE_GRADIENT: store(s.gradient, out); break;
            default: throw ArgumentError("vref_state_get: unsupported field");
        }
    });
}
int vref_compute_gradient(vref_objective* o, vref_state* s, double* g3) {
    return guard([&] {
        o->obj->compute_gradient(s->s);
        if (g3) store(s->s.gradient, g3);
    });
}
int vref_hessian_matvec(vref_objective* o, vref_state* s, const double* vt3, double* out3) {
    return guard([&] { store(o->obj->hessian_matvec(s->s, load_vector(o->g, vt3)), out3); });
}
int vref_hessian_data_matvec(vref_objective* o, vref_state* s, const double* vt3, double* out3) {
    return guard([&] { store(o->obj->hessian_data_matvec(s->s, load_vector(o->g, vt3)), out3); });
}
int vref_objective_apply_reg(vref_objective* o, const double* u3, int mode, double* out3) {
    return guard([&] {
        store(o->obj->apply_reg(load_vector(o->g, u3), static_cast<RegOpMode>(mode)), out3);
    });
}
int vref_objective_apply_K(vref_objective* o, const double* u3, double* out3) {
    return guard([&] { store(o->obj->apply_K(load_vector(o->g, u3)), out3); });
}
int vref_pcg_solve(vref_objective* o, vref_state* s, const double* rhs3, double rel_tol,
                   int max_iter, int precond, double* x3, vr_pcg_stats* stats) {
    return guard([&] {
        LinearOp<double> op = [&](const VectorField<double>& u, VectorField<double>& y) {
            y = o->obj->hessian_matvec(s->s, u);
        };
        LinearOp<double> pc = [&](const VectorField<double>& r, VectorField<double>& z) {
            if (precond == VR_PRECOND_SPECTRAL)
                z = o->obj->apply_reg(r, RegOpMode::inverse);
            else
                z = r;
        };
        PcgStats st;
        auto x = pcg_solve<double>(op, load_vector(o->g, rhs3), rel_tol, max_iter, pc, st);
        store(x, x3);
        stats->iterations = st.iterations;
        stats->rel_residual = st.rel_residual;
        stats->converged = st.converged;
        stats->negative_curvature = st.negative_curvature;
        stats->hit_max_iterations = st.hit_max_iterations;
    });
}

// ---- solvers ----------------------------------------------------------------------
namespace {
extern "C++" template <typename T>
class IdentityPreconditionerT final : public KrylovPreconditioner<T> {
public:
    void rebuild(const Objective<T>&, const EvalState<T>&, double) override {}
    void apply(const VectorField<T>& r, VectorField<T>& z) override { z = r; }
};
using IdentityPreconditioner = IdentityPreconditionerT<double>;
} // namespace

// ---- Objective<float> (the reference's fp32 lane) ----
int vref_objective_f32_create(const int* d, const float* mR, const float* mT, const vr_model* m,
                              vref_objective_f32** out) {
    return guard([&] {
        auto o = std::make_unique<vref_objective_f32>();
        o->g = grid_of(d);
        o->m_R = load_scalar_f(o->g, mR);
        o->m_T = load_scalar_f(o->g, mT);
        o->obj = std::make_unique<Objective<float>>(o->m_R, o->m_T, to_model(*m), &o->counters);
        *out = o.release();
    });
}
void vref_objective_f32_destroy(vref_objective_f32* o) { delete o; }
int vref_evaluate_f32(vref_objective_f32* o, const float* v3, vref_state_f32** out) {
    return guard([&] {
        auto s = std::make_unique<vref_state_f32>();
        s->s = o->obj->evaluate(load_vector_f(o->g, v3));
        *out = s.release();
    });
}
void vref_state_f32_destroy(vref_state_f32* s) { delete s; }
int vref_state_f32_scalars(vref_state_f32* s, double* J, double* mis, double* mis_rel) {
    return guard([&] {
        *J = s->s.objective;
        *mis = s->s.mismatch;
        *mis_rel = s->s.mismatch_rel;
    });
}
int vref_compute_gradient_f32(vref_objective_f32* o, vref_state_f32* s, float* g3) {
    return guard([&] {
        o->obj->compute_gradient(s->s);
        if (g3) store_f(s->s.gradient, g3);
    });
}
int vref_hessian_matvec_f32(vref_objective_f32* o, vref_state_f32* s, const float* vt3, float* out3) {
    return guard([&] { store_f(o->obj->hessian_matvec(s->s, load_vector_f(o->g, vt3)), out3); });
}
int vref_objective_f32_counters(vref_objective_f32* o, vr_counters* c) {
    return guard([&] { fill_counters(o->counters, c); });
}
int vref_gauss_newton_solve_f32(const int* d, const float* mR, const float* mT, const float* v0,
                                const vr_model* m, const vr_solver_params* p, int precond,
                                float* v_out, vr_solve_report* rep, vr_iteration_record* recs,
                                int max_recs) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto R = load_scalar_f(g, mR), T = load_scalar_f(g, mT);
        SpectralPreconditioner<float> spec;
        IdentityPreconditionerT<float> ident;
        KrylovPreconditioner<float>& pc =
            precond == VR_PRECOND_SPECTRAL ? static_cast<KrylovPreconditioner<float>&>(spec)
                                           : static_cast<KrylovPreconditioner<float>&>(ident);
        auto res = gauss_newton_solve(R, T, load_vector_f(g, v0), to_model(*m), to_params(*p), pc);
        store_f(res.v, v_out);
        fill_report(res.report, rep, recs, max_recs, 0);
    });
}

int vref_gauss_newton_solve_two_level_f32(const int* d, const float* mR, const float* mT, const float* v0,
                                          const vr_model* m, const vr_solver_params* p,
                                          const vr_twolevel_options* opts, float* v_out,
                                          vr_solve_report* rep, vr_iteration_record* recs, int max_recs) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto R = load_scalar_f(g, mR), T = load_scalar_f(g, mT);
        TwoLevelPreconditioner<float> pre(to_tl(opts));
        auto res = gauss_newton_solve(R, T, load_vector_f(g, v0), to_model(*m), to_params(*p), pre,
                                      pre.coarse_counters());
        store_f(res.v, v_out);
        fill_report(res.report, rep, recs, max_recs, 0);
    });
}

int vref_parameter_continuation_f32(const int* d, const float* mR, const float* mT, const float* v0,
                                    const vr_model* m, const vr_solver_params* p, int precond,
                                    float* v_out, vr_solve_report* reps, int max_levels,
                                    int* n_levels, vr_iteration_record* recs, int max_recs) {
    return guard([&] {
        if (!(m->beta_v <= 1.0)) throw ArgumentError("parameter continuation: target beta_v > 1");
        std::vector<double> levels;
        for (int i = 0;; ++i) {
            double b = std::pow(10.0, -i);
            if (b <= m->beta_v * (1.0 + 1e-9)) break;
            levels.push_back(b);
        }
        levels.push_back(m->beta_v);
        Grid3 g = grid_of(d);
        auto R = load_scalar_f(g, mR), T = load_scalar_f(g, mT);
        auto v = load_vector_f(g, v0);
        SpectralPreconditioner<float> spec;
        IdentityPreconditionerT<float> ident;
        KrylovPreconditioner<float>& pc =
            precond == VR_PRECOND_SPECTRAL ? static_cast<KrylovPreconditioner<float>&>(spec)
                                           : static_cast<KrylovPreconditioner<float>&>(ident);
        int off = 0;
        *n_levels = 0;
        for (std::size_t l = 0; l < levels.size(); ++l) {
            RegModel model = to_model(*m);
            model.beta_v = levels[l];
            auto res = gauss_newton_solve(R, T, v, model, to_params(*p), pc);
            if (static_cast<int>(l) < max_levels) fill_report(res.report, &reps[l], recs, max_recs, off);
            off += static_cast<int>(res.report.iterations.size());
            *n_levels = static_cast<int>(l) + 1;
            v = std::move(res.v);
            if (res.report.stop == StopReason::line_search_failure) break;
        }
        store_f(v, v_out);
    });
}

// gauss_newton_solve + the reference's SolveReport::write_csv (solver.cpp:29-47) into buf
int vref_gauss_newton_solve_csv(const int* d, const double* mR, const double* mT, const double* v0,
                                const vr_model* m, const vr_solver_params* p, char* buf, int len) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto R = load_scalar(g, mR), T = load_scalar(g, mT);
        SpectralPreconditioner<double> spec;
        auto res = gauss_newton_solve(R, T, load_vector(g, v0), to_model(*m), to_params(*p), spec);
        std::ostringstream os;
        const std::vector<std::string> comments{"reference"};
        res.report.write_csv(os, comments);
        const std::string out = os.str();
        if (static_cast<int>(out.size()) + 1 > len) throw ArgumentError("csv buffer too small");
        std::memcpy(buf, out.c_str(), out.size() + 1);
    });
}

int vref_gauss_newton_solve(const int* d, const double* mR, const double* mT, const double* v0,
                            const vr_model* m, const vr_solver_params* p, int precond,
                            double* v_out, vr_solve_report* rep, vr_iteration_record* recs,
                            int max_recs) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto R = load_scalar(g, mR), T = load_scalar(g, mT);
        SpectralPreconditioner<double> spec;
        IdentityPreconditioner ident;
        KrylovPreconditioner<double>& pc =
            precond == VR_PRECOND_SPECTRAL ? static_cast<KrylovPreconditioner<double>&>(spec)
                                           : static_cast<KrylovPreconditioner<double>&>(ident);
        auto res = gauss_newton_solve(R, T, load_vector(g, v0), to_model(*m), to_params(*p), pc);
        store(res.v, v_out);
        fill_report(res.report, rep, recs, max_recs, 0);
    });
}

// Parameter continuation, absent from the reference code: a
// warm-started loop over the reference's own gauss_newton_solve
// (solver.hpp:159-164), levels 1, 1e-1, ... with the last snapped to the target.
int vref_parameter_continuation(const int* d, const double* mR, const double* mT,
                                const double* v0, const vr_model* m, const vr_solver_params* p,
                                int precond, double* v_out, vr_solve_report* reps, int max_levels,
                                int* n_levels, vr_iteration_record* recs, int max_recs) {
    return guard([&] {
        if (!(m->beta_v <= 1.0)) throw ArgumentError("parameter continuation: target beta_v > 1");
        std::vector<double> levels;
        for (int i = 0;; ++i) {
            double b = std::pow(10.0, -i);
            if (b <= m->beta_v * (1.0 + 1e-9)) break;
            levels.push_back(b);
        }
        levels.push_back(m->beta_v);
        Grid3 g = grid_of(d);
        auto R = load_scalar(g, mR), T = load_scalar(g, mT);
        auto v = load_vector(g, v0);
        SpectralPreconditioner<double> spec;
        IdentityPreconditioner ident;
        KrylovPreconditioner<double>& pc =
            precond == VR_PRECOND_SPECTRAL ? static_cast<KrylovPreconditioner<double>&>(spec)
                                           : static_cast<KrylovPreconditioner<double>&>(ident);
        int off = 0;
        *n_levels = 0;
        for (std::size_t l = 0; l < levels.size(); ++l) {
            RegModel model = to_model(*m);
            model.beta_v = levels[l];
            auto res = gauss_newton_solve(R, T, v, model, to_params(*p), pc);
            if (static_cast<int>(l) < max_levels) fill_report(res.report, &reps[l], recs, max_recs, off);
            off += static_cast<int>(res.report.iterations.size());
            *n_levels = static_cast<int>(l) + 1;
            v = std::move(res.v);
            if (res.report.stop == StopReason::line_search_failure) break;
        }
        store(v, v_out);
    });
}

// ---- postprocess (postprocess.hpp:9-56): the reference functions as they are ----
int vref_det_deformation_gradient(const int* d, const double* v, int nt, double* det) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(det_deformation_gradient(load_vector(g, v), nt), det);
    });
}
int vref_deformation_map(const int* d, const double* v, int nt, int absolute, double* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(deformation_map(load_vector(g, v), nt, absolute != 0), out);
    });
}
int vref_det_stats(const int* d, const double* det, const double* fg, double thr, double* out3) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto f = load_scalar(g, det);
        DetStats st;
        if (fg) {
            auto m = load_scalar(g, fg);
            st = det_stats(f, &m, thr);
        } else {
            st = det_stats(f, static_cast<const ScalarField<double>*>(nullptr), thr);
        }
        out3[0] = st.min, out3[1] = st.mean, out3[2] = st.max;
    });
}
// make_ball_labels (synthetic.cpp:36-66): the labelled balls of the reference's postprocess tests
int vref_make_ball_labels(const int* d, int count, double* out) {
    return guard([&] { store(make_ball_labels<double>(grid_of(d), count), out); });
}
int vref_transport_labels(const int* d, const double* labels, const double* v, int nt, double* out) {
    return guard([&] {
        Grid3 g = grid_of(d);
        store(transport_labels(load_scalar(g, labels), load_vector(g, v), nt), out);
    });
}
// per_label / uni: (dice, false_positive_rate, false_negative_rate) triples
int vref_overlap_scores(const int* d, const double* ref, const double* test, const double* mask,
                        int max_labels, int* n_labels, int* codes, double* per_label, double* uni) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto a = load_scalar(g, ref), b = load_scalar(g, test);
        OverlapReport rep;
        if (mask) {
            auto m = load_scalar(g, mask);
            rep = overlap_scores(a, b, &m);
        } else {
            rep = overlap_scores(a, b, static_cast<const ScalarField<double>*>(nullptr));
        }
        int k = 0;
        for (const auto& [code, sc] : rep.per_label) {
            if (k < max_labels) {
                codes[k] = code;
                per_label[3 * k] = sc.dice;
                per_label[3 * k + 1] = sc.false_positive_rate;
                per_label[3 * k + 2] = sc.false_negative_rate;
            }
            ++k;
        }
        *n_labels = k;
        uni[0] = rep.union_scores.dice;
        uni[1] = rep.union_scores.false_positive_rate;
        uni[2] = rep.union_scores.false_negative_rate;
    });
}

// ---- continuation, absent from the reference code: restated as
// loops over the reference's own gauss_newton_solve, spectral_resample,
// gaussian_smooth, det_deformation_gradient and det_stats ----
namespace {
struct PcHolder {
    SpectralPreconditioner<double> spec;
    IdentityPreconditioner ident;
    KrylovPreconditioner<double>& get(int precond) {
        return precond == VR_PRECOND_SPECTRAL ? static_cast<KrylovPreconditioner<double>&>(spec)
                                              : static_cast<KrylovPreconditioner<double>&>(ident);
    }
};
}  // namespace

int vref_grid_continuation(const int* d, const double* mR, const double* mT, const double* v0,
                           const vr_model* m, const vr_solver_params* p, int precond, int n_grid,
                           double* v_out, vr_solve_report* reps, int max_levels, int* n_levels,
                           vr_iteration_record* recs, int max_recs) {
    return guard([&] {
        if (n_grid < 1) throw ArgumentError("grid continuation: at least one level");
        for (int a = 0; a < 3; ++a)
            if ((d[a] >> (n_grid - 1)) < 16 || d[a] % (1 << (n_grid - 1)) != 0)
                throw ArgumentError("grid continuation: the coarsest level must keep >= 16 points per axis");
        Grid3 gf = grid_of(d);
        auto R = load_scalar(gf, mR), T = load_scalar(gf, mT);
        auto vf = load_vector(gf, v0);
        PcHolder pc;
        const int sh0 = n_grid - 1;
        VectorField<double> v =
            n_grid == 1 ? vf : spectral_resample(vf, Grid3(d[0] >> sh0, d[1] >> sh0, d[2] >> sh0));
        int off = 0;
        *n_levels = 0;
        for (int l = 0; l < n_grid; ++l) {
            const int s = n_grid - 1 - l;
            auto res = [&] {
                if (s == 0) return gauss_newton_solve(R, T, v, to_model(*m), to_params(*p), pc.get(precond));
                Grid3 gl(d[0] >> s, d[1] >> s, d[2] >> s);
                auto Rl = gaussian_smooth(spectral_resample(R, gl), {1.0, 1.0, 1.0});
                auto Tl = gaussian_smooth(spectral_resample(T, gl), {1.0, 1.0, 1.0});
                return gauss_newton_solve(Rl, Tl, v, to_model(*m), to_params(*p), pc.get(precond));
            }();
            if (l < max_levels) fill_report(res.report, &reps[l], recs, max_recs, off);
            off += static_cast<int>(res.report.iterations.size());
            *n_levels = l + 1;
            if (s == 0) {
                v = std::move(res.v);
                break;
            }
            if (res.report.stop == StopReason::line_search_failure) {
                v = spectral_resample(res.v, gf);
                break;
            }
            const int s1 = s - 1;
            v = spectral_resample(res.v, Grid3(d[0] >> s1, d[1] >> s1, d[2] >> s1));
        }
        store(v, v_out);
    });
}

int vref_scale_continuation(const int* d, const double* mR, const double* mT, const double* v0,
                            const vr_model* m, const vr_solver_params* p, int precond,
                            const double* sigmas, int n, double* v_out, vr_solve_report* reps,
                            int max_levels, int* n_levels, vr_iteration_record* recs, int max_recs) {
    return guard([&] {
        if (n < 1) throw ArgumentError("scale continuation: at least one level");
        for (int l = 0; l < n; ++l) {
            if (!(sigmas[l] >= 0.0)) throw ArgumentError("scale continuation: sigmas must be >= 0");
            if (l > 0 && !(sigmas[l] < sigmas[l - 1]))
                throw ArgumentError("scale continuation: sigmas must be strictly decreasing");
        }
        Grid3 g = grid_of(d);
        auto R = load_scalar(g, mR), T = load_scalar(g, mT);
        auto v = load_vector(g, v0);
        PcHolder pc;
        int off = 0;
        *n_levels = 0;
        for (int l = 0; l < n; ++l) {
            const double sg = sigmas[l];
            auto res = sg > 0.0 ? gauss_newton_solve(gaussian_smooth(R, {sg, sg, sg}),
                                                     gaussian_smooth(T, {sg, sg, sg}), v,
                                                     to_model(*m), to_params(*p), pc.get(precond))
                                : gauss_newton_solve(R, T, v, to_model(*m), to_params(*p), pc.get(precond));
            if (l < max_levels) fill_report(res.report, &reps[l], recs, max_recs, off);
            off += static_cast<int>(res.report.iterations.size());
            *n_levels = l + 1;
            v = std::move(res.v);
            if (res.report.stop == StopReason::line_search_failure) break;
        }
        store(v, v_out);
    });
}

// trials: (beta, feasible, det min, det mean, det max) x n; reps: their solve reports
int vref_beta_search(const int* d, const double* mR, const double* mT, const double* v0,
                     const vr_model* m, const vr_solver_params* p, int precond,
                     const vr_beta_search_params* bp, double* beta_out, double* v_out,
                     double* trials, vr_solve_report* reps, int max_trials, int* n_trials) {
    return guard([&] {
        if (!(bp->eps_J > 0.0 && bp->eps_J < 1.0)) throw ArgumentError("beta search: eps_J must be in (0, 1)");
        if (!(bp->beta_lo > 0.0 && bp->beta_lo < bp->beta_hi))
            throw ArgumentError("beta search: need 0 < beta_lo < beta_hi");
        if (bp->max_bisections < 0 || !(bp->min_width_decades > 0.0))
            throw ArgumentError("beta search: max_bisections >= 0 and min_width_decades > 0");
        Grid3 g = grid_of(d);
        auto R = load_scalar(g, mR), T = load_scalar(g, mT);
        auto vprev = load_vector(g, v0);
        VectorField<double> vbest(g, 0.0);
        PcHolder pc;
        int k = 0;
        double best = 0.0;
        auto trial = [&](double beta) {
            RegModel model = to_model(*m);
            model.beta_v = beta;
            auto res = gauss_newton_solve(R, T, vprev, model, to_params(*p), pc.get(precond));
            auto det = det_deformation_gradient(res.v, m->nt);
            DetStats st = det_stats(det, static_cast<const ScalarField<double>*>(nullptr), 0.0);
            const bool feas = st.min >= bp->eps_J && st.max <= 1.0 / bp->eps_J;
            if (k < max_trials) {
                double* t = trials + 5 * k;
                t[0] = beta, t[1] = feas ? 1.0 : 0.0, t[2] = st.min, t[3] = st.mean, t[4] = st.max;
                fill_report(res.report, &reps[k], nullptr, 0, 0);
            }
            ++k;
            vprev = res.v;
            if (feas) best = beta, vbest = std::move(res.v);
            return feas;
        };
        bool found = trial(bp->beta_hi);
        if (found && !trial(bp->beta_lo)) {
            double lo = std::log10(bp->beta_lo), hi = std::log10(bp->beta_hi);
            for (int it = 0; it < bp->max_bisections && hi - lo >= bp->min_width_decades; ++it) {
                const double mid = 0.5 * (lo + hi);
                if (trial(std::pow(10.0, mid)))
                    hi = mid;
                else
                    lo = mid;
            }
        }
        *n_trials = k;
        *beta_out = best;
        if (!found) throw NumericError("beta search: no feasible beta_v in the bracket");
        store(vbest, v_out);
    });
}

// ---- two-level preconditioner / grid transfer (precond.hpp, spectral.hpp:131-153) ----
int vref_spectral_resample(const int* ds, const double* in, int ncomp, const int* dd, double* out) {
    return guard([&] {
        Grid3 gs = grid_of(ds), gd = grid_of(dd);
        if (ncomp == 3)
            store(spectral_resample(load_vector(gs, in), gd), out);
        else
            store(spectral_resample(load_scalar(gs, in), gd), out);
    });
}
int vref_frequency_filter(const int* d, const double* in, int ncomp, int band, const int* cutoff,
                          double* out) {
    return guard([&] {
        Grid3 g = grid_of(d), c = grid_of(cutoff);
        const FreqBand b = band == 0 ? FreqBand::low : FreqBand::high;
        if (ncomp == 3)
            store(frequency_filter(load_vector(g, in), b, c), out);
        else
            store(frequency_filter(load_scalar(g, in), b, c), out);
    });
}
int vref_split_matvec(vref_objective* o, vref_state* s, const double* w3, double* out3) {
    return guard([&] { store(o->obj->split_matvec(s->s, load_vector(o->g, w3)), out3); });
}
int vref_twolevel_create(const vr_twolevel_options* opts, vref_twolevel** out) {
    return guard([&] { *out = new vref_twolevel(to_tl(opts)); });
}
void vref_twolevel_destroy(vref_twolevel* t) { delete t; }
int vref_twolevel_rebuild(vref_twolevel* t, vref_objective* o, vref_state* s, double eps_H) {
    return guard([&] {
        t->fine = o->g;
        t->pre.rebuild(*o->obj, s->s, eps_H);
    });
}
int vref_twolevel_apply(vref_twolevel* t, const double* r3, double* z3) {
    return guard([&] {
        VectorField<double> z;
        t->pre.apply(load_vector(t->fine, r3), z);
        store(z, z3);
    });
}
int vref_twolevel_coarse_matvec(vref_twolevel* t, const double* u3, double* out3) {
    return guard([&] {
        auto& c = t->pre.context();
        store(c.coarse_matvec(load_vector(c.coarse_grid(), u3)), out3);
    });
}
int vref_twolevel_info(vref_twolevel* t, int* dims, int* lanczos_runs, int* inner_diverged,
                       double* bounds, vr_counters* coarse) {
    return guard([&] {
        auto& c = t->pre.context();
        for (int a = 0; a < 3; ++a) dims[a] = c.ready() ? c.coarse_grid().dims[a] : 0;
        *lanczos_runs = c.lanczos_runs();
        *inner_diverged = c.inner_diverged();
        bounds[0] = c.eig_bounds().first;
        bounds[1] = c.eig_bounds().second;
        fill_counters(*t->pre.coarse_counters(), coarse);
    });
}
int vref_gauss_newton_solve_two_level(const int* d, const double* mR, const double* mT,
                                      const double* v0, const vr_model* m,
                                      const vr_solver_params* p, const vr_twolevel_options* opts,
                                      double* v_out, vr_solve_report* rep,
                                      vr_iteration_record* recs, int max_recs) {
    return guard([&] {
        Grid3 g = grid_of(d);
        auto R = load_scalar(g, mR), T = load_scalar(g, mT);
        TwoLevelPreconditioner<double> pre(to_tl(opts));
        auto res = gauss_newton_solve(R, T, load_vector(g, v0), to_model(*m), to_params(*p), pre,
                                      pre.coarse_counters());
        store(res.v, v_out);
        fill_report(res.report, rep, recs, max_recs, 0);
    });
}

int vref_generate_synthetic(const int* d, int nt, double amplitude, double* mR, double* mT,
                            double* vstar) {
    return guard([&] {
        auto p = generate_synthetic<double>(grid_of(d), nt, amplitude);
        store(p.m_R, mR);
        store(p.m_T, mT);
        store(p.v_star, vstar);
    });
}

// ---- reference test-suite generators (proj/tests/test_support.hpp) -------------
int vref_random_smooth_scalar(const int* d, int max_mode, unsigned long long seed, double amp,
                              double* out) {
    return guard([&] {
        store(testing::random_smooth_scalar<double>(grid_of(d), max_mode, seed, amp), out);
    });
}
int vref_random_smooth_vector(const int* d, int max_mode, unsigned long long seed, double amp,
                              double* out3) {
    return guard([&] {
        store(testing::random_smooth_vector<double>(grid_of(d), max_mode, seed, amp), out3);
    });
}
int vref_random_rough_scalar(const int* d, unsigned long long seed, double* out) {
    return guard([&] { store(testing::random_rough_scalar<double>(grid_of(d), seed), out); });
}

} // extern "C"
