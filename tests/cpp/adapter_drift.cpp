// tests/cpp/adapter_drift.cpp -- compile-time drift check of the C++ drop-in against the
// reference headers (compiled with -fsyntax-only by tests/test_adapter_cpp.py when
// /root/reference is present). If the reference renames a RegModel / RegNorm /
// SolverParams field or renumbers an enum, this stops compiling.
#define VELOREG_GPU_REFERENCE_ERRORS
#include "veloreg/objective.hpp"
#include "veloreg/solver.hpp"
#include "veloreg_gpu.hpp"

namespace vg = veloreg_gpu;

static_assert(static_cast<int>(veloreg::RegKind::h1_seminorm) == VR_REG_H1);
static_assert(static_cast<int>(veloreg::RegKind::h2_seminorm) == VR_REG_H2);
static_assert(static_cast<int>(veloreg::RegKind::h3_seminorm) == VR_REG_H3);
static_assert(static_cast<int>(veloreg::RegKind::helmholtz) == VR_REG_HELMHOLTZ);
static_assert(static_cast<int>(veloreg::RegOpMode::inverse_sqrt) == VR_REGOP_INVERSE_SQRT);
static_assert(static_cast<int>(veloreg::ProjectionKind::near_incompressible) == VR_PROJ_NEAR_INCOMPRESSIBLE);
static_assert(static_cast<int>(veloreg::StopReason::line_search_failure) ==
              static_cast<int>(vg::StopReason::line_search_failure));
static_assert(static_cast<int>(veloreg::ErrorCategory::numerics) == VR_ERR_NUMERICS);
static_assert(static_cast<int>(veloreg::ErrorCategory::logic) == VR_ERR_LOGIC);

// field-by-field conversion from the reference's structs: breaks on any rename
vg::RegModel from_reference(const veloreg::RegModel& m) {
    vg::RegModel o;
    o.norm.kind = static_cast<vg::RegKind>(static_cast<int>(m.norm.kind));
    o.norm.gamma = m.norm.gamma;
    o.norm.helmholtz_squared = m.norm.helmholtz_squared;
    o.norm.div_penalty = m.norm.div_penalty;
    o.norm.beta_w = m.norm.beta_w;
    o.projection = static_cast<vg::ProjectionKind>(static_cast<int>(m.projection));
    o.beta_v = m.beta_v;
    o.nt = m.nt;
    o.gauss_newton = m.gauss_newton;
    return o;
}
vg::SolverParams from_reference(const veloreg::SolverParams& p) {
    vg::SolverParams o;
    o.eps_opt = p.eps_opt;
    o.abs_grad_tol = p.abs_grad_tol;
    o.max_newton = p.max_newton;
    o.max_krylov = p.max_krylov;
    o.armijo_c1 = p.armijo_c1;
    o.armijo_backtrack = p.armijo_backtrack;
    o.armijo_max_trials = p.armijo_max_trials;
    o.squared_norm_stop = p.squared_norm_stop;
    return o;
}
// the report rows carry the reference's IterationRecord fields
static_assert(sizeof(veloreg::IterationRecord{}.k) == sizeof(vg::IterationRecord{}.k));
// the adapter's exceptions ARE the reference's with VELOREG_GPU_REFERENCE_ERRORS
static_assert(std::is_same_v<vg::NumericError, veloreg::NumericError>);

// same method set as Objective<double>: every call a reference driver makes on it
template <class Obj, class State, class Vec>
void uses(const Obj& obj, State& s, const Vec& v) {
    (void)obj.evaluate(v);
    obj.compute_gradient(s);
    (void)obj.hessian_matvec(s, v);
    (void)obj.hessian_data_matvec(s, v);
    (void)obj.split_matvec(s, v);
    (void)obj.apply_reg(v, vg::RegOpMode::apply);
    (void)obj.apply_K(v);
    (void)obj.model();
    (void)obj.initial_mismatch();
    (void)obj.counters();
}
template void uses<vg::Objective, vg::EvalState, vg::DeviceField>(const vg::Objective&, vg::EvalState&,
                                                                 const vg::DeviceField&);
// and the reference's own Objective<double> has that set too (both sides of the contract)
template <class T>
void reference_uses(const veloreg::Objective<T>& obj, veloreg::EvalState<T>& s, const veloreg::VectorField<T>& v) {
    (void)obj.evaluate(v);
    obj.compute_gradient(s);
    (void)obj.hessian_matvec(s, v);
    (void)obj.hessian_data_matvec(s, v);
    (void)obj.split_matvec(s, v);
    (void)obj.apply_reg(v, veloreg::RegOpMode::apply);
    (void)obj.apply_K(v);
    (void)obj.model();
    (void)obj.initial_mismatch();
    (void)obj.counters();
}
template void reference_uses<double>(const veloreg::Objective<double>&, veloreg::EvalState<double>&,
                                     const veloreg::VectorField<double>&);
