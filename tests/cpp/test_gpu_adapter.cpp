// tests/cpp/test_gpu_adapter.cpp -- the reference's own objective / solver property tests
// re-run on the GPU through the compiled C++ drop-in (include/veloreg_gpu.hpp).
//
// Cases follow proj/tests/test_objective.cpp:160-215 (PDE-solve counting, pure-
// regularisation limit, zero direction, Gauss-Newton symmetry / PSD) and
// proj/tests/test_solver.cpp:138-178 (GN synthetic solve: descent, counters, unit steps,
// CSV), plus the error contract (errors.hpp:9-67) and the reference-shaped host PCG over
// a LinearOp. Inputs come from the reference's own test generators (test_support.hpp)
// through the oracle harness (oracle/_ref/libveloreg_ref.so, test infrastructure only).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <cmath>
#include <limits>
#include <sstream>

#include "doctest.h"
#include "veloreg_gpu.hpp"

extern "C" {  // oracle harness (ref_capi.cpp): test_support.hpp / synthetic.cpp generators
int vref_random_smooth_scalar(const int* d, int max_mode, unsigned long long seed, double amp, double* out);
int vref_random_smooth_vector(const int* d, int max_mode, unsigned long long seed, double amp, double* out3);
int vref_generate_synthetic(const int* d, int nt, double amplitude, double* mR, double* mT, double* vstar);
}

using namespace veloreg_gpu;

namespace {

constexpr int kN = 16;
const int kDims[3] = {kN, kN, kN};
constexpr long long kPts = static_cast<long long>(kN) * kN * kN;

Context& ctx() {
    static Context c(kN);
    return c;
}

std::vector<double> smooth_vector(int max_mode, unsigned long long seed, double amp) {
    std::vector<double> v(3 * kPts);
    REQUIRE(vref_random_smooth_vector(kDims, max_mode, seed, amp, v.data()) == 0);
    return v;
}

// test_objective.cpp:13-33
RegModel h2_model(int nt = 4, double beta_v = 1e-3) {
    RegModel m;
    m.norm.kind = RegKind::h2_seminorm;
    m.beta_v = beta_v;
    m.nt = nt;
    return m;
}
std::pair<DeviceField, DeviceField> smooth_image_pair(int max_mode, unsigned long long seed) {
    std::vector<double> r1(kPts), r2(kPts);
    REQUIRE(vref_random_smooth_scalar(kDims, max_mode, seed, 0.3, r1.data()) == 0);
    REQUIRE(vref_random_smooth_scalar(kDims, max_mode, seed + 1, 0.3, r2.data()) == 0);
    for (long long i = 0; i < kPts; ++i) r1[i] += 0.5, r2[i] += 0.5;
    return {DeviceField(ctx(), r1, 1), DeviceField(ctx(), r2, 1)};
}

double max_abs_diff(const DeviceField& a, const DeviceField& b) {
    auto x = a.download(), y = b.download();
    double m = 0;
    for (size_t i = 0; i < x.size(); ++i) m = std::max(m, std::fabs(x[i] - y[i]));
    return m;
}

}  // namespace

TEST_CASE("hessian_matvec: zero direction, pure-regularization limit, PDE-solve counting") {
    SolveCounters counters;
    DeviceField mconst(ctx(), std::vector<double>(kPts, 0.5), 1);
    RegModel model = h2_model(4, 2.5e-3);
    Objective obj(ctx(), mconst, mconst, model, &counters);
    DeviceField zero(ctx(), 3);
    auto s = obj.evaluate(zero);
    obj.compute_gradient(s);

    long before = counters.pde_solves;
    CHECK(before == 2);  // state + adjoint

    DeviceField vt(ctx(), smooth_vector(2, 90, 1.0), 3);
    auto Hvt = obj.hessian_matvec(s, vt);
    CHECK(counters.pde_solves - before == 2);  // incremental state + adjoint

    auto reg = apply_reg_operator(ctx(), vt, model.norm, RegOpMode::apply, model.beta_v);
    CHECK(max_abs_diff(Hvt, reg) < 1e-14);

    DeviceField zdir(ctx(), 3);
    auto hz = obj.hessian_matvec(s, zdir);
    CHECK(max_abs(hz) == 0.0);
}

TEST_CASE("hessian_matvec: Gauss-Newton symmetry and positive semidefiniteness") {
    auto [mR, mT] = smooth_image_pair(2, 91);
    Objective obj(ctx(), mR, mT, h2_model(4));
    DeviceField zero(ctx(), 3);
    auto s0 = obj.evaluate(zero);
    obj.compute_gradient(s0);
    for (int probe = 0; probe < 5; ++probe) {
        DeviceField u(ctx(), smooth_vector(2, 100 + 2 * probe, 1.0), 3);
        DeviceField w(ctx(), smooth_vector(2, 101 + 2 * probe, 1.0), 3);
        auto Hu = obj.hessian_matvec(s0, u);
        auto Hw = obj.hessian_matvec(s0, w);
        double a = inner_product(Hu, w), b = inner_product(u, Hw);
        CHECK(std::abs(a - b) / std::max(std::abs(a), std::abs(b)) < 1e-6);
        double quad = inner_product(Hu, u);
        CHECK(quad >= -1e-10 * std::max(1.0, std::abs(quad)));
    }
    DeviceField v(ctx(), smooth_vector(2, 120, 0.05), 3);
    auto sv = obj.evaluate(v);
    obj.compute_gradient(sv);
    DeviceField u(ctx(), smooth_vector(2, 121, 1.0), 3);
    DeviceField w(ctx(), smooth_vector(2, 122, 1.0), 3);
    double a = inner_product(obj.hessian_matvec(sv, u), w);
    double b = inner_product(u, obj.hessian_matvec(sv, w));
    CHECK(std::abs(a - b) / std::max(std::abs(a), std::abs(b)) < 5e-3);
}

TEST_CASE("error contract: the reference's exception classes") {
    auto [mR, mT] = smooth_image_pair(2, 91);
    Objective obj(ctx(), mR, mT, h2_model(4));
    DeviceField zero(ctx(), 3);
    auto s = obj.evaluate(zero);
    DeviceField vt(ctx(), smooth_vector(2, 90, 1.0), 3);
    CHECK_THROWS_AS(obj.hessian_matvec(s, vt), LogicError);  // before the gradient
    obj.compute_gradient(s);
    auto bad = smooth_vector(2, 90, 1.0);
    bad[7] = std::numeric_limits<double>::quiet_NaN();
    DeviceField nan_dir(ctx(), bad, 3);
    CHECK_THROWS_AS(obj.hessian_matvec(s, nan_dir), NumericError);
    CHECK_THROWS_AS(obj.evaluate(nan_dir), NumericError);
    DeviceField scalar(ctx(), 1);
    CHECK_THROWS_AS(obj.hessian_matvec(s, scalar), DimensionError);
    RegModel m = h2_model(4);
    m.beta_v = -1.0;
    CHECK_THROWS_AS(Objective(ctx(), mR, mT, m), ArgumentError);
    CHECK_THROWS_AS(Context(2, 16, 16), DimensionError);
}

TEST_CASE("pcg_solve over a LinearOp: the reference's host PCG against the library's") {
    auto [mR, mT] = smooth_image_pair(2, 91);
    RegModel model = h2_model(4, 1e-2);
    Objective obj(ctx(), mR, mT, model);
    DeviceField v(ctx(), smooth_vector(2, 120, 0.05), 3);
    auto s = obj.evaluate(v);
    obj.compute_gradient(s);
    DeviceField rhs = s.gradient(ctx());
    scale(rhs, -1.0);
    SpectralPreconditioner pc;
    pc.rebuild(obj, s, 0.1);
    LinearOp H = [&](const DeviceField& x, DeviceField& y) { y = obj.hessian_matvec(s, x); };
    LinearOp P = [&](const DeviceField& r, DeviceField& z) { pc.apply(r, z); };
    PcgStats st;
    auto x = pcg_solve(H, rhs, 1e-6, 100, P, st);
    CHECK(st.converged);
    CHECK(st.rel_residual < 1e-6);
    // the library's device PCG (vr_pcg_solve) takes the same iterations to the same answer
    DeviceField x2(ctx(), 3);
    vr_pcg_stats st2{};
    check(vr_pcg_solve(obj.get(), s.get(), rhs.data(), 1e-6, 100, VR_PRECOND_SPECTRAL, x2.data(), &st2));
    CHECK(std::abs(st.iterations - st2.iterations) <= 1);
    DeviceField d = x.clone();
    add_scaled(d, -1.0, x2);
    CHECK(norm_l2(d) <= 1e-5 * norm_l2(x));
    // the residual really is small: |H x - rhs| / |rhs|
    DeviceField hx = obj.hessian_matvec(s, x);
    add_scaled(hx, -1.0, rhs);
    CHECK(norm_l2(hx) <= 2e-6 * norm_l2(rhs));
}

TEST_CASE("gauss_newton_solve: synthetic problem, descent and counters") {
    std::vector<double> r(kPts), t(kPts), vs(3 * kPts);
    REQUIRE(vref_generate_synthetic(kDims, 4, 1.0, r.data(), t.data(), vs.data()) == 0);
    DeviceField m_R(ctx(), r, 1), m_T(ctx(), t, 1), v0(ctx(), 3);
    RegModel model;
    model.norm.kind = RegKind::h1_seminorm;
    model.norm.div_penalty = true;
    model.norm.beta_w = 1e-4;
    model.projection = ProjectionKind::near_incompressible;
    model.beta_v = 1e-3;
    model.nt = 4;
    SolverParams params;
    params.eps_opt = 1e-2;
    SpectralPreconditioner precond;
    auto res = gauss_newton_solve(ctx(), m_R, m_T, v0, model, params, precond);

    CHECK(res.report.success);
    CHECK(res.report.stop == StopReason::converged_rel);
    CHECK(res.report.final_mismatch_rel < 0.2);
    CHECK(res.report.final_grad_rel * res.report.final_grad_rel <= params.eps_opt);
    for (size_t i = 1; i < res.report.iterations.size(); ++i)
        CHECK(res.report.iterations[i].objective < res.report.iterations[i - 1].objective);
    const auto& f = res.report.fine;
    CHECK(f.pde_solves == f.objective_evals + f.gradient_evals + 2 * f.hessian_matvecs);
    CHECK(res.report.coarse.pde_solves == 0);
    int unit = 0, total = 0;
    for (const auto& row : res.report.iterations) {
        if (row.k == 0) continue;
        ++total;
        if (row.step_length == 1.0) ++unit;
    }
    CHECK(unit * 2 >= total);

    // SolveReport::write_csv (solver.cpp:29-47): the reference's header and one row per record
    std::ostringstream os;
    res.report.write_csv(os, {"gpu"});
    std::istringstream is(os.str());
    std::string line;
    std::getline(is, line);
    CHECK(line == "# gpu");
    std::getline(is, line);
    CHECK(line == SolveReport::csv_header());
    int rows = 0;
    while (std::getline(is, line)) ++rows;
    CHECK(rows == static_cast<int>(res.report.iterations.size()));
    CHECK(rows == res.report.outer_iterations + 1);
}

TEST_CASE("gauss_newton_solve: two-level preconditioner on the split system") {
    std::vector<double> r(kPts), t(kPts), vs(3 * kPts);
    REQUIRE(vref_generate_synthetic(kDims, 4, 1.0, r.data(), t.data(), vs.data()) == 0);
    DeviceField m_R(ctx(), r, 1), m_T(ctx(), t, 1), v0(ctx(), 3);
    SolverParams params;
    params.eps_opt = 1e-2;
    TwoLevelPreconditioner tl;
    auto res = gauss_newton_solve(ctx(), m_R, m_T, v0, h2_model(4, 1e-2), params, tl);
    CHECK(res.report.success);
    CHECK(res.report.coarse.hessian_matvecs > 0);
}
