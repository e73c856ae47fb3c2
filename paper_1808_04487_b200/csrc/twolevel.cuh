// twolevel.cuh -- spectral grid transfer, split matvec, Lanczos / Chebyshev and
// the two-level preconditioner (twolevel.cu; proj/src/precond.cpp, spectral.cpp:228-385).
#pragma once

#include <utility>

#include "objective.cuh"

namespace vr {

// spectral_resample of one scalar field between grids of one device (src -> dst)
void resample_scalar(vr_ctx* src, const double* in, vr_ctx* dst, double* out);
// frequency_filter: band 0 = low (F_L), 1 = high (F_H = id - F_L) w.r.t. the cutoff grid
void frequency_filter(vr_ctx* ctx, const double* in, int band, const int cutoff[3], double* out);
// Objective::split_matvec (objective.cpp:158-176)
void split_matvec(vr_objective* o, const vr_state* s, const double* w3, double* out3);
std::pair<double, double> lanczos_bounds(vr_ctx* ctx, const DevOp& op, int iterations,
                                         unsigned long long seed);
void cheb_solve(vr_ctx* ctx, const DevOp& op, const double* rhs, int k,
                std::pair<double, double> bounds, double* x);

// TwoLevelContext + TwoLevelPreconditioner (precond.hpp:55-110)
struct TwoLevel {
    explicit TwoLevel(const vr_twolevel_options& o);
    ~TwoLevel();
    void rebuild(vr_objective* fine_obj, const vr_state* fine_state, double eps_H);
    void apply(vr_ctx* fine, const double* s, double* u);
    void coarse_matvec(const double* u, double* out);
    vr_counters counters() const;  // cumulative coarse counters (coarse_counters_)

    vr_twolevel_options opts;
    vr_ctx* cctx = nullptr;        // n/2 sibling of the fine context (shares its stream)
    double *mRc = nullptr, *mTc = nullptr;
    vr_objective* cobj = nullptr;
    vr_state* cstate = nullptr;
    double eps_M = 0.1;
    std::pair<double, double> bounds{0.0, 0.0};
    int lanczos_runs = 0;
    bool inner_diverged = false;

private:
    vr_counters done{};
    void release();
    void destroy_ctx();
    void add_counters(const vr_counters& c);
    void resample_vec(vr_ctx* src, const double* in, vr_ctx* dst, double* out);
};

}  // namespace vr
