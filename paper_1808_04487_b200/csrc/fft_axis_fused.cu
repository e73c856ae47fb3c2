// fft_axis_fused.cu -- the fused strided passes: x1 forward -> spectral multiplier -> inverse
// (MODE 1: any multiplier; MODE 3: the regularisation symbol applied in the forward FFT's last
// stores) and the one-axis derivative of a real field (MODE 2). Kernel: fft_axis.cuh.
#include "fft_axis.cuh"

namespace vr {

void pass_x1_mult(vr_ctx* ctx, const double* src, double* dst, const MultParams& mult) {
    const GridDims& g = ctx->g;
    const auto* s = reinterpret_cast<const double2*>(src);
    auto* d = reinterpret_cast<double2*>(dst);
    const long long inner = (long long)g.n2s * g.nh;
    if (mult.kind == Mult::reg)
        launch_axis<-1, 3>(ctx, g.n1, s, d, inner, 1, 0, ctx->fft->tw1, to_dev(mult));
    else
        launch_axis<-1, 1>(ctx, g.n1, s, d, inner, 1, 0, ctx->fft->tw1, to_dev(mult));
}

// d f / d x_axis of a real field on one GPU for the strided axes: forward, i k / n, inverse in
// one pass over f viewed as complex pairs (MODE 2)
void deriv_axis_strided(vr_ctx* ctx, int axis, const double* f, double* out) {
    const GridDims& g = ctx->g;
    const auto* s = reinterpret_cast<const double2*>(f);
    auto* d = reinterpret_cast<double2*>(out);
    const long long h3 = g.n3 / 2;
    MultDev m{};
    if (axis == 0) {
        m.beta = 1.0 / g.n1;
        launch_axis<-1, 2>(ctx, g.n1, s, d, static_cast<long long>(g.n2) * h3, 1, 0, ctx->fft->tw1, m);
    } else {
        m.beta = 1.0 / g.n2;
        launch_axis<-1, 2>(ctx, g.n2, s, d, h3, g.L, static_cast<long long>(g.n2) * h3, ctx->fft->tw2, m);
    }
}

}  // namespace vr
