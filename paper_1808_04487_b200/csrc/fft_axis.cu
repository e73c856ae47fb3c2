// fft_axis.cu -- the strided (x1 / x2) passes of the fp64 3D FFT, plain transforms: TMA-fed
// persistent column tiles, Stockham radix-16 stages, and the x1-slab variants whose stores /
// loads carry the all-to-all pack / unpack (kernel: fft_axis.cuh; fused passes: fft_axis_fused.cu).
#include "fft_axis.cuh"

namespace vr {

void pass_x2(vr_ctx* ctx, double* spec, int dir) {
    const GridDims& g = ctx->g;
    auto* s = reinterpret_cast<double2*>(spec);
    MultDev none{};
    if (dir < 0)
        launch_axis<-1, 0>(ctx, g.n2, s, s, g.nh, g.L, (long long)g.n2 * g.nh, ctx->fft->tw2, none);
    else
        launch_axis<+1, 0>(ctx, g.n2, s, s, g.nh, g.L, (long long)g.n2 * g.nh, ctx->fft->tw2, none);
}
namespace {
int ilog2(int v) {
    int s = 0;
    while ((1 << s) < v) ++s;
    return s;
}
}  // namespace
// x1 slabs: forward x2 pass of the slab spectrum [L][n2][nh], stored straight into the
// all-to-all send layout (block q = [L][n2s][nh], the k2 rows of rank q)
void pass_x2_to_blocks(vr_ctx* ctx, const double* slab, double* send) {
    const GridDims& g = ctx->g;
    const auto* s = reinterpret_cast<const double2*>(slab);
    auto* d = reinterpret_cast<double2*>(send);
    MultDev none{};
    const long long blk = static_cast<long long>(g.L) * g.n2s * g.nh;
    const int sh = ilog2(g.n2s);
    switch (g.n2) {
#define VR_CASE(NN)                                                                                  \
    case NN:                                                                                         \
        launch_axis_t<NN, -1, 0, true>(ctx, s, d, g.nh, g.L, (long long)g.n2 * g.nh, ctx->fft->tw2, none, \
                                       RowGroups{}, sh, blk);                                       \
        break;
        VR_CASE(4)
        VR_CASE(8)
        VR_CASE(16)
        VR_CASE(32)
        VR_CASE(64)
        VR_CASE(128)
        VR_CASE(256)
        VR_CASE(512)
        VR_CASE(1024)
#undef VR_CASE
        default: throw_dimension("fft: unsupported axis length " + std::to_string(g.n2));
    }
}
// x1 slabs: inverse x2 pass reading the all-to-all receive layout (block q = [L][n2s][nh] from
// rank q) through a tensor map whose row groups are the peer blocks, into the slab [L][n2][nh]
void pass_x2_from_blocks(vr_ctx* ctx, const double* recv, double* slab) {
    const GridDims& g = ctx->g;
    const auto* s = reinterpret_cast<const double2*>(recv);
    auto* d = reinterpret_cast<double2*>(slab);
    MultDev none{};
    const long long blk = static_cast<long long>(g.L) * g.n2s * g.nh;
    const RowGroups rg{g.n2s, blk, static_cast<long long>(g.n2s) * g.nh};
    switch (g.n2) {
#define VR_CASE(NN)                                                                                   \
    case NN:                                                                                          \
        launch_axis_t<NN, +1, 0>(ctx, s, d, g.nh, g.L, (long long)g.n2 * g.nh, ctx->fft->tw2, none, rg);  \
        break;
        VR_CASE(4)
        VR_CASE(8)
        VR_CASE(16)
        VR_CASE(32)
        VR_CASE(64)
        VR_CASE(128)
        VR_CASE(256)
        VR_CASE(512)
        VR_CASE(1024)
#undef VR_CASE
        default: throw_dimension("fft: unsupported axis length " + std::to_string(g.n2));
    }
}
void pass_x1(vr_ctx* ctx, const double* src, double* dst, int dir, const MultParams* mult) {
    if (mult) {
        pass_x1_mult(ctx, src, dst, *mult);  // fft_axis_fused.cu
        return;
    }
    const GridDims& g = ctx->g;
    const auto* s = reinterpret_cast<const double2*>(src);
    auto* d = reinterpret_cast<double2*>(dst);
    const long long inner = (long long)g.n2s * g.nh;
    MultDev none{};
    if (dir < 0)
        launch_axis<-1, 0>(ctx, g.n1, s, d, inner, 1, 0, ctx->fft->tw1, none);
    else
        launch_axis<+1, 0>(ctx, g.n1, s, d, inner, 1, 0, ctx->fft->tw1, none);
}

}  // namespace vr
