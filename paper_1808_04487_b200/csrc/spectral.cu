// spectral.cu -- spectral operators (proj/src/spectral.cpp:84-222, fft.cpp:66-115)
// composed from the FFT pass primitives of fft.cu, on one GPU or on x1 slabs.
//
// One GPU:  r2c(x3) -> x2 -> x1 [fused multiplier] -> x2 -> c2r(x3) on (n1, n2, nh).
// x1 slabs: the x3 and x2 passes are local to the slab [L][n2][nh]; the x1 pass
//           needs whole x1 columns, so an all-to-all transposes the slab into the
//           k2-slab [n1][n2s][nh] (rank r keeps k2 in [r n2s, (r+1) n2s)), the x1
//           kernel runs there (the multiplier decodes global k2 via k2_off), and a
//           second all-to-all transposes back. The forward x2 pass stores straight into
//           the send blocks and the inverse x2 pass reads the received blocks through a
//           tensor map (TMA), so neither direction has a pack / unpack copy.
#include "vr_common.cuh"

namespace vr {
namespace {

double* sbuf(vr_ctx* ctx, int i) { return spec_buf(ctx, i); }
// the one-axis derivative passes move 16-byte pairs with cp.async
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// doubles in one complex row block [n2s][nh]
size_t row_block(const GridDims& g) { return static_cast<size_t>(g.n2s) * g.nh * 2; }

// x1 slabs: forward x2 pass of the slab spectrum `slab` ([L][n2][nh], after the row pass) and
// the transpose into the x1 layout `xl` ([n1][n2s][nh]). The x2 pass stores straight into the
// all-to-all send blocks (no pack copy); the received blocks ARE the x1 layout.
void x2_forward_to_x1(vr_ctx* ctx, const double* slab, double* xl) {
    const GridDims& g = ctx->g;
    double* send = sbuf(ctx, 7);
    pass_x2_to_blocks(ctx, slab, send);
    ctx->dist->alltoall(ctx, send, xl, g.L * row_block(g));
}

// x1 layout `xl` -> transpose back -> inverse x2 pass into the slab spectrum `slab`. The x1
// layout is already the send blocks; the x2 pass reads the received blocks through a tensor
// map whose row groups are the peer blocks (no unpack copy).
void x1_to_x2_inverse(vr_ctx* ctx, const double* xl, double* slab) {
    const GridDims& g = ctx->g;
    double* recv = sbuf(ctx, 7);
    ctx->dist->alltoall(ctx, xl, recv, g.L * row_block(g));
    pass_x2_from_blocks(ctx, recv, slab);
}

double inv_n(const GridDims& g) { return 1.0 / static_cast<double>(g.Ng); }

MultParams reg_mult(const vr_regnorm& norm, int mode, double beta) {
    MultParams mp;
    mp.kind = Mult::reg;
    mp.reg_kind = norm.kind;
    mp.reg_mode = mode;
    mp.gamma = norm.gamma;
    mp.helm_sq = norm.helmholtz_squared;
    mp.beta = beta;
    return mp;
}

// in (real slab) -> out (real slab) through the fused x1 multiplier; leaves the
// x2-inverse-transformed slab spectrum in `s` when `out` is null
void scalar_multiplier(vr_ctx* ctx, const double* in, double* s, double* out, const MultParams& mp,
                       const double* add) {
    pass_rows_forward(ctx, in, s);
    if (ctx->dist) {
        double* t = sbuf(ctx, 8);
        x2_forward_to_x1(ctx, s, t);
        pass_x1(ctx, t, t, 0, &mp);
        x1_to_x2_inverse(ctx, t, s);
    } else {
        pass_x2(ctx, s, -1);
        pass_x1(ctx, s, s, 0, &mp);
        pass_x2(ctx, s, +1);
    }
    if (out) pass_rows_inverse(ctx, s, out, inv_n(ctx->g), add);
}

}  // namespace

// r2c: on slabs the result is left in the x1 layout (what the elementwise
// spectral kernels and fft_c2r expect)
void fft_r2c(vr_ctx* ctx, const double* in, double* spec) {
    Range nvtx("fft_r2c");
    if (ctx->dist) {
        double* s = sbuf(ctx, 8);
        pass_rows_forward(ctx, in, s);
        x2_forward_to_x1(ctx, s, spec);
    } else {
        pass_rows_forward(ctx, in, spec);
        pass_x2(ctx, spec, -1);
    }
    pass_x1(ctx, spec, spec, -1, nullptr);
}

void fft_c2r(vr_ctx* ctx, double* spec, double* out, double scale, const double* add) {
    Range nvtx("fft_c2r");
    pass_x1(ctx, spec, spec, +1, nullptr);
    double* s = spec;
    if (ctx->dist) {
        s = sbuf(ctx, 8);
        x1_to_x2_inverse(ctx, spec, s);
    } else {
        pass_x2(ctx, s, +1);
    }
    pass_rows_inverse(ctx, s, out, scale, add);
}

void spectral_scalar_op(vr_ctx* ctx, const double* in, double* out, const MultParams& mp,
                        const double* add) {
    scalar_multiplier(ctx, in, sbuf(ctx, 0), out, mp, add);
}

void op_gradient(vr_ctx* ctx, const double* f, double* out3) {
    Range nvtx("gradient");
    const GridDims& g = ctx->g;
    if (!ctx->dist && aligned16(f) && aligned16(out3)) {  // d_a f needs only transforms along a
        // (gradient, spectral.cpp:108-122)
        for (int a = 0; a < 3; ++a) deriv_axis(ctx, a, f, out3 + a * g.N, sbuf(ctx, 0));
        return;
    }
    double* s0 = sbuf(ctx, 0);
    double* s1 = sbuf(ctx, 1);
    pass_rows_forward(ctx, f, s0);
    double* src = s0;
    if (ctx->dist) {
        src = sbuf(ctx, 8);
        x2_forward_to_x1(ctx, s0, src);
    } else {
        pass_x2(ctx, s0, -1);
    }
    for (int a = 0; a < 3; ++a) {
        MultParams mp;
        mp.kind = static_cast<Mult>(static_cast<int>(Mult::deriv0) + a);
        pass_x1(ctx, src, s1, 0, &mp);
        double* s = s1;
        if (ctx->dist) {
            s = sbuf(ctx, 2);
            x1_to_x2_inverse(ctx, s1, s);
        } else {
            pass_x2(ctx, s, +1);
        }
        pass_rows_inverse(ctx, s, out3 + a * g.N, inv_n(g), nullptr);
    }
}

void op_divergence(vr_ctx* ctx, const double* v3, double* out) {
    Range nvtx("divergence");
    const GridDims& g = ctx->g;
    if (!ctx->dist && aligned16(v3) && aligned16(out)) {  // sum_a d_a v_a with one-axis
        // derivatives (divergence, spectral.cpp:124-140)
        double* t = field_buf(ctx, 9);
        deriv_axis(ctx, 0, v3, t, sbuf(ctx, 0));
        deriv_axis(ctx, 1, v3 + g.N, out, sbuf(ctx, 0));
        add_scaled(ctx, out, 1.0, t, g.N);
        deriv_axis(ctx, 2, v3 + 2 * g.N, t, sbuf(ctx, 0));
        add_scaled(ctx, out, 1.0, t, g.N);
        return;
    }
    double* s[3];
    for (int a = 0; a < 3; ++a) {
        s[a] = sbuf(ctx, a);
        fft_r2c(ctx, v3 + a * g.N, s[a]);
    }
    double* acc = sbuf(ctx, 3);
    pass_spec_div(ctx, s[0], s[1], s[2], acc);
    fft_c2r(ctx, acc, out, inv_n(g), nullptr);
}

void op_projection(vr_ctx* ctx, const double* in3, double* out3, int kind, double beta_v,
                   double beta_w) {
    Range nvtx("projection");
    const GridDims& g = ctx->g;
    if (kind == VR_PROJ_IDENTITY) {
        if (in3 != out3)
            VR_CUDA(cudaMemcpyAsync(out3, in3, sizeof(double) * 3 * g.N, cudaMemcpyDeviceToDevice,
                                    ctx->stream));
        return;
    }
    if (kind == VR_PROJ_NEAR_INCOMPRESSIBLE && (beta_v <= 0.0 || beta_w <= 0.0))
        throw_argument("apply_projection: near-incompressible K needs beta_v, beta_w > 0");
    if (kind != VR_PROJ_INCOMPRESSIBLE && kind != VR_PROJ_NEAR_INCOMPRESSIBLE)
        throw_argument("apply_projection: unknown projection kind");
    double* s[3];
    for (int a = 0; a < 3; ++a) {
        s[a] = sbuf(ctx, a);
        fft_r2c(ctx, in3 + a * g.N, s[a]);
    }
    pass_spec_project(ctx, s[0], s[1], s[2], kind, beta_v, beta_w);
    for (int a = 0; a < 3; ++a) fft_c2r(ctx, s[a], out3 + a * g.N, inv_n(g), nullptr);
}

double reg_symbol(const vr_regnorm& n, double k2) {
    switch (n.kind) {
        case VR_REG_H1: return k2;
        case VR_REG_H2: return k2 * k2;
        case VR_REG_H3: return k2 * k2 * k2;
        case VR_REG_HELMHOLTZ: {
            const double s = k2 + n.gamma;
            return n.helmholtz_squared ? s * s : s;
        }
    }
    return 0.0;
}

void op_reg(vr_ctx* ctx, const double* in3, double* out3, const vr_regnorm& norm, int mode,
            double beta, const double* add3) {
    Range nvtx("reg_operator");
    const MultParams mp = reg_mult(norm, mode, beta);
    const long long N = ctx->g.N;
    for (int c = 0; c < 3; ++c)
        scalar_multiplier(ctx, in3 + c * N, sbuf(ctx, 0), out3 + c * N, mp,
                          add3 ? add3 + c * N : nullptr);
}

void op_reg_begin(vr_ctx* ctx, const double* in3, const vr_regnorm& norm, int mode, double beta) {
    Range nvtx("reg_operator_begin");
    const MultParams mp = reg_mult(norm, mode, beta);
    for (int c = 0; c < 3; ++c)
        scalar_multiplier(ctx, in3 + c * ctx->g.N, sbuf(ctx, 4 + c), nullptr, mp, nullptr);
}

// fp32 lane, one GPU: the forward half of op_reg on fp32 fields (rows widened in the
// r2c pass), leaving the spectra in sbuf(4..6) for op_reg_finish_f32
void op_reg_begin_f32(vr_ctx* ctx, const float* in3, const vr_regnorm& norm, int mode, double beta) {
    const MultParams mp = reg_mult(norm, mode, beta);
    for (int c = 0; c < 3; ++c) {
        double* s = sbuf(ctx, 4 + c);
        pass_rows_forward_f32(ctx, in3 + c * ctx->g.N, s);
        pass_x2(ctx, s, -1);
        pass_x1(ctx, s, s, 0, &mp);
        pass_x2(ctx, s, +1);
    }
}

void op_reg_finish_f32(vr_ctx* ctx, float* out3, const float* add3) {
    const GridDims& g = ctx->g;
    for (int c = 0; c < 3; ++c)
        pass_rows_inverse_f32(ctx, sbuf(ctx, 4 + c), out3 + c * g.N, inv_n(g),
                              add3 ? add3 + c * g.N : nullptr);
}

void op_reg_finish(vr_ctx* ctx, double* out3, const double* add3) {
    Range nvtx("reg_operator_finish");
    const GridDims& g = ctx->g;
    for (int c = 0; c < 3; ++c)
        pass_rows_inverse(ctx, sbuf(ctx, 4 + c), out3 + c * g.N, inv_n(g),
                          add3 ? add3 + c * g.N : nullptr);
}

}  // namespace vr
