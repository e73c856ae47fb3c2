"""cufft_compare.py -- library baseline for the FFT passes: cuFFT (via torch.fft) fp64
r2c / c2r of one 256^3 field vs this library's vr_fft_r2c / vr_fft_c2r (same sizes)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_04487_b200 as vr  # noqa: E402
import paper_1808_04487_b200.veloreg as V  # noqa: E402


def timeit(fn, stream, reps=50):
    for _ in range(5):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


n = int(os.environ.get("N", "256"))
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda")
X = torch.fft.rfftn(x)
res = {"n": n}
s = torch.cuda.current_stream()
res["cufft_r2c_us"] = timeit(lambda: torch.fft.rfftn(x), s)
res["cufft_c2r_us"] = timeit(lambda: torch.fft.irfftn(X, s=(n, n, n)), s)
ctx = vr.Context(n)
f = ctx.to_device(x.cpu().numpy())
spec = ctx.empty(1, complex_spectrum=True)
out = ctx.empty(1)
st = torch.cuda.ExternalStream(ctx.stream)
res["ours_r2c_us"] = timeit(lambda: V._lib.call("vr_fft_r2c", ctx.handle, f.ptr, spec.ptr), st)
res["ours_c2r_us"] = timeit(lambda: V._lib.call("vr_fft_c2r", ctx.handle, spec.ptr, out.ptr), st)
print(json.dumps(res))
# the fused spectral operator: beta A v (H2) on 3 components, cuFFT r2c * multiplier * c2r vs
# this library's vr_apply_reg_operator (5 passes per component, multiplier fused in the x1 pass)
k = torch.fft.fftfreq(n, 1.0 / n, device="cuda", dtype=torch.float64)
k3 = torch.arange(n // 2 + 1, device="cuda", dtype=torch.float64)
mult = 1e-2 * (k[:, None, None] ** 2 + k[None, :, None] ** 2 + k3[None, None, :] ** 2) ** 2
v3 = torch.randn(3, n, n, n, dtype=torch.float64, device="cuda")
res["cufft_reg_op_3_us"] = timeit(lambda: [torch.fft.irfftn(torch.fft.rfftn(v3[c]) * mult, s=(n, n, n))
                                           for c in range(3)], s, reps=10)
dv3 = ctx.to_device(v3.cpu().numpy())
o3 = ctx.empty(3)
norm = V.make_norm("h2")
res["ours_reg_op_3_us"] = timeit(lambda: V._lib.call("vr_apply_reg_operator", ctx.handle, dv3.ptr, o3.ptr,
                                                     V.C.byref(norm), 0, 1e-2), st, reps=10)
print(json.dumps(res))
