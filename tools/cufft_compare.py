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
