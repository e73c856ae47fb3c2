"""GPU memory contract (proj/tests/test_objective.cpp:238-270, FieldAllocStats of
proj/include/veloreg/field.hpp:16-33) measured with the library's own device accounting
(vr_ctx_memory): peak of the allocations made during evaluate + compute_gradient and during
one GN Hessian matvec, in units of one fp64 field.

The reference's bounds are (n_t + 7 + 12) fields for the gradient and (n_t + 10 + 8) for the
matvec, growing by one field per extra time step. This design keeps the grad m_j cache in
the EvalState on purpose (3 (n_t + 1) fields: it removes 40 of the reference's 46 FFTs per
matvec), so the gradient bound here is the reference's plus that cache,
growing by 1 + 3 = 4 fields per step; the matvec allocates nothing per call (its workspace
belongs to the Objective) and must stay within the reference's bound.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_memory_contract(vr, ref):
    dims = (32, 32, 32)
    c = vr.Context(dims)
    F = 8.0 * np.prod(dims)
    a = 0.5 + ref.random_smooth_scalar(dims, 2, 140, 0.3)
    b = 0.5 + ref.random_smooth_scalar(dims, 2, 141, 0.3)
    mR, mT = c.to_device(a), c.to_device(b)

    def measure(nt):
        o = vr.Objective(c, mR, mT, vr.make_model("h2", beta_v=1e-3, nt=nt))
        v = c.to_device(ref.random_smooth_vector(dims, 2, 141, 0.2))
        vt = c.to_device(ref.random_smooth_vector(dims, 2, 142, 1.0))
        c.synchronize()
        live0 = c.memory()["live_bytes"]
        c.reset_memory_peak()
        s = o.evaluate(v)
        o.compute_gradient(s)
        grad_peak = (c.memory()["peak_bytes"] - live0) / F
        live1 = c.memory()["live_bytes"]
        c.reset_memory_peak()
        hv = o.hessian_matvec(s, vt)  # returns a new vector field, as the reference does
        matvec_peak = (c.memory()["peak_bytes"] - live1) / F
        state_fields = (live1 - live0) / F
        hv.free()
        s.close()
        o.close()
        return grad_peak, matvec_peak, state_fields

    measure(4)  # first use creates the context's persistent spectral / field scratch
    g4, h4, s4 = measure(4)
    g16, h16, s16 = measure(16)
    print(f"fields: gradient peak nt=4 {g4:.2f} nt=16 {g16:.2f}; matvec peak nt=4 {h4:.2f} nt=16 {h16:.2f}; "
          f"EvalState nt=4 {s4:.2f} nt=16 {s16:.2f}")
    for nt, g, h in ((4, g4, h4), (16, g16, h16)):
        assert g <= (nt + 7 + 12) + 3 * (nt + 1), (nt, g)
        assert h <= nt + 10 + 8, (nt, h)
    assert g16 - g4 <= 12 * 4 + 0.5  # one m_j + three d_a m_j per extra time step
    assert h16 - h4 <= 12.5
    # footprint report: EvalState = v, X_bwd, m history, X_fwd, factor, grad m cache, gradient
    assert abs(s4 - (3 + 3 + 5 + 3 + 1 + 15 + 3)) <= 0.5
