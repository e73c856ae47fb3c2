"""CPU: the bench's byte model and measurement contract helpers."""
import json
import os

import pytest

import bench


def test_matvec_byte_model_matches_survey():
    # B_mv = 8N [9 + 8(nt+1) + 12 nt] + 6 F_c  (SURVEY 8(d) "Bytes at each config")
    for n, gb in ((64, 0.216), (128, 1.730), (256, 13.83), (512, 110.6)):
        b, per_launch = bench.bytes_model(n, 4)
        assert abs(b / 1e9 - gb) <= 0.005 * gb
    b, per_launch = bench.bytes_model(256, 4)
    F = 8.0 * 256 ** 3
    assert per_launch["sl_incstate_step"] == 11 * F and per_launch["sl_adjoint_step"] == 6 * F


def test_measured_peak_source():
    peak, kind = bench.measured_peak()
    assert peak > 1000.0 and kind in ("measured", "fallback")
    if os.path.exists(os.path.join(bench.ROOT, "MEASURED_PEAKS.json")):
        assert kind == "measured"


def test_profiles_bench_line_contract():
    # the committed bench line carries the keys the driver and the judge read
    p = os.path.join(bench.ROOT, "profiles", "r01_bench.json")
    if not os.path.exists(p):
        pytest.skip("no committed bench line")
    d = json.load(open(p))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline",
              "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["warmup"] >= 3 and d["dtype"] == "f64" and d["gpu_launches"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert abs(d["roofline"]["frac"] - d["roofline"]["achieved"] / d["roofline"]["peak"]) < 1e-9
