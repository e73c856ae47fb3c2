"""The compiled C++ drop-in (include/veloreg_gpu.hpp) over the C ABI.

* CPU: the adapter compiles and links against libveloreg_gpu.so and the oracle harness;
  a drift check compiles it next to the reference's own headers (enum values, field
  names of RegModel / RegNorm / SolverParams, the Objective<double> method set).
* GPU: tests/cpp/test_gpu_adapter.cpp re-runs the reference's property tests
  (proj/tests/test_objective.cpp:160-215, proj/tests/test_solver.cpp:138-178) through the
  adapter on the device.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GPU_SO = os.path.join(ROOT, "paper_1808_04487_b200", "libveloreg_gpu.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libveloreg_ref.so")
REF_INC = "/root/reference/proj/include"


def _build(out):
    for so in (GPU_SO, REF_SO):
        if not os.path.exists(so):
            pytest.skip(f"{so} not built")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(ROOT, "oracle", "shims"), os.path.join(ROOT, "tests", "cpp", "test_gpu_adapter.cpp"),
           GPU_SO, REF_SO, f"-Wl,-rpath,{os.path.dirname(GPU_SO)}:{os.path.dirname(REF_SO)}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return out


def test_adapter_compiles_and_links(tmp_path):
    _build(str(tmp_path / "test_gpu_adapter"))


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present (GPU box)")
def test_adapter_has_no_drift_against_reference_headers():
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), "-I", REF_INC,
                        os.path.join(ROOT, "tests", "cpp", "adapter_drift.cpp")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_reference_property_tests_through_the_adapter(tmp_path):
    exe = _build(str(tmp_path / "test_gpu_adapter"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout + r.stderr
