import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libveloreg_gpu.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b.ravel())
    d = np.linalg.norm((a - b).ravel())
    return d / nb if nb > 0 else d


def periodic_diff(a, b):
    d = np.mod(np.asarray(a) - np.asarray(b) + np.pi, 2 * np.pi) - np.pi
    return np.abs(d)


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as _ref
    if not _ref.available():
        pytest.skip("oracle/_ref/libveloreg_ref.so not built (make -C oracle lib)")
    _ref.load()
    _ref.set_workers(min(8, os.cpu_count() or 1))
    return _ref


@pytest.fixture(scope="session")
def vr():
    import paper_1808_04487_b200 as _vr
    return _vr


_CTX = {}


@pytest.fixture
def ctx(vr):
    def get(dims):
        dims = (dims,) * 3 if isinstance(dims, int) else tuple(dims)
        if dims not in _CTX:
            _CTX[dims] = vr.Context(dims)
        return _CTX[dims]
    return get
