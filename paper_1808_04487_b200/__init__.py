"""B200-native (sm_100a) Gauss-Newton-Krylov registration hot path (CLAIRE, arXiv 1808.04487).

The product is libveloreg_gpu.so (C ABI: include/veloreg_gpu.h). This package
is a thin Python mirror of the reference's operator API over that ABI; it has
no CPU fallback and raises ImportError if the library is not built.
"""
from . import _lib
from ._lib import (ArgumentError, ConvergenceError, DimensionError, FormatError,  # noqa: F401
                   IoError, LogicError, NumericError, ResourceError, VelouregError)

_lib.load()

from .veloreg import *  # noqa: F401,F403,E402
from .veloreg import Context, DeviceArray, EvalState, Objective  # noqa: F401,E402

__all__ = [n for n in dir() if not n.startswith("_")]
