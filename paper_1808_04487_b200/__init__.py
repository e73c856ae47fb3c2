"""B200-native (sm_100a) Gauss-Newton-Krylov registration hot path (CLAIRE, arXiv 1808.04487).

The product is libveloreg_gpu.so (C ABI: include/veloreg_gpu.h). This package
is a thin Python mirror of the reference's operator API over that ABI; it has
no CPU fallback. The library is loaded on first use of the mirror (any public
name below, or ``import paper_1808_04487_b200.veloreg``) and that raises
ImportError if it is not built. ``_abi_types`` (POD layouts) and ``phantom``
(numpy input generator) import without mapping the library, so the reference
CPU arm of bench.py never loads product code.
"""
import importlib

from ._abi_types import (ArgumentError, ConvergenceError, DimensionError, FormatError,  # noqa: F401
                         IoError, LogicError, NumericError, ResourceError, VelouregError)


def _mirror():
    return importlib.import_module(__name__ + ".veloreg")  # loads libveloreg_gpu.so (raises if absent)


def __getattr__(name):
    if name.startswith("__"):
        raise AttributeError(name)
    if name in ("veloreg", "phantom", "_lib", "_abi_types"):
        return importlib.import_module(f"{__name__}.{name}")
    veloreg = _mirror()
    try:
        return getattr(veloreg, name)
    except AttributeError:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}") from None


def __dir__():
    veloreg = _mirror()
    return sorted(set(globals()) | {n for n in dir(veloreg) if not n.startswith("_")})
