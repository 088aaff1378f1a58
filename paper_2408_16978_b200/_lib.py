"""ctypes loading of the in-tree CUDA libraries (argument marshalling only; no compute here).

There is deliberately no fallback: if ``libfpdt.so`` is missing or fails to load, every
entry point raises.  Build it with ``python -m paper_2408_16978_b200.build``.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
_LIB = None
_DIAG = None
_GEN = None

c_int, c_int64, c_float, c_void_p, c_char_p, c_size_t = (ctypes.c_int, ctypes.c_int64, ctypes.c_float,
                                                         ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t)


class FpdtLibraryMissing(RuntimeError):
    pass


def _declare(lib):
    from . import fpdt as _f
    _f._declare(lib)
    return lib


def load():
    global _LIB
    if _LIB is None:
        path = os.path.join(PKG, "libfpdt.so")
        if not os.path.exists(path):
            raise FpdtLibraryMissing(f"{path} not built (run python -m paper_2408_16978_b200.build)")
        _LIB = _declare(ctypes.CDLL(path))
    return _LIB


def load_diag():
    global _DIAG
    if _DIAG is None:
        load()
        path = os.path.join(PKG, "libfpdt_diag.so")
        if not os.path.exists(path):
            raise FpdtLibraryMissing(f"{path} not built (run python -m paper_2408_16978_b200.build)")
        from . import fpdt as _f
        _DIAG = ctypes.CDLL(path)
        _f._declare_diag(_DIAG)
    return _DIAG


def load_generator():
    global _GEN
    if _GEN is None:
        path = os.path.join(ROOT, "fpdt_inputs", "libfpdt_gen.so")
        if not os.path.exists(path):
            raise FpdtLibraryMissing(f"{path} not built")
        g = ctypes.CDLL(path)
        g.fpdt_gen_fill.argtypes = [c_void_p, c_int, c_int, c_int, ctypes.c_uint32, c_int64, c_int, c_int, c_int64,
                                    c_int, c_int, c_int64, c_void_p]
        g.fpdt_gen_fill.restype = c_int
        _GEN = g
    return _GEN
