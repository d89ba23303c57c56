"""ctypes binding to the in-tree C-ABI library (include/hybridcache.h).

Loading fails loudly: there is no CPU fallback anywhere in the package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import CapacityError, ConfigError, HcError, InputError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhybridcache_b200.so")

_lib = None

c_int_p = C.POINTER(C.c_int)
c_long_p = C.POINTER(C.c_long)
c_double_p = C.POINTER(C.c_double)
c_u16_p = C.POINTER(C.c_uint16)


def lib() -> C.CDLL:
    """Load libhybridcache_b200.so (built by paper_2501_01792_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() "
                              "(python -m paper_2501_01792_b200.build)")
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().hc_last_error().decode()
    raise {1: InputError, 2: CapacityError, 3: ConfigError}.get(rc, HcError)(msg)


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def _declare(L: C.CDLL) -> None:
    from . import _signatures
    for name, (res, args) in _signatures.SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
