"""Measured per-pipe issue peaks of the SM (lib/libpf_pipes.so, include/pf_pipes.h).

Measurement support for bench.py's roofline.pipes: the denominators of the
pipe-utilisation figures are measured on the box, not taken from a datasheet.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Dict

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libpf_pipes.so")

SIGNATURES = [
    ("pf_pipe_count", C.c_int, []),
    ("pf_pipe_name", C.c_char_p, [C.c_int]),
    ("pf_pipe_error", C.c_char_p, []),
    ("pf_pipe_peaks", C.c_int, [C.c_void_p, C.c_int32]),
]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it first (__graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def pipe_peaks(device: int = 0) -> Dict[str, float]:
    """{instruction kind: warp-instructions per SM per clock} measured on `device`."""
    L = lib()
    n = L.pf_pipe_count()
    out = (C.c_double * n)()
    rc = L.pf_pipe_peaks(out, device)
    if rc:
        raise RuntimeError(f"pf_pipe_peaks failed ({rc}): {L.pf_pipe_error().decode()}")
    return {L.pf_pipe_name(i).decode(): float(out[i]) for i in range(n)}
