"""ctypes wrapper over the C oracle (oracle/lib/liborc.so) -- TEST INFRASTRUCTURE ONLY.

Used by tests/ (checker) and by bench.py's CPU-baseline / `--impl reference`
legs (timed CPU port of the reference runtime).  See oracle/rbx_oracle.c.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "lib", "liborc.so")
_CODES = {"f32": 0, "f64": 1, "i64": 2}
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.orc_replay.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_void_p)]
        _lib.orc_runtime_port.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_double)]
        _lib.orc_chunk_bounds.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    return _lib


def chunk_bounds(count: int, n: int, i: int) -> tuple[int, int]:
    off, ln = ctypes.c_int64(), ctypes.c_int64()
    if lib().orc_chunk_bounds(count, n, i, ctypes.byref(off), ctypes.byref(ln)) != 0:
        raise ValueError("bad chunk request")
    return off.value, ln.value


def _args(dims, bufs):
    d = (ctypes.c_int * len(dims))(*dims)
    ptrs = (ctypes.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
    return d, ptrs


def replay_inplace(dims, bufs: list, dtype: str) -> None:
    """replay(multiring_schedule(Grid(dims), n), bufs) applied in place."""
    assert all(b.flags.c_contiguous for b in bufs)
    d, ptrs = _args(dims, bufs)
    if lib().orc_replay(d, len(dims), len(bufs[0]), _CODES[dtype], ptrs) != 0:
        raise ValueError(f"bad dims {dims}")


def runtime_port(dims, bufs: list, dtype: str) -> float:
    """The reference runtime's phase loop, one thread per rank, in place; returns seconds."""
    d, ptrs = _args(dims, bufs)
    secs = ctypes.c_double()
    if lib().orc_runtime_port(d, len(dims), len(bufs[0]), _CODES[dtype], ptrs, ctypes.byref(secs)) != 0:
        raise ValueError(f"bad dims {dims}")
    return secs.value


def replay(dims, bufs: list, dtype: str) -> list:
    out = [np.array(b, copy=True) for b in bufs]
    replay_inplace(dims, out, dtype)
    return out
