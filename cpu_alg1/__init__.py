"""ctypes binding of libww_cpu.so: the paper's Algorithm 1 on AVX-512F + BMI2 with OpenMP
(SURVEY §8f NEXT-4), a CPU baseline beside the GPU kernel.  Not a fallback of the CUDA
product path and independent of the oracle."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libww_cpu.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(_PATH)
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        L.wwc_supported.restype = ctypes.c_int
        L.wwc_max_threads.restype = ctypes.c_int
        L.wwc_wl_gemv.restype = ctypes.c_int
        L.wwc_wl_gemv.argtypes = [vp, i64, i64, vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int]
        _lib = L
    return _lib


def supported() -> bool:
    return bool(lib().wwc_supported())


def max_threads() -> int:
    return int(lib().wwc_max_threads())


def wl_gemv(planar, n, m, scales, x, conv=0, nthreads=0):
    """y (complex64, n) from App. H planar words (4, n, W) uint32, scales (n, 4) or (4,)."""
    pl = np.ascontiguousarray(planar, dtype=np.uint32)
    sc = np.ascontiguousarray(scales, dtype=np.float32)
    xx = np.ascontiguousarray(x, dtype=np.complex64).reshape(-1)
    y = np.empty(n, dtype=np.complex64)
    rc = lib().wwc_wl_gemv(pl.ctypes.data, n, m, sc.ctypes.data, int(sc.ndim == 2), conv,
                           xx.ctypes.data, y.ctypes.data, nthreads)
    if rc == -2:
        raise RuntimeError("CPU lacks AVX-512F or BMI2")
    if rc != 0:
        raise ValueError(f"wwc_wl_gemv: error {rc}")
    return y
