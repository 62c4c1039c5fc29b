"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic: only the counter-based SplitMix64 draws
described in ``gen.h`` (codes, scales, complex N(0,1) activations) and the
layer shapes / distributions BASELINE.json's configs name.  Both ``oracle/``
(via the tests) and the product benchmark import this module; neither imports
the other.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HOST_LIB = os.path.join(_HERE, "libww_inputs.so")
_DEV_LIB = os.path.join(_HERE, "libww_inputs_cuda.so")

_host = None
_dev = None

# code-distribution thresholds (t0 = P(0), t1 = P(0) + P(+1)), DESIGN.md "Input recipe"
UNIFORM3 = (1.0 / 3.0, 1.0 / 3.0 + 1.0 / 3.0)  # config 1: i.i.d. uniform over {-1,0,+1}
LLAMA = (0.4, 0.4 + 0.3)  # configs 2-5: P(0)=0.4, P(+1)=P(-1)=0.3

STREAM_SCALES = 4
STREAM_X = 5


def _lib():
    global _host
    if _host is None:
        if not os.path.exists(_HOST_LIB):
            raise RuntimeError(f"{_HOST_LIB} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(_HOST_LIB)
        u64, i64, dbl = ctypes.c_uint64, ctypes.c_int64, ctypes.c_double
        L.wwi_mix64.restype = u64
        L.wwi_mix64.argtypes = [u64]
        L.wwi_draw.restype = u64
        L.wwi_draw.argtypes = [u64, u64, u64]
        L.wwi_uniform.restype = dbl
        L.wwi_uniform.argtypes = [u64, u64, u64]
        L.wwi_layer_seed.restype = u64
        L.wwi_layer_seed.argtypes = [u64, i64, i64]
        L.wwi_gen_codes.restype = None
        L.wwi_gen_codes.argtypes = [u64, u64, i64, i64, i64, dbl, dbl, ctypes.c_void_p, i64]
        L.wwi_gen_uniform_f32.restype = None
        L.wwi_gen_uniform_f32.argtypes = [u64, u64, i64, i64, dbl, dbl, ctypes.c_void_p]
        L.wwi_gen_normal_c64.restype = None
        L.wwi_gen_normal_c64.argtypes = [u64, u64, i64, i64, ctypes.c_void_p]
        _host = L
    return _host


def _devlib():
    global _dev
    if _dev is None:
        if not os.path.exists(_DEV_LIB):
            raise RuntimeError(f"{_DEV_LIB} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(_DEV_LIB)
        u64, i64, dbl = ctypes.c_uint64, ctypes.c_int64, ctypes.c_double
        L.wwi_gen_codes_device.restype = ctypes.c_int
        L.wwi_gen_codes_device.argtypes = [u64, u64, i64, i64, i64, dbl, dbl, ctypes.c_void_p,
                                           i64, ctypes.c_void_p]
        _dev = L
    return _dev


def layer_seed(seed: int, layer: int, proj: int) -> int:
    return int(_lib().wwi_layer_seed(seed, layer, proj))


def draw(seed: int, stream: int, k: int) -> int:
    return int(_lib().wwi_draw(seed, stream, k))


def uniform(seed: int, stream: int, k: int) -> float:
    return float(_lib().wwi_uniform(seed, stream, k))


def codes(seed: int, plane: int, n: int, m: int, dist=LLAMA, row0: int = 0,
          nrows: int | None = None) -> np.ndarray:
    """Dense int8 codes of one plane (rows row0..row0+nrows of an n x m plane)."""
    if nrows is None:
        nrows = n - row0
    out = np.empty((nrows, m), dtype=np.int8)
    if nrows and m:
        _lib().wwi_gen_codes(seed, plane, m, row0, nrows, dist[0], dist[1],
                             out.ctypes.data, m)
    return out


def planes(seed: int, n: int, m: int, dist=LLAMA, row0: int = 0,
           nrows: int | None = None) -> np.ndarray:
    """(4, nrows, m) int8: U_re, U_im, W_re, W_im (App. H plane order)."""
    return np.stack([codes(seed, p, n, m, dist, row0, nrows) for p in range(4)])


def codes_device(seed: int, plane: int, n: int, m: int, out, dist=LLAMA, stream=None,
                 row0: int = 0):
    """Fill a (n, m) int8 CUDA tensor ``out`` (leading dim out.stride(0)) on the GPU with
    rows row0 .. row0+n of the plane (same values as ``codes(..., row0=row0)``)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    rc = _devlib().wwi_gen_codes_device(seed, plane, m, row0, n, dist[0], dist[1],
                                        out.data_ptr(), out.stride(0), s.cuda_stream)
    if rc != 0:
        raise RuntimeError("wwi_gen_codes_device failed")


def scales(seed: int, n: int, per_row: bool, lo: float, hi: float) -> np.ndarray:
    """Per-row (n,4) or per-tensor (4,) fp32 scales [sUr, sUi, sWr, sWi]."""
    cnt = 4 * n if per_row else 4
    out = np.empty(cnt, dtype=np.float32)
    _lib().wwi_gen_uniform_f32(seed, STREAM_SCALES, 0, cnt, lo, hi, out.ctypes.data)
    return out.reshape(n, 4) if per_row else out


def activations(seed: int, m: int, B: int = 1) -> np.ndarray:
    """(B, m) complex64 activations, Re, Im ~ N(0,1) i.i.d."""
    out = np.empty(2 * B * m, dtype=np.float32)
    if B * m:
        _lib().wwi_gen_normal_c64(seed, STREAM_X, 0, B * m, out.ctypes.data)
    return out.view(np.complex64).reshape(B, m)


@dataclass(frozen=True)
class LayerSpec:
    """One widely-linear layer of a BASELINE config (complex n x m)."""
    name: str
    n: int
    m: int
    dist: tuple
    per_row: bool
    scale_lo: float
    scale_hi: float


# BASELINE.json configs (complex shapes; real LLaMA-2-7B d=4096 -> 2048, d_ff=11008 -> 5504)
C1 = LayerSpec("c1_128x128", 128, 128, UNIFORM3, False, 0.5, 2.0)
C2 = LayerSpec("c2_qkvo_2048x2048", 2048, 2048, LLAMA, True, 0.01, 0.1)
C3A = LayerSpec("c3a_gateup_5504x2048", 5504, 2048, LLAMA, True, 0.01, 0.1)
C3B = LayerSpec("c3b_down_2048x5504", 2048, 5504, LLAMA, True, 0.01, 0.1)
# config 4: per decoder layer, projections q,k,v,o,gate,up,down (proj index 0..6)
C4_PROJS = (C2, C2, C2, C2, C3A, C3A, C3B)
C4_LAYERS = 32
C5_BATCHES = (1, 2, 4, 8, 16)
