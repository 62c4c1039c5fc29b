"""ctypes binding of the plain C fp64 oracle (``oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs, never by the product
package.  Independent of the CUDA path: no shared code, headers or constants.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_OMP_PATH = os.path.join(_HERE, "liboracle_omp.so")  # same source, OpenMP over rows
_lib = None
_libs = {}

CONV_EQ1, CONV_ALG1 = 0, 1
SCALES_PER_TENSOR, SCALES_PER_ROW = 0, 1


class OracleError(RuntimeError):
    pass


def lib(omp: bool = False):
    """The single-threaded oracle, or (omp=True) the same source built with OpenMP."""
    global _lib
    path = _OMP_PATH if omp else _LIB_PATH
    if path not in _libs:
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        i64, vp = ctypes.c_int64, ctypes.c_void_p
        L.orc_words_per_row.restype = i64
        L.orc_words_per_row.argtypes = [i64]
        L.orc_pack_slots.restype = ctypes.c_int
        L.orc_pack_slots.argtypes = [vp, vp]
        L.orc_unpack_slots.restype = ctypes.c_int
        L.orc_unpack_slots.argtypes = [ctypes.c_uint32, vp]
        L.orc_decode_masks.restype = None
        L.orc_decode_masks.argtypes = [ctypes.c_uint32, vp, vp]
        L.orc_pack_plane.restype = ctypes.c_int
        L.orc_pack_plane.argtypes = [vp, i64, i64, i64, vp]
        L.orc_unpack_plane.restype = ctypes.c_int
        L.orc_unpack_plane.argtypes = [vp, i64, i64, vp, i64]
        for name in ("orc_wl_direct", "orc_wl_embedding"):
            f = getattr(L, name)
            f.restype = ctypes.c_int
            f.argtypes = [vp, i64, i64, vp, ctypes.c_int, ctypes.c_int, vp, i64, vp, i64, vp]
        L.orc_wl_alg1.restype = ctypes.c_int
        L.orc_wl_alg1.argtypes = [vp, i64, i64, vp, ctypes.c_int, vp, vp, i64, vp, vp]
        L.orc_build_dense.restype = ctypes.c_int
        L.orc_build_dense.argtypes = [vp, i64, i64, vp, ctypes.c_int, vp, i64, vp, vp]
        L.orc_eval_dense.restype = ctypes.c_int
        L.orc_eval_dense.argtypes = [vp, vp, i64, i64, ctypes.c_int, vp, i64, vp]
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_num_threads.argtypes = []
        _libs[path] = L
        if not omp:
            _lib = L
    return _libs[path]


def _check(rc: int, what: str):
    if rc == -2:
        raise OracleError(f"{what}: invalid encoding (slot pattern (1,1))")
    if rc != 0:
        raise OracleError(f"{what}: error {rc}")


def words_per_row(m: int) -> int:
    return int(lib().orc_words_per_row(m))


def pack_slots(t) -> int:
    a = np.ascontiguousarray(t, dtype=np.int8)
    assert a.shape == (16,)
    out = np.zeros(1, dtype=np.uint32)
    _check(lib().orc_pack_slots(a.ctypes.data, out.ctypes.data), "pack_slots")
    return int(out[0])


def unpack_slots(p: int) -> np.ndarray:
    t = np.zeros(16, dtype=np.int8)
    _check(lib().orc_unpack_slots(p, t.ctypes.data), "unpack_slots")
    return t


def decode_masks(p: int) -> tuple[int, int]:
    kp = np.zeros(1, dtype=np.uint32)
    kn = np.zeros(1, dtype=np.uint32)
    lib().orc_decode_masks(p, kp.ctypes.data, kn.ctypes.data)
    return int(kp[0]), int(kn[0])


def pack_plane(dense: np.ndarray) -> np.ndarray:
    d = np.ascontiguousarray(dense, dtype=np.int8)
    n, m = d.shape
    out = np.zeros((n, words_per_row(m)), dtype=np.uint32)
    _check(lib().orc_pack_plane(d.ctypes.data, n, m, m, out.ctypes.data), "pack_plane")
    return out


def unpack_plane(words: np.ndarray, m: int) -> np.ndarray:
    w = np.ascontiguousarray(words, dtype=np.uint32)
    n = w.shape[0]
    out = np.zeros((n, m), dtype=np.int8)
    _check(lib().orc_unpack_plane(w.ctypes.data, n, m, out.ctypes.data, m), "unpack_plane")
    return out


def pack_planar(planes: np.ndarray) -> np.ndarray:
    """(4, n, m) int8 -> (4, n, W) uint32 planar words (App. H)."""
    return np.stack([pack_plane(planes[p]) for p in range(4)])


def _eval(fn, planar, n, m, scales, conv, x, rows):
    planar = np.ascontiguousarray(planar, dtype=np.uint32)
    assert planar.size == 4 * n * words_per_row(m)
    sc = np.ascontiguousarray(scales, dtype=np.float32)
    mode = SCALES_PER_ROW if sc.size == 4 * n and sc.ndim == 2 else SCALES_PER_TENSOR
    if mode == SCALES_PER_TENSOR:
        assert sc.size == 4
    xx = np.ascontiguousarray(x, dtype=np.complex64)
    if xx.ndim == 1:
        xx = xx[None, :]
    B = xx.shape[0]
    assert xx.shape[1] == m
    if rows is None:
        rows_arr, nrows, rp = None, n, None
    else:
        rows_arr = np.ascontiguousarray(rows, dtype=np.int64)
        nrows, rp = rows_arr.size, rows_arr.ctypes.data
    y = np.zeros((B, nrows), dtype=np.complex128)
    _check(fn(planar.ctypes.data, n, m, sc.ctypes.data, mode, conv, xx.ctypes.data, B, rp,
              nrows, y.ctypes.data), fn.__name__)
    return y


def wl_direct(planar, n, m, scales, x, conv=CONV_EQ1, rows=None) -> np.ndarray:
    """(B, nrows) complex128: y = Ux + W conj(x) (EQ1) or (U + conj W) x (ALG1)."""
    return _eval(lib().orc_wl_direct, planar, n, m, scales, conv, x, rows)


def wl_embedding(planar, n, m, scales, x, conv=CONV_EQ1, rows=None) -> np.ndarray:
    return _eval(lib().orc_wl_embedding, planar, n, m, scales, conv, x, rows)


def num_threads(omp: bool = False) -> int:
    return int(lib(omp).orc_num_threads())


def build_dense(planar, n, m, scales, rows=None, omp=False):
    """Phase (a): unpack + dense complex rows of U and W, each (nrows, m) complex128."""
    planar = np.ascontiguousarray(planar, dtype=np.uint32)
    assert planar.size == 4 * n * words_per_row(m)
    sc = np.ascontiguousarray(scales, dtype=np.float32)
    mode = SCALES_PER_ROW if sc.ndim == 2 else SCALES_PER_TENSOR
    if rows is None:
        rp, nrows = None, n
    else:
        rows_arr = np.ascontiguousarray(rows, dtype=np.int64)
        rp, nrows = rows_arr.ctypes.data, rows_arr.size
    U = np.empty((nrows, m), dtype=np.complex128)
    Wd = np.empty((nrows, m), dtype=np.complex128)
    _check(lib(omp).orc_build_dense(planar.ctypes.data, n, m, sc.ctypes.data, mode, rp, nrows,
                                    U.ctypes.data, Wd.ctypes.data), "build_dense")
    return U, Wd


def eval_dense(U, Wd, x, conv=CONV_EQ1, omp=False):
    """Phase (b): (B, nrows) complex128 from dense rows (bitwise == wl_direct)."""
    nrows, m = U.shape
    xx = np.ascontiguousarray(x, dtype=np.complex64)
    if xx.ndim == 1:
        xx = xx[None, :]
    B = xx.shape[0]
    y = np.zeros((B, nrows), dtype=np.complex128)
    _check(lib(omp).orc_eval_dense(U.ctypes.data, Wd.ctypes.data, nrows, m, conv, xx.ctypes.data,
                                   B, y.ctypes.data), "eval_dense")
    return y


def wl_alg1(planar, n, m, scales, x, rows=None):
    """Algorithm 1 literally (ALG1 convention, one vector).  Returns (y, counts)."""
    planar = np.ascontiguousarray(planar, dtype=np.uint32)
    sc = np.ascontiguousarray(scales, dtype=np.float32)
    mode = SCALES_PER_ROW if sc.ndim == 2 else SCALES_PER_TENSOR
    xx = np.ascontiguousarray(x, dtype=np.complex64).reshape(-1)
    assert xx.size == m
    if rows is None:
        rp, nrows = None, n
    else:
        rows_arr = np.ascontiguousarray(rows, dtype=np.int64)
        rp, nrows = rows_arr.ctypes.data, rows_arr.size
    y = np.zeros(nrows, dtype=np.complex128)
    counts = np.zeros(5, dtype=np.int64)
    _check(lib().orc_wl_alg1(planar.ctypes.data, n, m, sc.ctypes.data, mode, xx.ctypes.data,
                             rp, nrows, y.ctypes.data, counts.ctypes.data), "wl_alg1")
    return y, {"slots": int(counts[0]), "adds": int(counts[1]), "subs": int(counts[2]),
               "scale_muls": int(counts[3]), "inner_muls": int(counts[4])}


def tolerance_check(y, y_ref, scales, x, n_rows_idx=None):
    """North-star bar: rel L2 <= 1e-5 and per element |err| <= 1e-4 * max_c s_c(i) * sum_j |x_j|
    (|x_j| = |re| + |im|, checked for re and im separately).  Returns (ok, rel_l2, worst_ratio)."""
    y = np.asarray(y).astype(np.complex128)
    y_ref = np.asarray(y_ref).astype(np.complex128)
    B = y_ref.shape[0]
    err = y - y_ref
    rel = np.sqrt(np.sum(np.abs(err) ** 2)) / max(np.sqrt(np.sum(np.abs(y_ref) ** 2)), 1e-30)
    xx = np.asarray(x, dtype=np.complex64).reshape(B, -1)
    l1 = np.sum(np.abs(xx.real.astype(np.float64)) + np.abs(xx.imag.astype(np.float64)), axis=1)
    sc = np.asarray(scales, dtype=np.float64)
    if sc.ndim == 2:
        smax = sc.max(axis=1)
        if n_rows_idx is not None:
            smax = smax[np.asarray(n_rows_idx)]
    else:
        smax = np.full(y_ref.shape[1], sc.max())
    bound = 1e-4 * smax[None, :] * l1[:, None]
    ratio = np.maximum(np.abs(err.real), np.abs(err.imag)) / np.maximum(bound, 1e-300)
    worst = float(ratio.max()) if ratio.size else 0.0
    return (rel <= 1e-5 and worst <= 1.0), float(rel), worst
