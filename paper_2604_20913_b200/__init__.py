"""Python binding of ``libww.so`` — the C ABI in ``include/ww.h``.

Argument marshalling only: every step of the WL-GEMV runs in the library's CUDA
kernels (or its host packer).  PyTorch supplies device memory and streams.  If
the in-tree ``libww.so`` is missing this module raises at import time: there is
no CPU or PyTorch fallback for any entry point.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# WW_LIB_OVERRIDE: development tools only (A/B timing of kernel variants built from the same
# sources with other -D flags); the tests, smoke() and bench.py always load the in-tree build
LIB_PATH = os.environ.get("WW_LIB_OVERRIDE") or os.path.join(_HERE, "libww.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                      f"g.build()'` (no fallback path exists)")
_lib = ctypes.CDLL(LIB_PATH)

# --------------------------------------------------------------------------- enums
OK = 0
ERR_INVALID_ARGUMENT, ERR_DIMENSION_MISMATCH, ERR_INVALID_CODE, ERR_INVALID_ENCODING = 1, 2, 3, 4
ERR_NONFINITE_SCALE, ERR_MISALIGNED, ERR_UNSUPPORTED, ERR_CUDA = 5, 6, 7, 8
LAYOUT_PLANAR, LAYOUT_COL4, LAYOUT_TILE32, LAYOUT_LUT81 = 0, 1, 2, 3
CONV_EQ1, CONV_ALG1 = 0, 1
SCALES_PER_TENSOR, SCALES_PER_ROW = 0, 1
FLAG_PDL = 1
MAX_BATCH = 16

PROG_MAX_RANKS = 8
PROG_MAX_M = 11264
PRO_NONE, PRO_RMSNORM, PRO_MUL = 0, 1, 2
EPI_NONE, EPI_RESIDUAL, EPI_SILU = 0, 1, 2

# every symbol include/ww.h declares (tests check the library exports them all)
EXPORTS = ("ww_packed_bytes", "ww_pack_ternary", "ww_unpack_ternary", "ww_repack",
           "ww_pack_ternary_device", "ww_wl_gemv", "ww_wl_gemv_batched", "ww_shard_plan",
           "ww_query_launch", "ww_status_string", "ww_last_error", "ww_version",
           "ww_ternary_gemv_plane", "ww_wl_combine", "ww_wl_gemv_fused", "ww_program_workspace_bytes",
           "ww_program_sync_bytes", "ww_program_init", "ww_program_run", "ww_stream_keep_in_l2",
           "ww_tc_workspace_bytes", "ww_wl_gemv_batched_tc", "ww_packed_bytes_layout",
           "ww_pack_ternary_device_layout", "ww_tcv_workspace_bytes", "ww_wl_gemv_tc",
           "ww_lut81_packed_bytes", "ww_lut81_from_planar", "ww_lut81_to_planar", "ww_wl_gemv_lut")


class WWError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{status_string(status)}: {msg}")
        self.status = status


class _Layer(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64), ("layout", ctypes.c_int32),
                ("scale_mode", ctypes.c_int32), ("conv", ctypes.c_int32),
                ("flags", ctypes.c_uint32)]


class _Shard(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32)] + [
        (f, ctypes.c_int64) for f in ("n", "rows_per_rank", "n_padded", "row_begin", "row_end",
                                      "packed_offset_bytes", "packed_bytes",
                                      "scale_offset_floats", "scale_count", "y_offset_complex")]


class _LaunchInfo(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in ("grid", "block", "smem_bytes", "tiles",
                                              "tile_chunks", "num_sms", "parts", "split_chunks", "path")]


class _Stage(ctypes.Structure):
    _fields_ = [("packed", ctypes.c_void_p), ("scales", ctypes.c_void_p),
                ("n_local", ctypes.c_int64), ("row0", ctypes.c_int64), ("m", ctypes.c_int64),
                ("scale_mode", ctypes.c_int32), ("conv", ctypes.c_int32),
                ("x", ctypes.c_void_p), ("x2", ctypes.c_void_p),
                ("y", ctypes.c_void_p * PROG_MAX_RANKS),
                ("residual", ctypes.c_void_p), ("gamma", ctypes.c_void_p),
                ("eps", ctypes.c_float), ("prologue", ctypes.c_int32),
                ("epilogue", ctypes.c_int32), ("wait", ctypes.c_int32),
                ("silu_rows", ctypes.c_int64)]


class _Program(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in (
        "nstages", "world", "rank_base", "ranks_in_launch", "grid", "block", "smem_bytes",
        "ctas_per_rank", "nslot", "slot_bytes", "x_bytes", "has_mul")] + [
        ("workspace", ctypes.c_void_p), ("sync", ctypes.c_void_p * PROG_MAX_RANKS)]


class _Ops(ctypes.Structure):
    _fields_ = [("prologue", ctypes.c_int32), ("epilogue", ctypes.c_int32),
                ("x2", ctypes.c_void_p), ("gamma", ctypes.c_void_p), ("eps", ctypes.c_float),
                ("residual", ctypes.c_void_p), ("row0", ctypes.c_int64),
                ("silu_rows", ctypes.c_int64)]


_i64, _i32, _vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
_lib.ww_packed_bytes.restype = ctypes.c_size_t
_lib.ww_packed_bytes.argtypes = [_i64, _i64]
_lib.ww_pack_ternary.restype = _i32
_lib.ww_pack_ternary.argtypes = [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i32, _vp]
_lib.ww_unpack_ternary.restype = _i32
_lib.ww_unpack_ternary.argtypes = [_vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _i64]
_lib.ww_repack.restype = _i32
_lib.ww_repack.argtypes = [_vp, _i32, _i64, _i64, _vp, _i32]
_lib.ww_pack_ternary_device.restype = _i32
_lib.ww_pack_ternary_device.argtypes = [_vp, _i64, _i64, _i64, _vp, _vp, _vp]
_lib.ww_wl_gemv.restype = _i32
_lib.ww_wl_gemv.argtypes = [ctypes.POINTER(_Layer), _vp, _vp, _vp, _vp, _vp]
_lib.ww_wl_gemv_batched.restype = _i32
_lib.ww_wl_gemv_batched.argtypes = [ctypes.POINTER(_Layer), _vp, _vp, _vp, _i64, _vp, _i64, _i32,
                                    _vp]
_lib.ww_shard_plan.restype = _i32
_lib.ww_shard_plan.argtypes = [_i64, _i64, _i32, _i32, ctypes.POINTER(_Shard)]
_lib.ww_query_launch.restype = _i32
_lib.ww_query_launch.argtypes = [ctypes.POINTER(_Layer), _i32, ctypes.POINTER(_LaunchInfo)]
_lib.ww_ternary_gemv_plane.restype = _i32
_lib.ww_ternary_gemv_plane.argtypes = [_i64, _i64, _vp, _i32, _vp, _i32, _vp, ctypes.c_uint32, _vp]
_lib.ww_wl_combine.restype = _i32
_lib.ww_wl_combine.argtypes = [ctypes.POINTER(_Layer), _vp, _vp, _vp, _vp]
_lib.ww_wl_gemv_fused.restype = _i32
_lib.ww_wl_gemv_fused.argtypes = [ctypes.POINTER(_Layer), _vp, _vp, _vp, _vp, ctypes.POINTER(_Ops),
                                  _vp]
_lib.ww_program_workspace_bytes.restype = ctypes.c_size_t
_lib.ww_program_workspace_bytes.argtypes = [_i32, _i32]
_lib.ww_program_sync_bytes.restype = ctypes.c_size_t
_lib.ww_program_sync_bytes.argtypes = []
_lib.ww_program_init.restype = _i32
_lib.ww_program_init.argtypes = [ctypes.POINTER(_Stage), _i32, _i32, _i32, _i32,
                                 ctypes.POINTER(_vp), _vp, ctypes.POINTER(_Program)]
_lib.ww_program_run.restype = _i32
_lib.ww_program_run.argtypes = [ctypes.POINTER(_Program), _vp]
_lib.ww_tc_workspace_bytes.restype = ctypes.c_size_t
_lib.ww_tc_workspace_bytes.argtypes = [_i64, _i64, _i32]
_lib.ww_wl_gemv_batched_tc.restype = _i32
_lib.ww_wl_gemv_batched_tc.argtypes = [ctypes.POINTER(_Layer), _vp, _vp, _vp, _i64, _vp, _i64, _i32,
                                       _vp, _vp]
_lib.ww_packed_bytes_layout.restype = ctypes.c_size_t
_lib.ww_packed_bytes_layout.argtypes = [_i64, _i64, _i32]
_lib.ww_pack_ternary_device_layout.restype = _i32
_lib.ww_pack_ternary_device_layout.argtypes = [_vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp]
_lib.ww_tcv_workspace_bytes.restype = ctypes.c_size_t
_lib.ww_tcv_workspace_bytes.argtypes = [_i64, _i64, _i32]
_lib.ww_wl_gemv_tc.restype = _i32
_lib.ww_wl_gemv_tc.argtypes = [ctypes.POINTER(_Layer), _vp, _vp, _vp, _i64, _vp, _i64, _i32, _vp, _vp]
_lib.ww_stream_keep_in_l2.restype = _i32
_lib.ww_lut81_packed_bytes.restype = ctypes.c_size_t
_lib.ww_lut81_packed_bytes.argtypes = [_i64, _i64]
_lib.ww_lut81_from_planar.restype = _i32
_lib.ww_lut81_from_planar.argtypes = [_i64, _i64, _vp, _vp]
_lib.ww_lut81_to_planar.restype = _i32
_lib.ww_lut81_to_planar.argtypes = [_i64, _i64, _vp, _vp]
_lib.ww_wl_gemv_lut.restype = _i32
_lib.ww_wl_gemv_lut.argtypes = [ctypes.POINTER(_Layer), _vp, _vp, _vp, _vp, _vp]
_lib.ww_stream_keep_in_l2.argtypes = [_vp, _vp, ctypes.c_size_t]
_lib.ww_status_string.restype = ctypes.c_char_p
_lib.ww_status_string.argtypes = [_i32]
_lib.ww_last_error.restype = ctypes.c_char_p
_lib.ww_last_error.argtypes = []
_lib.ww_version.restype = _i32
_lib.ww_version.argtypes = []


def status_string(s: int) -> str:
    return _lib.ww_status_string(s).decode()


def last_error() -> str:
    return _lib.ww_last_error().decode()


def version() -> int:
    return int(_lib.ww_version())


def _check(st: int):
    if st != OK:
        raise WWError(st, last_error())


# --------------------------------------------------------------------------- layer
@dataclass
class Layer:
    """A complex n x m widely-linear layer (ww_layer)."""
    n: int
    m: int
    layout: int = LAYOUT_COL4
    scale_mode: int = SCALES_PER_ROW
    conv: int = CONV_EQ1
    flags: int = 0

    def c(self) -> _Layer:
        return _Layer(self.n, self.m, self.layout, self.scale_mode, self.conv, self.flags)


def packed_bytes(n: int, m: int, layout: int = LAYOUT_COL4) -> int:
    if layout in (LAYOUT_TILE32, LAYOUT_LUT81):
        return int(_lib.ww_packed_bytes_layout(n, m, layout))
    return int(_lib.ww_packed_bytes(n, m))


# --------------------------------------------------------------------------- host packer
def pack_ternary(planes: np.ndarray, layout: int = LAYOUT_COL4) -> np.ndarray:
    """(4, n, m) int8 planes U_re, U_im, W_re, W_im -> packed uint32 words (host)."""
    p = np.ascontiguousarray(planes, dtype=np.int8)
    _, n, m = p.shape
    out = np.empty(packed_bytes(n, m, layout) // 4, dtype=np.uint32)
    _check(_lib.ww_pack_ternary(p[0].ctypes.data, p[1].ctypes.data, p[2].ctypes.data,
                                p[3].ctypes.data, n, m, m, layout, out.ctypes.data))
    return out


def unpack_ternary(packed: np.ndarray, n: int, m: int, layout: int = LAYOUT_COL4) -> np.ndarray:
    w = np.ascontiguousarray(packed, dtype=np.uint32)
    assert w.nbytes == packed_bytes(n, m, layout)
    out = np.empty((4, n, m), dtype=np.int8)
    _check(_lib.ww_unpack_ternary(w.ctypes.data, n, m, layout, out[0].ctypes.data,
                                  out[1].ctypes.data, out[2].ctypes.data, out[3].ctypes.data, m))
    return out


def repack(packed: np.ndarray, n: int, m: int, src_layout: int, dst_layout: int) -> np.ndarray:
    w = np.ascontiguousarray(packed, dtype=np.uint32)
    assert w.nbytes == packed_bytes(n, m, src_layout)
    out = np.empty(packed_bytes(n, m, dst_layout) // 4, dtype=np.uint32)
    _check(_lib.ww_repack(w.ctypes.data, src_layout, n, m, out.ctypes.data, dst_layout))
    return out


# --------------------------------------------------------------------------- device entry points
def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def pack_ternary_device(planes, bad=None, stream=None, out=None, layout: int = LAYOUT_COL4):
    """(4, n, ld) int8 CUDA tensor -> packed uint8 CUDA tensor of packed_bytes(n, m, layout)
    (COL4 for the CUDA-core kernels, TILE32 for the tensor-core path)."""
    import torch
    assert planes.is_cuda and planes.dtype == torch.int8 and planes.is_contiguous()
    _, n, ld = planes.shape
    m = ld
    nb = packed_bytes(n, m, layout)
    if out is None:
        out = torch.empty(nb, dtype=torch.uint8, device=planes.device)
    if out.numel() * out.element_size() < nb:
        raise ValueError(f"out has {out.numel() * out.element_size()} bytes, needs {nb}")
    _check(_lib.ww_pack_ternary_device_layout(planes.data_ptr(), n, m, ld, layout, out.data_ptr(),
                                              bad.data_ptr() if bad is not None else None,
                                              _stream_ptr(stream)))
    return out


def _check_args(layer: Layer, packed, scales, X, Y, B: int):
    """Marshalling checks the C ABI cannot make on raw pointers: devices, dtypes, inner
    strides and buffer sizes (a view such as Z[:, ::2] or a complex128 tensor would
    otherwise pass the C-side checks and give silently wrong results)."""
    import torch
    for name, t in (("packed", packed), ("scales", scales), ("x", X), ("y", Y)):
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise TypeError(f"{name} must be a CUDA tensor")
    for name, t in (("x", X), ("y", Y)):
        if t.dtype != torch.complex64:
            raise TypeError(f"{name} must be complex64 (got {t.dtype})")
        if t.stride(-1) != 1:
            raise ValueError(f"{name} must have unit inner stride (got {t.stride()})")
    if X.shape[-1] != layer.m or Y.shape[-1] < layer.n:
        raise ValueError(f"x has {X.shape[-1]} columns (m={layer.m}), y {Y.shape[-1]} (n={layer.n})")
    if B > 1 and (X.shape[0] < B or Y.shape[0] < B):
        raise ValueError(f"batch {B} but x {tuple(X.shape)}, y {tuple(Y.shape)}")
    if scales.dtype != torch.float32 or not scales.is_contiguous():
        raise TypeError("scales must be a contiguous float32 tensor")
    need = 4 * layer.n if layer.scale_mode == SCALES_PER_ROW else 4
    if scales.numel() < need:
        raise ValueError(f"scales has {scales.numel()} floats, needs {need}")
    need = packed_bytes(layer.n, layer.m, layer.layout)
    if not packed.is_contiguous() or packed.numel() * packed.element_size() < need:
        raise ValueError(f"packed must be contiguous with >= {need} bytes")


def wl_gemv(layer: Layer, packed, scales, x, y=None, stream=None):
    """y = WL-GEMV(x) for one complex64 CUDA vector x of length m."""
    import torch
    if y is None:
        y = torch.empty(layer.n, dtype=torch.complex64, device=x.device)
    _check_args(layer, packed, scales, x, y, 1)
    L = layer.c()
    _check(_lib.ww_wl_gemv(ctypes.byref(L), packed.data_ptr(), scales.data_ptr(), x.data_ptr(),
                           y.data_ptr(), _stream_ptr(stream)))
    return y


@dataclass
class Ops:
    """ww_ops: fused decode-block ops of ww_wl_gemv_fused (B = 1)."""
    prologue: int = 0
    epilogue: int = 0
    x2: object = None
    gamma: object = None
    eps: float = 1e-5
    residual: object = None
    row0: int = 0
    silu_rows: int = 0

    def c(self) -> _Ops:
        return _Ops(self.prologue, self.epilogue, None if self.x2 is None else self.x2.data_ptr(),
                    None if self.gamma is None else self.gamma.data_ptr(), self.eps,
                    None if self.residual is None else self.residual.data_ptr(), self.row0,
                    self.silu_rows)


def wl_gemv_fused(layer: Layer, packed, scales, x, y=None, ops: Ops | None = None, stream=None):
    """y = epilogue(WL-GEMV(prologue(x))) for one complex64 CUDA vector (ww_wl_gemv_fused)."""
    import torch
    if y is None:
        y = torch.empty(layer.n, dtype=torch.complex64, device=x.device)
    _check_args(layer, packed, scales, x, y, 1)
    for name, t, dt in (("x2", ops and ops.x2, torch.complex64), ("gamma", ops and ops.gamma, torch.float32),
                        ("residual", ops and ops.residual, torch.complex64)):
        if t is not None and (not t.is_cuda or t.dtype != dt or t.stride(-1) != 1):
            raise TypeError(f"{name} must be a unit-stride CUDA {dt} tensor")
    L = layer.c()
    O = ops.c() if ops is not None else None
    _check(_lib.ww_wl_gemv_fused(ctypes.byref(L), packed.data_ptr(), scales.data_ptr(), x.data_ptr(),
                                 y.data_ptr(), ctypes.byref(O) if O is not None else None,
                                 _stream_ptr(stream)))
    return y


GROUP = 4  # ww.h: batches above 4 vectors run as groups of 4, one launch each


def launches_for_batch(B: int) -> int:
    """Kernel launches one ww_wl_gemv_batched call makes for B vectors."""
    return 1 if B <= GROUP else -(-B // GROUP)


def wl_gemv_batched(layer: Layer, packed, scales, X, Y=None, stream=None):
    """Y[b] = WL-GEMV(X[b]) for a (B, m) complex64 CUDA tensor (row stride X.stride(0))."""
    import torch
    B = X.shape[0]
    if Y is None:
        Y = torch.empty((B, layer.n), dtype=torch.complex64, device=X.device)
    if X.dim() != 2 or Y.dim() != 2:
        raise ValueError("X and Y must be 2-D (B, m) / (B, n) tensors")
    _check_args(layer, packed, scales, X, Y, B)
    L = layer.c()
    _check(_lib.ww_wl_gemv_batched(ctypes.byref(L), packed.data_ptr(), scales.data_ptr(),
                                   X.data_ptr(), X.stride(0), Y.data_ptr(), Y.stride(0), B,
                                   _stream_ptr(stream)))
    return Y


# --------------------------------------------------------------------------- sharding / launch
@dataclass(frozen=True)
class Shard:
    world: int
    rank: int
    n: int
    rows_per_rank: int
    n_padded: int
    row_begin: int
    row_end: int
    packed_offset_bytes: int
    packed_bytes: int
    scale_offset_floats: int
    scale_count: int
    y_offset_complex: int


def shard_plan(n: int, m: int, world: int, rank: int) -> Shard:
    s = _Shard()
    _check(_lib.ww_shard_plan(n, m, world, rank, ctypes.byref(s)))
    return Shard(*[getattr(s, f) for f, _ in _Shard._fields_])


def query_launch(layer: Layer, B: int = 1) -> dict:
    li = _LaunchInfo()
    L = layer.c()
    _check(_lib.ww_query_launch(ctypes.byref(L), B, ctypes.byref(li)))
    return {f: getattr(li, f) for f, _ in _LaunchInfo._fields_}


# --------------------------------------------------------------------------- unfused ablation
def wl_gemv_unfused(layer: Layer, planar, scales, x, y=None, acc=None, stream=None):
    """The paper's unfused baseline on the GPU: eight real ternary GEMVs
    (ww_ternary_gemv_plane: planes U_re, U_im, W_re, W_im of a WW_LAYOUT_PLANAR buffer
    against x.re and x.im) plus ww_wl_combine.  Ablation only; the product is wl_gemv."""
    import torch
    n, m = layer.n, layer.m
    if y is None:
        y = torch.empty(n, dtype=torch.complex64, device=x.device)
    if acc is None:
        acc = torch.empty((8, n), dtype=torch.float32, device=x.device)
    s = _stream_ptr(stream)
    for plane in range(4):
        for comp in range(2):
            _check(_lib.ww_ternary_gemv_plane(n, m, planar.data_ptr(), plane, x.data_ptr(), comp,
                                              acc[2 * plane + comp].data_ptr(), layer.flags, s))
    L = layer.c()
    _check(_lib.ww_wl_combine(ctypes.byref(L), acc.data_ptr(), scales.data_ptr(), y.data_ptr(), s))
    return y


# --------------------------------------------------------------------------- program
@dataclass
class Stage:
    """One stage of a persistent program (ww_stage); tensors are CUDA tensors.
    y: list of the gathered complex64 output buffers of every rank (index = rank)."""
    packed: object
    scales: object
    n_local: int
    row0: int
    m: int
    x: object
    y: list
    scale_mode: int = SCALES_PER_ROW
    conv: int = CONV_EQ1
    x2: object = None
    residual: object = None
    gamma: object = None
    eps: float = 1e-5
    prologue: int = PRO_NONE
    epilogue: int = EPI_NONE
    wait: int = 1
    silu_rows: int = 0


def _ptr(t):
    return None if t is None else t.data_ptr()


class Program:
    """ww_program_init / ww_program_run: `stages[r][s]` = stage s of rank rank_base + r.
    ranks_in_launch = len(stages) ranks run in one launch (one GPU); `sync` is a list of
    `world` device tensors of ww_program_sync_bytes() zeroed bytes (rank g's sync words)."""

    def __init__(self, stages, world: int = 1, rank_base: int = 0, sync=None, device=None):
        import torch
        R, S = len(stages), len(stages[0])
        assert all(len(st) == S for st in stages)
        dev = device if device is not None else stages[0][0].x.device
        self.world, self.R, self.S = world, R, S
        nbytes = int(_lib.ww_program_workspace_bytes(S, R))
        self.workspace = torch.empty(nbytes + 128, dtype=torch.uint8, device=dev)
        ws = self.workspace.data_ptr()
        ws_al = (ws + 127) // 128 * 128
        sb = int(_lib.ww_program_sync_bytes())
        if sync is None:
            self._sync_buf = torch.zeros(world * sb + 128, dtype=torch.uint8, device=dev)
            b = (self._sync_buf.data_ptr() + 127) // 128 * 128
            sync_ptrs = [b + g * sb for g in range(world)]
        else:
            self._sync_buf = sync
            sync_ptrs = [t if isinstance(t, int) else t.data_ptr() for t in sync]
        self._keep = []
        arr = (_Stage * (R * S))()
        for r in range(R):
            for s_, st in enumerate(stages[r]):
                c = arr[r * S + s_]
                c.packed, c.scales = _ptr(st.packed), _ptr(st.scales)
                c.n_local, c.row0, c.m = st.n_local, st.row0, st.m
                c.scale_mode, c.conv = st.scale_mode, st.conv
                c.x, c.x2 = _ptr(st.x), _ptr(st.x2)
                for g in range(world):
                    yg = st.y[g]
                    c.y[g] = yg if isinstance(yg, int) else yg.data_ptr()
                c.residual, c.gamma, c.eps = _ptr(st.residual), _ptr(st.gamma), st.eps
                c.prologue, c.epilogue, c.wait, c.silu_rows = (st.prologue, st.epilogue, st.wait,
                                                               st.silu_rows)
                self._keep.append(st)
        sp = (_vp * world)(*sync_ptrs)
        self.prog = _Program()
        _check(_lib.ww_program_init(arr, S, world, rank_base, R, sp, ws_al, ctypes.byref(self.prog)))
        torch.cuda.synchronize(dev)

    def info(self) -> dict:
        return {f: getattr(self.prog, f) for f, _ in _Program._fields_[:12]}

    def run(self, stream=None):
        _check(_lib.ww_program_run(ctypes.byref(self.prog), _stream_ptr(stream)))


def keep_in_l2(tensor, stream=None):
    """ww_stream_keep_in_l2: keep `tensor` persisting in L2 for launches on `stream` (None:
    the current stream); tensor=None clears the window."""
    sp = _stream_ptr(stream)
    if tensor is None:
        _check(_lib.ww_stream_keep_in_l2(sp, None, 0))
    else:
        _check(_lib.ww_stream_keep_in_l2(sp, tensor.data_ptr(), tensor.numel() * tensor.element_size()))


def tc_workspace_bytes(n: int, m: int, B: int) -> int:
    """Bytes of the zero-initialised workspace ww_wl_gemv_batched_tc needs (0: unsupported)."""
    return int(_lib.ww_tc_workspace_bytes(n, m, B))


def wl_gemv_batched_tc(layer: Layer, packed, scales, X, Y=None, workspace=None, stream=None):
    """Y[b] = WL-GEMV(X[b]) on the tensor cores (ww_wl_gemv_batched_tc; 1 <= B <= 16)."""
    import torch
    B = X.shape[0]
    if Y is None:
        Y = torch.empty((B, layer.n), dtype=torch.complex64, device=X.device)
    if X.dim() != 2 or Y.dim() != 2:
        raise ValueError("X and Y must be 2-D (B, m) / (B, n) tensors")
    _check_args(layer, packed, scales, X, Y, B)
    nb = tc_workspace_bytes(layer.n, layer.m, B)
    if nb == 0:
        raise ValueError(f"batch {B} unsupported by the tensor-core path (1..16)")
    if workspace is None or workspace.numel() * workspace.element_size() < nb + 128:
        workspace = torch.zeros(nb + 128, dtype=torch.uint8, device=X.device)  # zeroed (ww.h)
    wp = (workspace.data_ptr() + 127) // 128 * 128
    L = layer.c()
    _check(_lib.ww_wl_gemv_batched_tc(ctypes.byref(L), packed.data_ptr(), scales.data_ptr(),
                                      X.data_ptr(), X.stride(0), Y.data_ptr(), Y.stride(0), B, wp,
                                      _stream_ptr(stream)))
    return Y


def tcv_workspace_bytes(n: int, m: int, B: int = 1) -> int:
    """Bytes of the zero-initialised workspace ww_wl_gemv_tc needs (0: unsupported B)."""
    return int(_lib.ww_tcv_workspace_bytes(n, m, B))


def tcv_workspace(n: int, m: int, B: int = 1, device=None):
    """A zeroed workspace for ww_wl_gemv_tc (every call leaves it zeroed again)."""
    import torch
    nb = tcv_workspace_bytes(n, m, B)
    if nb == 0:
        raise ValueError(f"batch {B} unsupported by ww_wl_gemv_tc (1..4)")
    return torch.zeros(nb, dtype=torch.uint8, device=device if device is not None else "cuda")


def wl_gemv_tc(layer: Layer, packed, scales, X, Y=None, workspace=None, stream=None):
    """Y[b] = WL-GEMV(X[b]) on the tensor cores (ww_wl_gemv_tc; TILE32 weights, 1 <= B <= 4).
    X may be a (B, m) or an (m,) complex64 CUDA tensor; Y has the same rank."""
    import torch
    vec = X.dim() == 1
    X2 = X.view(1, -1) if vec else X
    B = X2.shape[0]
    if Y is None:
        Y = torch.empty((B, layer.n) if not vec else (layer.n,), dtype=torch.complex64, device=X.device)
    Y2 = Y.view(1, -1) if Y.dim() == 1 else Y
    if X2.dim() != 2 or Y2.dim() != 2:
        raise ValueError("X and Y must be (B, m) / (B, n) or 1-D tensors")
    if layer.layout != LAYOUT_TILE32:
        raise ValueError("wl_gemv_tc needs layout LAYOUT_TILE32")
    _check_args(layer, packed, scales, X2, Y2, B)
    nb = tcv_workspace_bytes(layer.n, layer.m, B)
    if nb == 0:
        raise ValueError(f"batch {B} unsupported by the tensor-core path (1..4)")
    if workspace is None:
        workspace = tcv_workspace(layer.n, layer.m, B, X.device)
    if workspace.numel() * workspace.element_size() < nb or workspace.data_ptr() % 16:
        raise ValueError(f"workspace needs {nb} zeroed, 16-B aligned bytes")
    L = layer.c()
    _check(_lib.ww_wl_gemv_tc(ctypes.byref(L), packed.data_ptr(), scales.data_ptr(), X2.data_ptr(),
                              X2.stride(0), Y2.data_ptr(), Y2.stride(0), B, workspace.data_ptr(),
                              _stream_ptr(stream)))
    return Y


# --------------------------------------------------------------------------- lookup path (LUT81)
def lut81_packed_bytes(n: int, m: int) -> int:
    return int(_lib.ww_lut81_packed_bytes(n, m))


def lut81_from_planar(planar: np.ndarray, n: int, m: int) -> np.ndarray:
    """App. H planar words -> WW_LAYOUT_LUT81 bytes (host, ww_lut81_from_planar)."""
    planar = np.ascontiguousarray(planar, dtype=np.uint32)
    if planar.size * 4 != packed_bytes(n, m, LAYOUT_PLANAR):
        raise ValueError("planar buffer has the wrong size")
    out = np.empty(lut81_packed_bytes(n, m), np.uint8)
    _check(_lib.ww_lut81_from_planar(n, m, planar.ctypes.data, out.ctypes.data))
    return out


def lut81_to_planar(lut: np.ndarray, n: int, m: int) -> np.ndarray:
    """WW_LAYOUT_LUT81 bytes -> App. H planar words (host, ww_lut81_to_planar)."""
    lut = np.ascontiguousarray(lut, dtype=np.uint8)
    if lut.size != lut81_packed_bytes(n, m):
        raise ValueError("LUT81 buffer has the wrong size")
    out = np.empty(packed_bytes(n, m, LAYOUT_PLANAR) // 4, np.uint32)
    _check(_lib.ww_lut81_to_planar(n, m, lut.ctypes.data, out.ctypes.data))
    return out


def pack_lut81(planes: np.ndarray) -> np.ndarray:
    """(4, n, m) int8 planes -> WW_LAYOUT_LUT81 bytes (host: App. H words, then the index bytes)."""
    _, n, m = planes.shape
    return lut81_from_planar(pack_ternary(planes, LAYOUT_PLANAR), n, m)


def wl_gemv_lut(layer: Layer, packed, scales, x, y=None, stream=None):
    """y = WL-GEMV(x) by ternary subset-sum lookup (ww_wl_gemv_lut; LUT81 weights, B = 1)."""
    import torch
    if layer.layout != LAYOUT_LUT81:
        raise ValueError("wl_gemv_lut needs layout LAYOUT_LUT81")
    if y is None:
        y = torch.empty(layer.n, dtype=torch.complex64, device=x.device)
    for name, t, dt in (("x", x, torch.complex64), ("y", y, torch.complex64), ("scales", scales, torch.float32)):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dt or not t.is_contiguous():
            raise TypeError(f"{name} must be a contiguous CUDA tensor of {dt}")
    if x.numel() != layer.m or y.numel() != layer.n:
        raise ValueError("x / y length does not match the layer")
    if scales.numel() != (4 * layer.n if layer.scale_mode == SCALES_PER_ROW else 4):
        raise ValueError("scales size does not match the layer")
    if not packed.is_cuda or packed.numel() * packed.element_size() < lut81_packed_bytes(layer.n, layer.m):
        raise ValueError("packed buffer too small for WW_LAYOUT_LUT81")
    L = layer.c()
    _check(_lib.ww_wl_gemv_lut(ctypes.byref(L), packed.data_ptr(), scales.data_ptr(), x.data_ptr(),
                               y.data_ptr(), _stream_ptr(stream)))
    return y
