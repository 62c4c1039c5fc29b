"""Time the tensor-core WL-GEMV (ww_wl_gemv_tc, TILE32) against the predicated-FADD2 kernel
(ww_wl_gemv_batched, COL4) on the config-4 stage shapes: HBM-cold weight replicas, one CUDA
graph of R back-to-back PDL launches per measurement (tools only)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_20913_b200 as ww  # noqa: E402
import ww_inputs as wi  # noqa: E402

SHAPES = [(6144, 2048), (2048, 2048), (11008, 2048), (2048, 5504)]


def timed(fn, R, s, reps=5):
    with torch.cuda.stream(s):
        for r in range(R):
            fn(r)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for r in range(R):
                fn(r)
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / R)
    return float(np.median(ts))


def main():
    import ctypes
    ww._lib.ww_debug_tcv_flags(ctypes.c_int(int(os.environ.get("TCV_DBG", "0"))))
    batches = [int(b) for b in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1"])]
    shapes = SHAPES if len(sys.argv) < 3 else [tuple(int(v) for v in a.split("x")) for a in sys.argv[2].split(",")]
    L2 = 126 * 2**20
    s = torch.cuda.Stream()
    for n, m in shapes:
        nb = ww.packed_bytes(n, m)
        R = max(2, int(np.ceil(4 * L2 / nb)))
        planes = torch.empty((4, n, m), dtype=torch.int8, device="cuda")
        for q in range(4):
            wi.codes_device(1, q, n, m, planes[q])
        col4 = ww.pack_ternary_device(planes)
        t32 = ww.pack_ternary_device(planes, layout=ww.LAYOUT_TILE32)
        del planes
        rc = torch.empty((R, col4.numel()), dtype=torch.uint8, device="cuda")
        rc[:] = col4
        rt = torch.empty((R, t32.numel()), dtype=torch.uint8, device="cuda")
        rt[:] = t32
        sc = torch.rand((n, 4), device="cuda") * 0.09 + 0.01
        Lc = ww.Layer(n, m, ww.LAYOUT_COL4, flags=ww.FLAG_PDL)
        Lt = ww.Layer(n, m, ww.LAYOUT_TILE32, flags=ww.FLAG_PDL)
        for B in batches:
            X = torch.randn((B, m), dtype=torch.complex64, device="cuda")
            Y = torch.empty((B, n), dtype=torch.complex64, device="cuda")
            ws = ww.tcv_workspace(n, m, B)
            torch.cuda.synchronize()  # the zeroing (default stream) before the timed stream
            t_tc = timed(lambda r: ww.wl_gemv_tc(Lt, rt[r], sc, X, Y, ws, stream=s), R, s)
            if os.environ.get("TCV_DEBUG"):
                print("tc done", t_tc, flush=True)
            t_fa = timed(lambda r: ww.wl_gemv_batched(Lc, rc[r], sc, X, Y, stream=s), R, s)
            byt = nb + 8 * m * B
            print(f"{n:5d}x{m:5d} B={B}: tensor-core {t_tc:7.2f} us ({byt / t_tc * 1e-3:6.0f} GB/s, "
                  f"{byt / t_tc * 1e-3 / 6561.3:5.1%} HBM)   FADD2 {t_fa:7.2f} us   x{t_fa / t_tc:4.2f}",
                  flush=True)
        del rc, rt


if __name__ == "__main__":
    main()
