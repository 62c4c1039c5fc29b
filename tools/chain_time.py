"""Per-launch cost of a PDL-chained CUDA graph of WL-GEMV launches (development aid, not the
bench contract), split into its parts with the library's debug switches
(ww_debug_set_flags: 1 = skip griddepcontrol.wait, 2 = skip the accumulation):

  pdl        the product configuration (graph, PDL, every launch waits for its predecessor)
  nopdl      graph without PDL (full launch serialisation)
  nowait     PDL without the wait: launches overlap freely (an unsafe lower bound on
             dependency cost -- only legal here because every launch has its own x and y)
  nocompute  PDL + wait but no accumulation: launch, dependency, x staging, weight stream,
             reductions and epilogue only
  l2pf       PDL + a bulk L2 prefetch of each CTA's weights at kernel start

Weights rotate over R replicas >= 4x L2 (HBM-cold).  The debug switches need a build with
-DWW_DEBUG_FLAGS=1: run with WW_LIB_OVERRIDE=build/libww_dbg.so (tools/build.py --variant dbg
WW_DEBUG_FLAGS=1); with the product library only the pdl / nopdl modes are meaningful.
Usage: chain_time.py [--product] [n m ...]."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_20913_b200 as ww  # noqa: E402
import ww_inputs as wi  # noqa: E402

ww._lib.ww_debug_set_flags.argtypes = [ctypes.c_int]
if os.environ.get("WW_FORCE_CP_ASYNC"):  # stage x with per-thread cp.async instead of TMA
    ww._lib.ww_debug_force_cp_async(1)


def chain(n, m, B=1, mode="pdl", l2=126 * 2**20, reps=15):
    nbytes = ww.packed_bytes(n, m)
    R = max(2, int(np.ceil(4 * l2 / nbytes)))
    planes = torch.empty((4, n, m), dtype=torch.int8, device="cuda")
    for p in range(4):
        wi.codes_device(1, p, n, m, planes[p])
    base = ww.pack_ternary_device(planes)
    del planes
    W = torch.empty((R, nbytes), dtype=torch.uint8, device="cuda")
    W[:] = base
    sc = torch.rand((n, 4), device="cuda") * 0.09 + 0.01
    X = torch.randn((R, B, m), dtype=torch.complex64, device="cuda")
    Y = torch.empty((R, B, n), dtype=torch.complex64, device="cuda")
    flags = 0 if mode == "nopdl" else ww.FLAG_PDL
    dbg = {"pdl": 0, "nopdl": 0, "nowait": 1, "nocompute": 2, "l2pf": 8,
           "nocompute_l2pf": 10}[mode]
    L = ww.Layer(n, m, flags=flags)
    s = torch.cuda.Stream()
    ww._lib.ww_debug_set_flags(dbg)
    try:
        with torch.cuda.stream(s):
            for r in range(R):
                ww.wl_gemv_batched(L, W[r], sc, X[r], Y[r], stream=s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for r in range(R):
                    ww.wl_gemv_batched(L, W[r], sc, X[r], Y[r], stream=s)
    finally:
        ww._lib.ww_debug_set_flags(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    with torch.cuda.stream(s):  # replay on the stream the events are recorded on
        g.replay()
        torch.cuda.synchronize()
        for _ in range(reps):
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / R)
    return float(np.median(ts))


if __name__ == "__main__":
    print(torch.cuda.get_device_name(), flush=True)
    shapes = [(2048, 2048), (5504, 2048), (2048, 5504), (6144, 2048), (11008, 2048)]
    nums = [v for v in sys.argv[1:] if not v.startswith("--")]
    if len(nums) >= 2:
        a = [int(v) for v in nums]
        shapes = list(zip(a[0::2], a[1::2]))
    if "--scan" in sys.argv:  # noqa: SIM102
        shapes = [(148 * k, m) for m in (2048, 5504) for k in (1, 4, 14, 28, 56)]
    for n, m in shapes:
        codes = 4 * n * m
        modes = ("pdl", "nopdl") if "--product" in sys.argv else (
            "pdl", "nopdl", "nowait", "nocompute", "l2pf", "nocompute_l2pf")
        res = {md: chain(n, m, mode=md) for md in modes}
        rate = codes / (res["pdl"] * 1e-6) / 148 / 1.965e9
        print(f"n={n:6d} m={m:5d}: " + "  ".join(f"{k} {v:6.2f} us" for k, v in res.items())
              + f"   ({rate:.1f} codes/clk/SM at pdl)", flush=True)
