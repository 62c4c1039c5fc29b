"""Per-block timeline of wl_tc_kernel's CTA 0 (tools only; SM cycles by event: 0-2 decode,
3-6 MMA warp, 60 entry / epilogue start / end, 61 epilogue steps).  The trace buffer is pinned
host memory, so even a launch that never finishes can be inspected from the host.
    python tools/tc_trace_pinned.py [big]"""
import ctypes, sys, time, threading, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2604_20913_b200 as ww, ww_inputs as wi
from _wl import LayerCase
def _t32(c):
    c.device(ww, torch)
    c.packed_d = torch.from_numpy(ww.pack_ternary(c.planes, ww.LAYOUT_TILE32).view(np.uint8)).cuda()
    return c


case = _t32(LayerCase(300, 517, seed=3, B=8))
buf = torch.zeros(2 * 64 * 8, dtype=torch.int64).pin_memory()
ww._lib.ww_debug_tc_trace(ctypes.c_void_p(buf.data_ptr()))
L = ww.Layer(case.n, case.m, ww.LAYOUT_TILE32)
n_arg = sys.argv[1:] and sys.argv[1]
if n_arg == "big":
    case = _t32(LayerCase.from_spec(wi.C3B, seed=5, B=8))
    L = ww.Layer(case.n, case.m, ww.LAYOUT_TILE32)
y = ww.wl_gemv_batched_tc(L, case.packed_d, case.scales_d, case.x_d)
done = []
th = threading.Thread(target=lambda: (torch.cuda.synchronize(), done.append(1)), daemon=True)
th.start()
th.join(5)
print("kernel finished:", bool(done), flush=True)
T = buf.numpy().reshape(2, 64, 8)
for c in range(2):
    t = T[c]
    print("CTA", c, "(clock64 is per SM: compare within a CTA only)")
    for kb in list(range(3)) + [int(np.nonzero(t[:59].any(axis=1))[0].max())] + [60, 61]:
        if t[kb].any():
            print(" ", kb, list(int(v - t[60][0]) for v in t[kb] if v))
print("done-check", flush=True)
import os; os._exit(0)
