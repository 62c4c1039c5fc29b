"""A few tensor-core batched calls (tools only: a short command for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_20913_b200 as ww  # noqa: E402
import ww_inputs as wi  # noqa: E402

n, m, B = 2048, 5504, int(sys.argv[1]) if len(sys.argv) > 1 else 16
planes = torch.empty((4, n, m), dtype=torch.int8, device="cuda")
for q in range(4):
    wi.codes_device(1, q, n, m, planes[q])
packed = ww.pack_ternary_device(planes, layout=ww.LAYOUT_TILE32)
sc = torch.rand((n, 4), device="cuda") * 0.09 + 0.01
X = torch.randn((B, m), dtype=torch.complex64, device="cuda")
ws = torch.zeros(ww.tc_workspace_bytes(n, m, B) + 256, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ww.wl_gemv_batched_tc(ww.Layer(n, m, ww.LAYOUT_TILE32), packed, sc, X, workspace=ws)
torch.cuda.synchronize()
print("ok")
if "--trace" in sys.argv:
    import ctypes
    import numpy as np
    tr = torch.zeros(64 * 8 * 8, dtype=torch.int64, device="cuda")
    ww._lib.ww_debug_tc_trace.argtypes = [ctypes.c_void_p]
    ww._lib.ww_debug_tc_trace(tr.data_ptr())
    ww.wl_gemv_batched_tc(ww.Layer(n, m, ww.LAYOUT_TILE32), packed, sc, X, workspace=ws)
    torch.cuda.synchronize()
    ww._lib.ww_debug_tc_trace(None)
    t = tr.view(-1, 8).cpu().numpy().astype(np.float64)
    nk = int((t[:60, 0] > 0).sum())
    t0 = t[0, 0]
    print(f"kernel entry {t[60, 0] - t0:.0f}, epilogue start {t[60, 1] - t0:.0f}, epilogue end {t[60, 2] - t0:.0f} (cycles from block 0 decode start)")
    print("per K-block (SM cycles): decode start, slot free, decoded (warp 0) | MMA warp: start, A ready, A+limbs ready, committed")
    for kb in list(range(0, min(nk, 10))) + [nk - 1]:
        print(kb, " ".join(f"{(t[kb, e] - t0):8.0f}" for e in (0, 1, 2, 6, 5, 3, 4)))
