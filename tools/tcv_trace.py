"""Per-phase timeline of wl_tcv_kernel (CTAs 0 and grid/2, globaltimer ns) for one launch
of each config-4 stage shape (tools only; ww_debug_tcv_trace is not part of the ABI)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_20913_b200 as ww  # noqa: E402
import ww_inputs as wi  # noqa: E402

EV = {0: "entry", 1: "setup", 2: "x: pdl_wait done", 3: "x: max done", 4: "x: limbs done (bready)",
      5: "mma: bready seen", 6: "mma: first unit issued", 7: "mma: last unit issued",
      8: "dec w4: first unit stored", 9: "dec w4: last unit stored",
      21: "x: landed in smem", 23: "x: decoder w4 joined", 22: "x: max reduced", 19: "x: tid0 item start", 30: "x: tid0 comp0 done", 31: "x: tid0 comp1 done", 28: "x: tid0 limbs done", 29: "x: tid0 fence done", 10: "epi seg0 dfull", 11: "epi seg0 done", 12: "epi seg1 dfull", 13: "epi seg1 done",
      14: "epi seg2 dfull", 15: "epi seg2 done", 16: "epi seg3 dfull", 20: "exit"}


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    buf = torch.zeros(64, dtype=torch.int64, device="cuda")
    for n, m in [(2048, 2048), (2048, 5504), (11008, 2048)]:
        planes = torch.empty((4, n, m), dtype=torch.int8, device="cuda")
        for q in range(4):
            wi.codes_device(1, q, n, m, planes[q])
        t32 = ww.pack_ternary_device(planes, layout=ww.LAYOUT_TILE32)
        sc = torch.rand((n, 4), device="cuda") * 0.09 + 0.01
        L = ww.Layer(n, m, ww.LAYOUT_TILE32)
        X = torch.randn((B, m), dtype=torch.complex64, device="cuda")
        ws = ww.tcv_workspace(n, m, B)
        for it in range(3):
            buf.zero_()
            ww._lib.ww_debug_tcv_trace(ctypes.c_void_p(buf.data_ptr() if it == 2 else 0))
            ww.wl_gemv_tc(L, t32, sc, X, workspace=ws)
            torch.cuda.synchronize()
        ww._lib.ww_debug_tcv_trace(ctypes.c_void_p(0))
        t = buf.cpu().view(2, 32)
        print(f"  cta0 cycles of the E computation: {int(t[0, 17])}")
        print(f"  cta0 cycles: mma waits on afull {int(t[0, 24])}, decoder w4 waits: full {int(t[0, 25])} "
              f"aempty {int(t[0, 26])} over {int(t[0, 27])} stages")
        print(f"--- {n}x{m} B={B}")
        t0 = int(t[0, 0])
        for ev, name in EV.items():
            a, b = int(t[0, ev]), int(t[1, ev])
            fa = f"{(a - t0) / 1e3:8.2f}" if a else "       -"
            fb = f"{(b - t0) / 1e3:8.2f}" if b else "       -"
            print(f"  {name:28s} cta0 {fa} us   mid {fb} us")


if __name__ == "__main__":
    main()
