"""One launch of ww_wl_gemv_lut per config-4 stage shape (after a warm-up pass), for ncu."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_20913_b200 as ww

g = torch.Generator(device="cuda").manual_seed(0)
cases = []
for n, m in [(6144, 2048), (2048, 2048), (11008, 2048), (2048, 5504)]:
    T = (m + 511) // 512
    w = torch.randint(0, 81, (n * T * 512,), dtype=torch.uint8, device="cuda", generator=g)
    cases.append((ww.Layer(n, m, ww.LAYOUT_LUT81), w, torch.rand(n, 4, device="cuda"),
                  torch.randn(m, dtype=torch.complex64, device="cuda"),
                  torch.empty(n, dtype=torch.complex64, device="cuda")))
for _ in range(2):
    for L, w, sc, x, y in cases:
        ww.wl_gemv_lut(L, w, sc, x, y)
    torch.cuda.synchronize()
