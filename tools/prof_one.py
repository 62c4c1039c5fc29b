"""Run a few launches of one WL-GEMV shape (for ncu -k regex:wl_gemv -s <warm> -c <n>)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_20913_b200 as ww  # noqa: E402
import ww_inputs as wi  # noqa: E402

n, m, B = (int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (2048, 5504, 1)
launches = int(sys.argv[4]) if len(sys.argv) >= 5 else 5
planes = torch.empty((4, n, m), dtype=torch.int8, device="cuda")
for p in range(4):
    wi.codes_device(1, p, n, m, planes[p])
packed = ww.pack_ternary_device(planes)
sc = torch.rand((n, 4), device="cuda") * 0.09 + 0.01
X = torch.randn((B, m), dtype=torch.complex64, device="cuda")
L = ww.Layer(n, m)
for _ in range(launches):
    Y = ww.wl_gemv_batched(L, packed, sc, X)
torch.cuda.synchronize()
print("ok", n, m, B, ww.query_launch(L, B))
