"""Time the batched variant (config 5, down shape) on the tensor-core path vs the predicated
FADD2 kernel: HBM-cold weight replicas in one CUDA graph (tools only)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_20913_b200 as ww  # noqa: E402
import ww_inputs as wi  # noqa: E402


def main(n=2048, m=5504, batches=(1, 2, 4, 8, 16)):
    L2 = 126 * 2**20
    nb = ww.packed_bytes(n, m)
    R = max(1, int(np.ceil(4 * L2 / nb)))
    planes = torch.empty((4, n, m), dtype=torch.int8, device="cuda")
    for q in range(4):
        wi.codes_device(1, q, n, m, planes[q])
    base = ww.pack_ternary_device(planes)
    t32 = ww.pack_ternary_device(planes, layout=ww.LAYOUT_TILE32)  # the tensor-core path's layout
    del planes
    reps = torch.empty((R, nb), dtype=torch.uint8, device="cuda")
    reps[:] = base
    rept = torch.empty((R, t32.numel()), dtype=torch.uint8, device="cuda")
    rept[:] = t32
    Lt = ww.Layer(n, m, ww.LAYOUT_TILE32)
    sc = torch.rand((n, 4), device="cuda") * 0.09 + 0.01
    L = ww.Layer(n, m)
    s = torch.cuda.Stream()

    def run(fn):
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
            for _ in range(5):
                a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                g.replay()
                b_.record(s)
                b_.synchronize()
                ts.append(a.elapsed_time(b_) * 1e3 / R)
        return float(np.median(ts))

    for B in batches:
        X = torch.randn((B, m), dtype=torch.complex64, device="cuda")
        Y = torch.empty((B, n), dtype=torch.complex64, device="cuda")
        ws = torch.zeros(ww.tc_workspace_bytes(n, m, B) + 256, dtype=torch.uint8, device="cuda")
        t_tc = run(lambda r: ww.wl_gemv_batched_tc(Lt, rept[r], sc, X, Y, ws, stream=s))
        t_fa = run(lambda r: ww.wl_gemv_batched(L, reps[r], sc, X, Y, stream=s)) if B <= 16 else float("nan")
        bytes_ = nb + 8 * m * B
        print(f"{n}x{m} B={B:2d}: tensor-core {t_tc:8.2f} us ({bytes_ / t_tc * 1e-3:7.0f} GB/s)   "
              f"predicated FADD2 {t_fa:8.2f} us   speedup {t_fa / t_tc:5.2f}x", flush=True)


if __name__ == "__main__":
    main()
