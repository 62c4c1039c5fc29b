"""NEXT-2 ablation: the fused WL-GEMV against the paper's unfused baseline on
B200 -- eight real ternary GEMVs (one per plane and component of x, each re-streaming its
plane) + one combine -- on the BASELINE layer shapes, B = 1,
HBM-cold (R weight replicas >= 4x L2 cycled inside one CUDA graph, PDL on).  Prints us per
layer and the fusion speedup."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_20913_b200 as ww  # noqa: E402
import ww_inputs as wi  # noqa: E402

L2 = 126 * 2**20


def timed(fn, R, reps=10):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for r in range(R):
            fn(r, s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for r in range(R):
                fn(r, s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / R)
    return float(np.median(ts))


def main():
    js = "--json" in sys.argv
    out = {}
    if not js:
        print(torch.cuda.get_device_name(), flush=True)
    for (n, m) in ((2048, 2048), (5504, 2048), (2048, 5504)):
        nb = ww.packed_bytes(n, m)
        R = max(2, int(np.ceil(4 * L2 / nb)))
        planes = wi.planes(5, n, m)
        col4 = torch.from_numpy(ww.pack_ternary(planes, ww.LAYOUT_COL4).view(np.uint8)).cuda()
        planar = torch.from_numpy(ww.pack_ternary(planes, ww.LAYOUT_PLANAR).view(np.uint8)).cuda()
        Wc = torch.empty((R, nb), dtype=torch.uint8, device="cuda")
        Wc[:] = col4
        Wp = torch.empty((R, nb), dtype=torch.uint8, device="cuda")
        Wp[:] = planar
        del col4, planar
        sc = torch.from_numpy(wi.scales(5, n, True, 0.01, 0.1)).cuda()
        X = torch.from_numpy(wi.activations(5, m, R)).cuda()
        Y = torch.empty((R, n), dtype=torch.complex64, device="cuda")
        acc = torch.empty((8, n), dtype=torch.float32, device="cuda")
        Lf = ww.Layer(n, m, flags=ww.FLAG_PDL)
        Lu = ww.Layer(n, m, ww.LAYOUT_PLANAR, flags=ww.FLAG_PDL)
        fused = timed(lambda r, s: ww.wl_gemv(Lf, Wc[r], sc, X[r], Y[r], stream=s), R)
        unfused = timed(lambda r, s: ww.wl_gemv_unfused(Lu, Wp[r], sc, X[r], Y[r], acc, stream=s), R)
        out[f"{n}x{m}"] = round(unfused, 3)
        if not js:
            print(f"complex {n}x{m}: fused {fused:7.2f} us   unfused 8x real + combine "
                  f"{unfused:7.2f} us   fusion speedup {unfused / fused:.2f}x", flush=True)
        del Wc, Wp
    if js:
        import json
        print(json.dumps(out))


if __name__ == "__main__":
    main()
