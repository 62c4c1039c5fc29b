"""Quick per-shape kernel timing (development aid, not the bench contract):
HBM-cold via rotating weight replicas (>= 4x L2) inside a CUDA graph."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_20913_b200 as ww  # noqa: E402
import ww_inputs as wi  # noqa: E402


def time_shape(n, m, B=1, reps_graph=20, flags=0, l2_bytes=126 * 2**20, warm=False):
    nbytes = ww.packed_bytes(n, m)
    R = max(1, int(np.ceil(4 * l2_bytes / nbytes)))
    if warm:  # one weight set, launched R times back to back (L2-resident)
        R_launch, R = R, 1
    planes = torch.empty((4, n, m), dtype=torch.int8, device="cuda")
    for p in range(4):
        wi.codes_device(1, p, n, m, planes[p])
    base = ww.pack_ternary_device(planes)
    del planes
    reps = torch.empty((R, nbytes), dtype=torch.uint8, device="cuda")
    reps[:] = base
    sc = torch.rand((n, 4), device="cuda") * 0.09 + 0.01
    X = torch.randn((B, m), dtype=torch.complex64, device="cuda")
    Y = torch.empty((B, n), dtype=torch.complex64, device="cuda")
    L = ww.Layer(n, m, flags=flags)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        NL = R_launch if warm else R
        for r in range(NL):
            ww.wl_gemv_batched(L, reps[r % R], sc, X, Y, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for r in range(NL):
                ww.wl_gemv_batched(L, reps[r % R], sc, X, Y, stream=s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps_graph):
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / NL)
    us = float(np.median(ts))
    algo = nbytes + 8 * m * B + 8 * n * B + 16 * n
    codes = 4 * n * m * B
    return us, algo / us * 1e-3, codes / us * 1e-6, R


if __name__ == "__main__":
    print(torch.cuda.get_device_name(), flush=True)
    if "--scan" in sys.argv:
        for m in (2048, 5504):
            for k in (1, 2, 4, 8, 14, 16, 28, 32, 48):
                n = 148 * k
                for flags in (0, ww.FLAG_PDL):
                    us, gbs, tcodes, R = time_shape(n, m, 1, flags=flags, warm=True)
                    print(f"m={m} rows/SM={k:3d} pdl={flags}: {us:8.2f} us  "
                          f"({tcodes*1e12/148/1.965e9:5.1f} codes/clk/SM)", flush=True)
        sys.exit(0)
    if "--split" in sys.argv:  # whole rows (stream / row-by-row producer) vs split halves
        lib = ww._lib
        for (n, m) in ((6144, 2048), (2048, 2048), (11008, 2048), (2048, 5504), (5504, 2048)):
            for name, split, rows in (("whole", 0, 0), ("whole-rows", 0, 1), ("split", 1, 0)):
                lib.ww_debug_force_split(split)
                lib.ww_debug_force_rows(rows)
                r = [time_shape(n, m, 1, flags=ww.FLAG_PDL)[0] for _ in range(3)]
                print(f"n={n} m={m} {name:10s}: {min(r):.3f} us (runs {', '.join(f'{v:.3f}' for v in r)})",
                      flush=True)
        lib.ww_debug_force_split(-1)
        lib.ww_debug_force_rows(0)
        sys.exit(0)
    if "--warm" in sys.argv:
        for (n, m) in ((2048, 2048), (5504, 2048), (2048, 5504)):
            for flags in (0, ww.FLAG_PDL):
                for warm in (False, True):
                    us, gbs, tcodes, R = time_shape(n, m, 1, flags=flags, warm=warm)
                    print(f"n={n} m={m} pdl={flags} {'L2-warm ' if warm else 'HBM-cold'}: {us:.2f} us "
                          f"({tcodes*1e12/148/1.965e9:.1f} codes/clk/SM)", flush=True)
        sys.exit(0)
    for (n, m) in ((2048, 2048), (5504, 2048), (2048, 5504)):
        for flags in (0, ww.FLAG_PDL):
            us, gbs, tcodes, R = time_shape(n, m, 1, flags=flags)
            print(f"n={n} m={m} B=1 pdl={flags}: {us:.2f} us  {gbs:.0f} GB/s  {tcodes:.2f} Tcodes/s "
                  f"({tcodes*1e12/148/1.965e9:.1f} codes/clk/SM @1965)  R={R}", flush=True)
    for B in (2, 4, 8, 16):
        us, gbs, tcodes, R = time_shape(2048, 5504, B)
        print(f"down B={B}: {us:.2f} us  {gbs:.0f} GB/s  {tcodes:.2f} T code-vectors/s", flush=True)
