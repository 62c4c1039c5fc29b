"""Time ww_wl_gemv_lut against ww_wl_gemv on the config-4 stage shapes (HBM-cold: each timed
graph chains 32 different weight sets per shape, as bench.py's per_shape_us does)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2604_20913_b200 as ww

SHAPES = [("qkv", 6144, 2048), ("o", 2048, 2048), ("gateup", 11008, 2048), ("down", 2048, 5504)]
NL = 32


def rand_lut(n, m, g):
    T = (m + 511) // 512
    return torch.randint(0, 81, (n * T * 512,), dtype=torch.uint8, device="cuda", generator=g)


def rand_col4(n, m, g):
    # random valid COL4 bytes: 2-bit fields never 0b11
    W = (m + 15) // 16
    a = torch.randint(0, 3, (n * W * 16, 4), dtype=torch.uint8, device="cuda", generator=g)
    return (a[:, 0] | (a[:, 1] << 2) | (a[:, 2] << 4) | (a[:, 3] << 6)).contiguous()


def time_graph(fn, iters=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn(s)
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.synchronize()
        e0.record(s)
        for _ in range(iters):
            g.replay()
        e1.record(s)
        s.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us per graph


def main():
    pdl = ww.FLAG_PDL if "--nopdl" not in sys.argv else 0
    g = torch.Generator(device="cuda").manual_seed(0)
    tot = {"lut": 0.0, "fadd2": 0.0}
    for name, n, m in SHAPES:
        x = torch.randn(m, dtype=torch.complex64, device="cuda")
        sc = torch.rand(n, 4, device="cuda") * 0.09 + 0.01
        y = torch.empty(n, dtype=torch.complex64, device="cuda")
        wl = [rand_lut(n, m, g) for _ in range(NL)]
        wc = [rand_col4(n, m, g) for _ in range(NL)]
        Ll = ww.Layer(n, m, ww.LAYOUT_LUT81, ww.SCALES_PER_ROW, ww.CONV_EQ1, pdl)
        Lc = ww.Layer(n, m, ww.LAYOUT_COL4, ww.SCALES_PER_ROW, ww.CONV_EQ1, pdl)
        t_l = time_graph(lambda s: [ww.wl_gemv_lut(Ll, w, sc, x, y, stream=s) for w in wl]) / NL
        t_c = time_graph(lambda s: [ww.wl_gemv(Lc, w, sc, x, y, stream=s) for w in wc]) / NL
        gb = n * ((m + 511) // 512) * 512 / 1e3
        print(f"{name:7s} {n:6d} x {m:5d}  lut {t_l:7.2f} us ({gb / t_l:7.1f} GB/s)   fadd2 {t_c:7.2f} us"
              f" ({n * ((m + 15) // 16) * 16 / 1e3 / t_c:7.1f} GB/s)   ratio {t_c / t_l:.2f}", flush=True)
        tot["lut"] += t_l
        tot["fadd2"] += t_c
    print(f"per decoder layer: lut {tot['lut']:.2f} us, fadd2 {tot['fadd2']:.2f} us; per token (x32): "
          f"lut {tot['lut'] * 32 / 1e3:.3f} ms, fadd2 {tot['fadd2'] * 32 / 1e3:.3f} ms")


if __name__ == "__main__":
    main()
