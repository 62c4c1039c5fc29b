"""NEXT-3: per-operation breakdown of one decode block on B200 in the style of the paper's
App. J table (SPEC BreakdownRow).  The block's non-GEMV ops are fused
into the GEMV launches (RMSNorm and SiLU(gate) (.) up as prologues, residual adds and SiLU
as epilogues), so an op's time is the increment of its launch over the same launch without
the op: each stage kind is timed as a CUDA graph of its 32 launches (HBM-cold weights, PDL),
once in the plain chain and once in the decode-block chain, in one process.

    python tools/appj_breakdown.py        # prints the table; profiles/r02/appj_breakdown.txt
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_20913_b200.stack import WLStack, block_gammas  # noqa: E402


def per_kind_us(stack, reps=10):
    s = torch.cuda.Stream()
    kinds = {}
    for i, st in enumerate(stack.stages):
        kinds.setdefault(st.name, []).append(i)
    with torch.cuda.stream(s):  # real inputs for the chained buffers
        stack.step(s)
    torch.cuda.synchronize()
    out = {}
    for name, idx in kinds.items():
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for i in idx:
                stack.launch(i, s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in idx:
                stack.launch(i, s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            g.replay()
            a.record(s)
            for _ in range(reps):
                g.replay()
            b.record(s)
        torch.cuda.synchronize()
        out[name] = a.elapsed_time(b) * 1e3 / (reps * len(idx))
    return out


def main():
    layers = 32
    plain = per_kind_us(WLStack(layers=layers, seed=0))
    gam = [tuple(torch.from_numpy(g).cuda() for g in p) for p in block_gammas(0, layers, 2048)]
    block = per_kind_us(WLStack(layers=layers, seed=0, chain="block", gammas=gam))
    rows = [("RMSNorm (attention)", block["qkv"] - plain["qkv"], False),
            ("Q/K/V projection (WL-GEMV)", plain["qkv"], True),
            ("Attention (identity over one token, S:502)", 0.0, False),
            ("O projection (WL-GEMV)", plain["o"], True),
            ("Residual add (after O)", block["o"] - plain["o"], True),
            ("RMSNorm (MLP) + SiLU of the gate rows", block["gateup"] - plain["gateup"], False),
            ("Gate+Up projection (WL-GEMV)", plain["gateup"], True),
            ("SiLU(gate) (.) up + residual add (after down)", block["down"] - plain["down"], False),
            ("Down projection (WL-GEMV)", plain["down"], True)]
    total = sum(r[1] for r in rows)
    gemv = sum(r[1] for r in rows if "WL-GEMV" in r[0])
    print(f"{torch.cuda.get_device_name()}: one decode block (complex d = 2048, d_ff = 5504, B = 1), "
          "us per layer, fused ops timed as increments of their launch")
    print(f"{'Operation':48s} {'Time (us)':>10s} {'Fraction':>9s}  Mul-free?")
    for name, t, mf in rows:
        print(f"{name:48s} {t:10.2f} {100 * t / total:8.1f}%  {'yes' if mf else 'no'}")
    print(f"{'Total per layer':48s} {total:10.2f}     100%")
    print(f"{'Fused WL-GEMV fraction':48s} {gemv:10.2f} {100 * gemv / total:8.1f}%  yes")
    print(f"(paper, Xeon 8558P, 48 threads: 942 us per layer, GEMV 855 us = 90.8%, P:705-731; "
          f"x {layers} layers = {layers * total / 1e3:.3f} ms per token here)")


if __name__ == "__main__":
    main()
