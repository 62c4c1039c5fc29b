"""Small launches for compute-sanitizer: C2, C3b and C5 (B = 16) through
the C ABI with both x-staging paths (TMA and the per-thread cp.async fallback), PDL on, plus
(--program) a 2-layer persistent program (plain and decode-block chains).  Checks the
results against the fp64 oracle so a run that 'passes' the sanitizer also computed right.

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py [--program]
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as orc  # noqa: E402
import paper_2604_20913_b200 as ww  # noqa: E402
import ww_inputs as wi  # noqa: E402
from _wl import LayerCase, assert_parity  # noqa: E402


def single_layers():
    cases = [("C2", wi.C2, 1), ("C3b", wi.C3B, 1), ("C5 B=16", wi.C3B, 16)]
    for name, spec, B in cases:
        case = LayerCase.from_spec(spec, seed=1, B=B).device(ww, torch)
        ref = case.oracle(orc.CONV_EQ1)
        for force in (0, 1):
            ww._lib.ww_debug_force_cp_async(force)
            try:
                y = case.gpu(ww, torch, ww.CONV_EQ1, flags=ww.FLAG_PDL)
            finally:
                ww._lib.ww_debug_force_cp_async(0)
            assert_parity(y, ref, case)
            print(f"{name}: {'cp.async' if force else 'TMA'} staging ok", flush=True)


def programs():
    from paper_2604_20913_b200.stack import WLStack, block_gammas, program_stages
    st = WLStack(layers=2, seed=0)
    ref = WLStack(layers=2, seed=0)
    ref.step()
    torch.cuda.synchronize()
    ww.Program([program_stages(st, [st], "plain")]).run()
    torch.cuda.synchronize()
    for a, b in zip(st.Y, ref.Y):
        assert torch.equal(a, b)
    print("program plain: ok", flush=True)
    gam = [tuple(torch.from_numpy(g).cuda() for g in p) for p in block_gammas(0, 2, 2048)]
    ww.Program([program_stages(st, [st], "block", gam)]).run()
    torch.cuda.synchronize()
    assert all(torch.isfinite(torch.view_as_real(y)).all() for y in st.Y)
    print("program block: ok", flush=True)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    single_layers()
    if "--program" in sys.argv:
        programs()
    print("sanitize cases done", flush=True)
