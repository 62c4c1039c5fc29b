"""Per-stage timeline of the persistent program kernel (tools only): globaltimer stamps per
CTA and stage -- start, readiness poll done, x landed, prologue done, producer done issuing,
warp 0 / warp 8 / warp 15 rows done -- summarised per stage kind (medians over CTAs and
layers, us relative to the stage's earliest start)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_20913_b200 as ww  # noqa: E402
from paper_2604_20913_b200.stack import WLStack, block_gammas, program_stages  # noqa: E402


def main(chain="plain", layers=32):
    st = WLStack(layers=layers, seed=0)
    gam = None
    if chain == "block":
        gam = [tuple(torch.from_numpy(g).cuda() for g in p) for p in block_gammas(0, layers, 2048)]
    prog = ww.Program([program_stages(st, [st], chain, gam)])
    info = prog.info()
    S, G = info["nstages"], info["grid"]
    buf = torch.zeros(G * S * 8, dtype=torch.int64, device="cuda")
    for _ in range(3):
        prog.run()
    torch.cuda.synchronize()
    ww._lib.ww_debug_program_trace(ctypes_ptr(buf))
    prog.run()
    torch.cuda.synchronize()
    ww._lib.ww_debug_program_trace(None)
    t = buf.view(G, S, 8).cpu().numpy().astype(np.float64)
    t0 = t[:, :, 0].min(axis=0)  # per stage: earliest CTA start
    names = ["start", "polled", "x_ready", "w0_fullwait", "producer_done", "w0_done", "w15_done", "w8_done"]
    print(f"chain={chain} stages={S} grid={G} nslot={info['nslot']} slot={info['slot_bytes']} "
          f"total={(t[:, -1, 5].max() - t[:, 0, 0].min()) / 1e3:.1f} us")
    for k, kind in enumerate(("qkv", "o", "gateup", "down")):
        idx = list(range(k, S, 4))
        rel = (t[:, idx, :] - t0[idx][None, :, None]) / 1e3
        rel[:, :, 3] = t[:, idx, 3] / 1e3  # a duration (ns of full-barrier waits), not a stamp
        med = np.median(rel, axis=(0, 1))
        mx = np.median(rel.max(axis=0), axis=0)
        dur = np.median((t0[[i + 1 for i in idx if i + 1 < S]] - t0[[i for i in idx if i + 1 < S]]) / 1e3)
        print(f"{kind:7s} stage-to-stage {dur:6.2f} us | median CTA: " +
              " ".join(f"{n}={v:6.2f}" for n, v in zip(names, med)))
        print(f"{'':7s} {'':25s}| slowest CTA: " + " ".join(f"{n}={v:6.2f}" for n, v in zip(names, mx)))


def ctypes_ptr(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


if __name__ == "__main__":
    ww._lib.ww_debug_program_trace.argtypes = [__import__("ctypes").c_void_p]
    main(sys.argv[1] if len(sys.argv) > 1 else "plain")
