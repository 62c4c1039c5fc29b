"""Per-warp timeline of one WL-GEMV launch (build/libww_trace.so, -DWW_TRACE): globaltimer
stamps at kernel entry (0), before/after griddepcontrol.wait (1, 2), after issuing the x
staging (3), then at the start of every sweep and after every unit's epilogue (4..29), the
SM id (30) and the warp's exit (31).  Prints event percentiles and the spread of per-CTA
finish times (by SM id).  Usage: trace_kernel.py [n m ...]; WW_DBG=<flags> as chain_time.py."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import build  # noqa: E402
import paper_2604_20913_b200 as ww  # noqa: E402
import ww_inputs as wi  # noqa: E402

_tp = os.path.join(ROOT, "build", "libww_trace.so")
lib = ctypes.CDLL(_tp if os.path.exists(_tp) else build.build_trace())
lib.ww_debug_set_trace.argtypes = [ctypes.c_void_p]
lib.ww_debug_set_flags.argtypes = [ctypes.c_int]
lib.ww_debug_set_flags(int(os.environ.get("WW_DBG", "0")))  # chain_time.py's debug switches
lib.ww_wl_gemv_batched.restype = ctypes.c_int
lib.ww_wl_gemv_batched.argtypes = [ctypes.POINTER(ww._Layer), ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]

shapes = [(2048, 5504), (2048, 2048), (11008, 2048)]
_args = [v for v in sys.argv[1:] if not v.startswith("--")]
if len(_args) >= 2:
    a = [int(v) for v in _args]
    shapes = list(zip(a[0::2], a[1::2]))
for (n, m) in ([] if "--chain" in sys.argv else shapes):
    planes = torch.empty((4, n, m), dtype=torch.int8, device="cuda")
    for p in range(4):
        wi.codes_device(1, p, n, m, planes[p])
    packed = ww.pack_ternary_device(planes)
    sc = torch.rand((n, 4), device="cuda") * 0.09 + 0.01
    X = torch.randn((1, m), dtype=torch.complex64, device="cuda")
    Y = torch.empty((1, n), dtype=torch.complex64, device="cuda")
    tr = torch.zeros(148 * 32 * 32, dtype=torch.int64, device="cuda")
    L = ww.Layer(n, m).c()
    s = torch.cuda.current_stream().cuda_stream
    for it in range(3):
        if it == 2:
            lib.ww_debug_set_trace(tr.data_ptr())
        rc = lib.ww_wl_gemv_batched(ctypes.byref(L), packed.data_ptr(), sc.data_ptr(), X.data_ptr(),
                                    m, Y.data_ptr(), n, 1, s)
        assert rc == 0
        torch.cuda.synchronize()
    lib.ww_debug_set_trace(None)
    t = tr.cpu().numpy().reshape(148, 32, 32).astype(np.int64)
    valid = t[:, :, 0] > 0
    t0 = t[valid][:, 0].min()
    print(f"== n={n} m={m}: warps traced {valid.sum()}")
    for ev in list(range(0, 12)) + [31]:
        col = t[:, :, ev][valid]
        col = col[col > 0] - t0
        if col.size:
            print(f"  ev{ev:2d}: min {col.min()/1e3:7.2f} us  median {np.median(col)/1e3:7.2f}  "
                  f"max {col.max()/1e3:7.2f}")
    # per-CTA finish (last warp exit) and start, by SM id
    cta_end = np.array([(t[c, :, 31][valid[c]].max() - t0) / 1e3 for c in range(148)
                        if valid[c].any()])
    cta_beg = np.array([(t[c, :, 0][valid[c]].min() - t0) / 1e3 for c in range(148)
                        if valid[c].any()])
    smid = np.array([t[c, :, 30][valid[c]][0] for c in range(148) if valid[c].any()])
    print(f"  CTA finish: min {cta_end.min():.2f} p10 {np.percentile(cta_end, 10):.2f} median "
          f"{np.median(cta_end):.2f} p90 {np.percentile(cta_end, 90):.2f} max {cta_end.max():.2f} us")
    dur = cta_end - cta_beg
    print(f"  CTA duration: min {dur.min():.2f} median {np.median(dur):.2f} max {dur.max():.2f} us")
    order = np.argsort(smid)
    buckets = [f"{int(smid[order][i]):3d}-{int(smid[order][min(i + 15, len(order) - 1)]):3d}:"
               f"{dur[order][i:i + 16].mean():6.2f}" for i in range(0, len(order), 16)]
    print("  mean CTA duration by SM id (16 SMs per bucket): " + "  ".join(buckets))


def chain(shapes, reps=2):
    """--chain n1 m1 n2 m2 ...: one PDL graph of launches of the listed shapes (distinct
    weights, x and y per launch, like the decode stack); per launch: when its CTAs start,
    clear griddepcontrol.wait, start their first sweep, finish sweeping, and exit."""
    bufs = []
    for (n, m) in shapes:
        planes = torch.empty((4, n, m), dtype=torch.int8, device="cuda")
        for p in range(4):
            wi.codes_device(7, p, n, m, planes[p])
        bufs.append((n, m, ww.pack_ternary_device(planes), torch.rand((n, 4), device="cuda") * 0.09 + 0.01,
                     torch.randn((1, m), dtype=torch.complex64, device="cuda"),
                     torch.empty((1, n), dtype=torch.complex64, device="cuda")))
    K = len(bufs)
    tr = torch.zeros(K * 148 * 32 * 32, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    flags = int(os.environ.get("WW_DBG", "0"))

    def launch_all():
        for k, (n, m, pk, sc, X, Y) in enumerate(bufs):
            lib.ww_debug_set_flags((k << 8) | flags)
            L = ww.Layer(n, m, flags=ww.FLAG_PDL).c()
            rc = lib.ww_wl_gemv_batched(ctypes.byref(L), pk.data_ptr(), sc.data_ptr(), X.data_ptr(),
                                        m, Y.data_ptr(), n, 1, s.cuda_stream)
            assert rc == 0
    lib.ww_debug_set_trace(tr.data_ptr())
    with torch.cuda.stream(s):
        launch_all()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            launch_all()
        for _ in range(reps):
            tr.zero_()
            g.replay()
        torch.cuda.synchronize()
    lib.ww_debug_set_trace(None)
    lib.ww_debug_set_flags(flags)
    t = tr.cpu().numpy().reshape(K, 148, 32, 32).astype(np.int64)
    t0 = t[:, :, :, 0][t[:, :, :, 0] > 0].min()
    print(f"== chain of {K} launches (times in us from the first CTA start)")
    prev_end = None
    for k in range(K):
        v = t[k, :, :, 0] > 0
        ev = lambda e: (t[k, :, :, e][v & (t[k, :, :, e] > 0)] - t0) / 1e3
        beg, w2, s4, s29, s31 = ev(0), ev(2), ev(4), ev(29), ev(31)
        n, m = bufs[k][0], bufs[k][1]
        gap = f" gap(prev last exit -> first wait release) {w2.min() - prev_end:6.2f}" if prev_end is not None else ""
        print(f"  L{k} {n}x{m}: CTA start {beg.min():7.2f}..{beg.max():7.2f}  wait released "
              f"{w2.min():7.2f}..{w2.max():7.2f}  first sweep {s4.min():7.2f}..{s4.max():7.2f}  "
              f"sweeps done {s29.min():7.2f}..{s29.max():7.2f}  exit {s31.min():7.2f}..{s31.max():7.2f}{gap}")
        prev_end = s31.max()
        # per CTA: last warp's sweeps-done time, and its spread over the CTA's warps
        cta_last = np.array([(t[k, c, :, 29][t[k, c, :, 29] > 0].max() - t0) / 1e3
                             for c in range(148) if (t[k, c, :, 29] > 0).any()])
        cta_first = np.array([(t[k, c, :, 29][t[k, c, :, 29] > 0].min() - t0) / 1e3
                              for c in range(148) if (t[k, c, :, 29] > 0).any()])
        print(f"       CTA last-warp done: min {cta_last.min():7.2f} median {np.median(cta_last):7.2f} "
              f"max {cta_last.max():7.2f};  within-CTA warp spread median "
              f"{np.median(cta_last - cta_first):5.2f} max {np.max(cta_last - cta_first):5.2f}")


if __name__ == "__main__" and "--chain" in sys.argv:
    chain(shapes)
