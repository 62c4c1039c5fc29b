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
if len(sys.argv) >= 3:
    a = [int(v) for v in sys.argv[1:]]
    shapes = list(zip(a[0::2], a[1::2]))
for (n, m) in shapes:
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
