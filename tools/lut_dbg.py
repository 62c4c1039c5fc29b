"""Debug helper: one ww_wl_gemv_lut launch per shape, each in its own process with
CUDA_LAUNCH_BLOCKING=1, so a faulting shape is reported without taking the others down."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import torch
    import paper_2604_20913_b200 as ww
    n, m = int(sys.argv[1]), int(sys.argv[2])
    T = (m + 511) // 512
    w = torch.full((n * T * 512,), 40, dtype=torch.uint8, device="cuda")
    y = ww.wl_gemv_lut(ww.Layer(n, m, ww.LAYOUT_LUT81), w, torch.ones(n, 4, device="cuda"),
                       torch.ones(m, dtype=torch.complex64, device="cuda"))
    torch.cuda.synchronize()
    print("ok", n, m, float(y.abs().max()))
else:
    for n, m in [(1, 128), (16, 512), (16, 1024), (64, 1024), (148, 1024), (2, 2048), (148, 2048), (2048, 2048), (4096, 1024)]:
        r = subprocess.run([sys.executable, __file__, str(n), str(m)], capture_output=True, text=True,
                           env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"))
        print(n, m, r.stdout.strip() or r.stderr.strip().splitlines()[-1][:150], flush=True)
