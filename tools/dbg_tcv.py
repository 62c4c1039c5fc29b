import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2604_20913_b200 as ww, oracle as orc, ww_inputs as wi
from _wl import LayerCase
n, m = int(sys.argv[1]), int(sys.argv[2])
case = LayerCase(n, m, seed=11)
ref = case.oracle(orc.CONV_EQ1)[0]
pk = torch.from_numpy(ww.pack_ternary(case.planes, ww.LAYOUT_TILE32).view(np.uint8)).cuda()
sc = torch.from_numpy(case.scales).cuda(); x = torch.from_numpy(case.x).cuda()
L = ww.Layer(n, m, ww.LAYOUT_TILE32)
y = ww.wl_gemv_tc(L, pk, sc, x).cpu().numpy()[0]
err = np.abs(y - ref) / (np.abs(ref) + 1e-3)
S = (m + 63) // 64; T = (n + 31) // 32; U = T * S; G = min(148, U)
own = lambda u: ((u + 1) * G - 1) // U
bad = [t for t in range(T) if err[t*32:(t+1)*32].max() > 1e-3]
print("bad tiles", len(bad), "of", T)
for t in bad[:10]:
    print(t, "c0", own(t*S), "c1", own((t+1)*S-1), "maxerr", err[t*32:(t+1)*32].max(), "rows bad", int((err[t*32:(t+1)*32] > 1e-3).sum()))
