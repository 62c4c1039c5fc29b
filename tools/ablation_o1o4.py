"""NEXT-2: the fused WL-GEMV with one of the paper's
optimisations removed at a time, on B200, B = 1, HBM-cold (weight replicas >= 4x L2 cycled
in one CUDA graph, PDL on):
  O1 mask reuse        -> WW_ABL_NO_O1: the re and im paths decode their own predicates
  O2 input reuse       -> WW_ABL_NO_O2: every plane re-loads its x pair from shared memory
  O4 register accums   -> WW_ABL_NO_O4: accumulators spilled / reloaded every 16 columns
  fusion (one pass)    -> the unfused path: 8 real ternary GEMVs + combine (ww_unfused.cu)
(O3 has no ablation: the sign swap is folded into the epilogue signs at zero cost in both
designs, R4.)  Each variant is a separate build of the same sources
(tools/build.py --variant), loaded in its own process.

    python tools/ablation_o1o4.py            # builds nothing; expects build/libww_abl_*.so
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = ((2048, 2048), (5504, 2048), (2048, 5504))
VARIANTS = (("fused", ""), ("no_O1", "build/libww_abl_NO_O1.so"),
            ("no_O2", "build/libww_abl_NO_O2.so"), ("no_O4", "build/libww_abl_NO_O4.so"))

CHILD = r'''
import json, sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tools!r})
import torch
import paper_2604_20913_b200 as ww
from quick_time import time_shape
out = {{}}
for n, m in {shapes!r}:
    us, gbs, tcodes, R = time_shape(n, m, 1, flags=ww.FLAG_PDL)
    out[f"{{n}}x{{m}}"] = round(us, 3)
print(json.dumps(out))
'''


def run_variant(lib):
    env = dict(os.environ)
    if lib:
        env["WW_LIB_OVERRIDE"] = os.path.join(ROOT, lib)
    code = CHILD.format(root=ROOT, tools=os.path.join(ROOT, "tools"), shapes=SHAPES)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def run_unfused():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ablation_unfused.py"),
                        "--json"], capture_output=True, text=True, timeout=900)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    res = {name: run_variant(lib) for name, lib in VARIANTS}
    res["unfused_8x"] = run_unfused()
    print(json.dumps(res))
    base = res["fused"]
    print(f"{'variant':12s} " + " ".join(f"{k:>14s}" for k in base))
    for name, r in res.items():
        print(f"{name:12s} " + " ".join(
            f"{r[k]:8.2f} ({r[k] / base[k]:4.2f}x)" for k in base))


if __name__ == "__main__":
    main()
