"""Build every native artefact in-tree (no JIT cache): the product library
libww.so (sm_100a CUDA + host C++), the input generator libraries and the
C oracle.  Called by ``__graft_entry__.build()``; also runnable directly.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# IEEE fp32: no fast-math, no FTZ (R7)
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-ftz=false",
                     "-prec-div=true", "-prec-sqrt=true", "-fmad=false", "-cudart", "static"]

PKG = os.path.join(ROOT, "paper_2604_20913_b200")
CSRC = os.path.join(PKG, "csrc")


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=ROOT)


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build_oracle(force=False):
    src = os.path.join(ROOT, "oracle", "oracle.c")
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    deps = [src, os.path.join(ROOT, "oracle", "oracle.h")]
    if force or _stale(out, deps):
        _run(["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-Wall",
              "-Wno-unknown-pragmas", "-o", out, src, "-lm"])
    # the same source with OpenMP over rows (CPU baseline's all-core mode; same results)
    out_omp = os.path.join(ROOT, "oracle", "liboracle_omp.so")
    if force or _stale(out_omp, deps):
        _run(["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-Wall",
              "-fopenmp", "-o", out_omp, src, "-lm"])


def build_inputs(force=False):
    d = os.path.join(ROOT, "ww_inputs")
    out = os.path.join(d, "libww_inputs.so")
    srcs = [os.path.join(d, "gen.c"), os.path.join(d, "gen.h")]
    if force or _stale(out, srcs):
        _run(["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-Wall",
              "-o", out, srcs[0], "-lm"])
    out2 = os.path.join(d, "libww_inputs_cuda.so")
    src2 = os.path.join(d, "gen_device.cu")
    if force or _stale(out2, [src2]):
        _run([NVCC] + NVCC_FLAGS + ["-shared", "-o", out2, src2])


def product_sources():
    srcs = []
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".cu", ".cc", ".cuh", ".h")):
            srcs.append(os.path.join(CSRC, f))
    return srcs


def build_product(force=False):
    out = os.path.join(PKG, "libww.so")
    srcs = product_sources() + [os.path.join(ROOT, "include", "ww.h")]
    if not (force or _stale(out, srcs)):
        return
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in product_sources():
        if not s.endswith((".cu", ".cc")):
            continue
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        if s.endswith(".cu"):
            _run([NVCC] + NVCC_FLAGS + ["-Xptxas", "-v", "-I", os.path.join(ROOT, "include"),
                                        "-c", "-o", o, s])
        else:
            _run(["g++", "-std=c++17", "-O2", "-fPIC", "-Wall", "-I",
                  os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", "-c", "-o", o, s])
        objs.append(o)
    _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", out] + objs)


def build_trace():
    """libww_trace.so: the product sources with -DWW_TRACE (per-warp timestamps); tools only."""
    out = os.path.join(ROOT, "build", "libww_trace.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = [s for s in product_sources() if s.endswith((".cu", ".cc"))]
    _run([NVCC] + NVCC_FLAGS + ["-DWW_TRACE", "-I", os.path.join(ROOT, "include"), "-shared",
                                "-o", out] + srcs)
    return out


def build_variant(name, defines):
    """build/libww_<name>.so: the product sources with extra -D flags (kernel A/B timing via
    WW_LIB_OVERRIDE in tools only)."""
    out = os.path.join(ROOT, "build", f"libww_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = [s for s in product_sources() if s.endswith((".cu", ".cc"))]
    _run([NVCC] + NVCC_FLAGS + [f"-D{d}" for d in defines] +
         ["-I", os.path.join(ROOT, "include"), "-shared", "-o", out] + srcs)
    return out


def build_cpu_alg1(force=False):
    """cpu_alg1/libww_cpu.so: the paper's AVX-512 + BMI2 Algorithm 1 (NEXT-4 CPU baseline).
    Compiled for x86-64 with the AVX-512 code in target-attributed functions (runtime check)."""
    d = os.path.join(ROOT, "cpu_alg1")
    out = os.path.join(d, "libww_cpu.so")
    srcs = [os.path.join(d, "ww_cpu.c"), os.path.join(d, "ww_cpu.h")]
    if force or _stale(out, srcs):
        _run(["gcc", "-std=c11", "-O3", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
              "-Wall", "-o", out, srcs[0]])


def build_all(force=False):
    build_oracle(force)
    build_cpu_alg1(force)
    build_inputs(force)
    build_product(force)


if __name__ == "__main__":
    if "--variant" in sys.argv:  # --variant NAME DEF1 DEF2 ...
        i = sys.argv.index("--variant")
        build_variant(sys.argv[i + 1], sys.argv[i + 2:])
    else:
        build_all(force="--force" in sys.argv)
