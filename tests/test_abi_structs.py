"""The ctypes mirrors of ww.h's structs (ww_layer, ww_shard, ww_launch_info, ww_ops,
ww_stage, ww_program) match the C layout: a tiny C program compiled against include/ww.h
prints sizeof / offsetof, compared with the binding's ctypes.Structure (CPU only)."""
import ctypes
import os
import shutil
import subprocess
import tempfile

import pytest

import paper_2604_20913_b200 as ww

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKS = [("ww_layer", ww._Layer, ["n", "m", "layout", "scale_mode", "conv", "flags"]),
          ("ww_shard", ww._Shard, ["world", "rank", "n", "rows_per_rank", "row_begin",
                                   "packed_offset_bytes", "y_offset_complex"]),
          ("ww_launch_info", ww._LaunchInfo, ["grid", "block", "smem_bytes", "path"]),
          ("ww_ops", ww._Ops, ["prologue", "epilogue", "x2", "gamma", "eps", "residual", "row0",
                               "silu_rows"]),
          ("ww_stage", ww._Stage, ["packed", "scales", "n_local", "row0", "m", "scale_mode", "conv",
                                   "x", "x2", "y", "residual", "gamma", "eps", "prologue",
                                   "epilogue", "wait", "silu_rows"]),
          ("ww_program", ww._Program, ["nstages", "world", "grid", "smem_bytes", "nslot",
                                       "has_mul", "workspace", "sync"])]


def test_struct_layouts_match_c():
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "ww.h"', "int main(void) {"]
    for cname, _, fields in CHECKS:
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f in fields:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "s.c"), os.path.join(d, "s")
        open(src, "w").write("\n".join(lines))
        subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), "-o", exe, src])
        got = dict(l.split() for l in subprocess.check_output([exe], text=True).splitlines())
    for cname, ct, fields in CHECKS:
        assert int(got[cname]) == ctypes.sizeof(ct), cname
        for f in fields:
            assert int(got[f"{cname}.{f}"]) == getattr(ct, f).offset, (cname, f)
