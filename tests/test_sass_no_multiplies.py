"""App. D on B200: the hot loop of the shipped sm_100a kernel contains no
floating-point multiply.  Disassembles libww.so with cuobjdump (CPU only) and inspects
the instructions between the first and last packed-fp32 add of the B = 1 kernel's
accumulation loop; the only FMULs allowed are the 8 scale multiplies of the epilogue,
which sit outside that region."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_20913_b200", "libww.so")
FP_MUL = re.compile(r"\b(FMUL2?|FFMA2?|DMUL|DFMA|HMUL2|FMUL32I|FFMA32I)\b")


def _kernels_sass(name_pat):
    """SASS of every function matching name_pat (both instantiations of a batch size: row
    stream and row-by-row producers)."""
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)
    found = [[ln.split(";")[0].strip() for ln in f.splitlines()
              if re.search(r"/\*[0-9a-f]{4}\*/", ln)] for f in funcs if re.match(name_pat, f)]
    if not found:
        pytest.fail(f"kernel {name_pat} not found in {LIB}")
    return found


def _strip(ln):
    return re.sub(r"^/\*[0-9a-f]+\*/\s*", "", ln)


@pytest.mark.parametrize("B", [1, 4])
def test_accumulation_loop_has_no_fp_multiply(B):
    for k in _kernels_sass(rf"_ZN\S*wl_gemv_kernelILi{B}E"):
        _check_loop(B, [_strip(l) for l in k])


def _check_loop(B, sass):
    # accumulation blocks: maximal runs of predicated FADD2 (Eqs. 6-7 as predicated packed
    # adds) no more than 12 instructions apart -- one block per unrolled 64-code chunk body
    idx = [i for i, l in enumerate(sass) if re.match(r"@!?P\d\s+FADD2\b", l)]
    blocks, start = [], idx[0]
    for a, b in zip(idx, idx[1:] + [None]):
        if b is None or b - a > 12:
            blocks.append((start, a))
            start = b
    big = [(a, b) for a, b in blocks if sum(1 for i in idx if a <= i <= b) >= 128 * B]
    assert big, "expected a block of >= 128*B predicated FADD2 (64 codes x 2 per chunk)"
    for a, b in big:
        region = sass[a:b + 1]
        bad = [l for l in region if FP_MUL.search(l)]
        # HFMA2 Rx, -RZ, RZ, c, c is ptxas' constant-materialisation idiom, not a multiply
        bad += [l for l in region if re.search(r"\bHFMA2\b", l) and "-RZ, RZ" not in l]
        assert not bad, bad[:5]


def test_scale_multiplies_exist_only_in_epilogue():
    for k in _kernels_sass(r"_ZN\S*wl_gemv_kernelILi1E"):
        _check_epilogue([_strip(l) for l in k])


def _check_epilogue(sass):
    fmul = [i for i, l in enumerate(sass) if re.search(r"\bFMUL\b", l)]
    fadd2 = [i for i, l in enumerate(sass) if re.match(r"@!?P\d\s+FADD2\b", l)]
    assert fmul, "the epilogue's scale multiplies (P:1002-1011) should be FMULs"
    # every FMUL lies outside the [first, last] span of some contiguous accumulation block:
    # i.e. no FMUL between two predicated FADD2 that are within 8 instructions of each other
    for i in fmul:
        before = [j for j in fadd2 if j < i]
        after = [j for j in fadd2 if j > i]
        assert not (before and after and after[0] - before[-1] <= 8), sass[i]


def test_program_kernel_accumulation_loop_has_no_fp_multiply():
    # the persistent program kernel (ww_program_*) runs the same sweep from shared memory
    for k in _kernels_sass(r"_ZN\S*wl_program_kernel"):
        _check_loop(1, [_strip(l) for l in k])
        _check_epilogue([_strip(l) for l in k])


def test_fused_ops_multiplies_stay_outside_the_loop():
    # the decode-block prologue (RMSNorm, product) and the epilogue (1/rms, SiLU) multiply;
    # the accumulation blocks of every B = 1 kernel still do not
    for pat in (r"_ZN\S*wl_gemv_kernelILi1E", r"_ZN\S*wl_program_kernel"):
        for k in _kernels_sass(pat):
            s = [_strip(l) for l in k]
            assert sum(1 for l in s if re.search(r"\bFMUL\b", l)) > 8  # ops present
            _check_loop(1, s)


def test_lookup_kernel_has_no_fp_multiply_before_the_epilogue():
    """wl_lut_kernel (ww_wl_gemv_lut): the table build and the lookup sweep are adds and
    subtracts only; every floating-point multiply sits after the last lookup (the 8 scale
    multiplies of the row epilogue), and the sweep really is one PRMT + one
    LDS.64 + one FADD2 per 4 codes (16 of each per 128-bit weight load)."""
    for k in _kernels_sass(r"_ZN\S*wl_lut_kernel"):
        sass = [_strip(l) for l in k]
        lds = [i for i, l in enumerate(sass) if re.search(r"\bLDS\.64\b", l)]
        assert len(lds) >= 16 * 8, "expected >= 16 lookups per ring slot"
        mul = [i for i, l in enumerate(sass) if FP_MUL.search(l)]
        mul += [i for i, l in enumerate(sass) if re.search(r"\bHFMA2\b", l) and "-RZ, RZ" not in l]
        assert mul, "the epilogue's scale multiplies should be FMULs"
        # lookup runs: LDS.64 no more than 24 instructions apart (the sweeps; ptxas places the
        # row epilogue between the two sweep instantiations, so the check is per run)
        runs, start = [], lds[0]
        for a, b in zip(lds, lds[1:] + [None]):
            if b is None or b - a > 24:
                runs.append((start, a))
                start = b
        assert sum(1 for a, b in runs if sum(1 for i in lds if a <= i <= b) >= 16) >= 2
        for a, b in runs:
            assert not [sass[i] for i in mul if a <= i <= b], (a, b)
            region = sass[a:b + 1]
            assert not any(re.match(r"@!?P\d\s+FADD2\b", l) for l in region), "no predicated adds here"
        n_prmt = sum(1 for l in sass if re.search(r"\bPRMT\b", l))
        n_add2 = sum(1 for l in sass if re.search(r"\bFADD2\b", l))
        assert n_add2 >= len(lds) and n_prmt >= len(lds)
