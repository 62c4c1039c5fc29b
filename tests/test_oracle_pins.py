"""Pins of the C fp64 oracle against what the paper and mathematics fix
(not against itself).  CPU only.

Each test cites the passage that fixes the expected value:
  P:n = PAPER.md line n, S:n = SPEC.md line n, golden = tests/golden/worked_examples.json.
"""
import json
import os

import numpy as np
import pytest

import oracle as orc
import ww_inputs as wi

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")
PLANES = ("U_re", "U_im", "W_re", "W_im")


# ---------------------------------------------------------------- packing (App. H)

def test_pack_slots_spec_examples():
    # S:57-60 / App. H equation
    z = np.zeros(16, np.int8)
    assert orc.pack_slots(z) == 0x00000000
    t = z.copy(); t[0] = 1
    assert orc.pack_slots(t) == 0x00000002          # bit 2k+1 for +1 at k=0
    t = z.copy(); t[0] = -1; t[1] = 1
    assert orc.pack_slots(t) == 0x00000009          # bit 0 + bit 3
    assert orc.pack_slots(np.ones(16, np.int8)) == 0xAAAAAAAA
    assert orc.pack_slots(-np.ones(16, np.int8)) == 0x55555555
    t = z.copy(); t[15] = 1
    assert orc.pack_slots(t) == 0x80000000          # bit 31 = slot 15 positive


def test_unpack_slots_examples_and_invalid():
    # inverse of App. H; (1,1) "unused" -> InvalidEncoding
    assert list(orc.unpack_slots(0x0)) == [0] * 16
    t = orc.unpack_slots(0x9)
    assert t[0] == -1 and t[1] == 1 and not t[2:].any()
    for bad in (0x3, 0xC0000000, 0xFFFFFFFF, 0x3 << 14):
        with pytest.raises(orc.OracleError):
            orc.unpack_slots(bad)


def test_decode_masks_eqs_4_5():
    # Eqs. 4-5; examples S:76-79
    assert orc.decode_masks(0x0) == (0, 0)
    assert orc.decode_masks(0xAAAAAAAA) == (0xFFFF, 0)
    assert orc.decode_masks(0x55555555) == (0, 0xFFFF)
    assert orc.decode_masks(0x9) == (0x2, 0x1)
    assert orc.decode_masks(0x80000001) == (0x8000, 0x0001)


def test_pack_plane_example_and_padding():
    # 1x3 [+1,-1,0] -> single word 0x6 with zero-code padding
    w = orc.pack_plane(np.array([[1, -1, 0]], np.int8))
    assert w.shape == (1, 1) and int(w[0, 0]) == 0x6
    # 1x17 -> two words; column 16 lands in slot 0 of word 1
    d = np.zeros((1, 17), np.int8); d[0, 16] = -1
    w = orc.pack_plane(d)
    assert w.shape == (1, 2) and int(w[0, 0]) == 0 and int(w[0, 1]) == 0x1


def _all_patterns(lo, hi):
    """Ternary digit expansion of integers lo..hi-1 into (count, 16) int8 arrays."""
    idx = np.arange(lo, hi, dtype=np.int64)
    out = np.empty((idx.size, 16), np.int8)
    for k in range(16):
        out[:, k] = (idx % 3) - 1
        idx //= 3
    return out


def test_pack_exhaustive_3_pow_16():
    # Every one of the 3^16 = 43,046,721 slot patterns: the word's pext masks equal the
    # +1 / -1 lanes (Eqs. 4-5 applied to App. H), round trip is exact, words are distinct.
    total = 3 ** 16
    step = 3 ** 13
    seen = np.zeros(2 ** 32 // 8, np.uint8)  # bitset over all words
    bit_pos = (1 << (2 * np.arange(16) + 1)).astype(np.uint64)
    bit_neg = (1 << (2 * np.arange(16))).astype(np.uint64)
    for lo in range(0, total, step):
        t = _all_patterns(lo, min(lo + step, total))
        w = orc.pack_plane(t)[:, 0]
        # the defining property of the encoding: bit 2k+1 <=> +1, bit 2k <=> -1
        w64 = w.astype(np.uint64)
        pos = (w64[:, None] & bit_pos[None, :]) != 0
        neg = (w64[:, None] & bit_neg[None, :]) != 0
        assert np.array_equal(pos, t == 1) and np.array_equal(neg, t == -1)
        assert np.array_equal(orc.unpack_plane(w[:, None], 16), t)
        byte, bit = w >> 3, (w & 7).astype(np.uint8)
        assert not np.any(seen[byte] & (1 << bit))
        np.bitwise_or.at(seen, byte, (1 << bit).astype(np.uint8))


def test_decode_masks_matches_lanes_sampled():
    rng = np.random.default_rng(7)
    t = rng.integers(-1, 2, size=(2000, 16)).astype(np.int8)
    w = orc.pack_plane(t)[:, 0]
    for row, word in zip(t, w):
        kp, kn = orc.decode_masks(int(word))
        assert kp == int(sum(1 << k for k in range(16) if row[k] == 1))
        assert kn == int(sum(1 << k for k in range(16) if row[k] == -1))
        assert kp & kn == 0


# ---------------------------------------------------------------- worked examples

def _golden():
    with open(GOLDEN) as f:
        return json.load(f)["examples"]


@pytest.mark.parametrize("ex", _golden(), ids=lambda e: e["name"])
def test_worked_examples(ex):
    n, m = ex["n"], ex["m"]
    planes = np.stack([np.array(ex[p], np.int8) for p in PLANES])
    planar = orc.pack_planar(planes)
    for p, name in enumerate(PLANES):
        assert [int(v) for v in planar[p, :, 0]] == ex["planar_words"][name], name
    scales = (np.array(ex["scales_per_row"], np.float32) if "scales_per_row" in ex
              else np.array(ex["scales_per_tensor"], np.float32))
    x = np.array([complex(a, b) for a, b in ex["x"]], np.complex64)
    for conv, key in ((orc.CONV_EQ1, "y_EQ1"), (orc.CONV_ALG1, "y_ALG1")):
        want = np.array([complex(a, b) for a, b in ex[key]])
        for fn in (orc.wl_direct, orc.wl_embedding):
            got = fn(planar, n, m, scales, x, conv)[0]
            assert np.array_equal(got, want), (fn.__name__, key, got, want)
    y, _ = orc.wl_alg1(planar, n, m, scales, x)
    assert np.array_equal(y, np.array([complex(a, b) for a, b in ex["y_ALG1"]]))


# ---------------------------------------------------------------- closed forms

def _rand_layer(seed, n, m, per_row=True, dist=wi.LLAMA, lo=0.01, hi=0.1):
    planes = wi.planes(seed, n, m, dist)
    scales = wi.scales(seed, n, per_row, lo, hi)
    x = wi.activations(seed, m, 1)[0]
    return planes, orc.pack_planar(planes), scales, x


@pytest.mark.parametrize("conv", [orc.CONV_EQ1, orc.CONV_ALG1])
def test_zero_weights_give_zero(conv):
    n, m = 37, 45
    planar = orc.pack_planar(np.zeros((4, n, m), np.int8))
    x = wi.activations(3, m)[0]
    y = orc.wl_direct(planar, n, m, np.ones((n, 4), np.float32), x, conv)
    assert np.array_equal(y, np.zeros_like(y))


@pytest.mark.parametrize("conv", [orc.CONV_EQ1, orc.CONV_ALG1])
def test_identity_gives_x(conv):
    # U_re = I, others 0, scales 1 -> y = x exactly (Eqs. 2-3 first term)
    n = m = 33
    planes = np.zeros((4, n, m), np.int8)
    planes[0] = np.eye(n, dtype=np.int8)
    x = wi.activations(4, m)[0]
    y = orc.wl_direct(orc.pack_planar(planes), n, m, np.ones(4, np.float32), x, conv)[0]
    assert np.array_equal(y, x.astype(np.complex128))


@pytest.mark.parametrize("conv", [orc.CONV_EQ1, orc.CONV_ALG1])
def test_w_zero_is_textbook_complex_matvec(conv):
    # W = 0 -> y = U x, a plain complex matrix-vector product (zgemv); numpy's BLAS is
    # the independent reference.  U = diag(sUr) U_re + i diag(sUi) U_im.
    n, m = 29, 70
    planes, _, scales, x = _rand_layer(11, n, m)
    planes[2:] = 0
    planar = orc.pack_planar(planes)
    U = scales[:, 0:1].astype(np.float64) * planes[0] + 1j * scales[:, 1:2] * planes[1]
    want = U @ x.astype(np.complex128)
    got = orc.wl_direct(planar, n, m, scales, x, conv)[0]
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13)


def test_real_only_reduces_to_real_gemvs():
    # U_im = W = 0, per-tensor scale s: y = s * U_re x_re + i s * U_re x_im (Eqs. 2-3)
    n, m = 40, 48
    planes, _, _, x = _rand_layer(12, n, m)
    planes[1:] = 0
    s = np.array([0.75, 9.0, 9.0, 9.0], np.float32)
    got = orc.wl_direct(orc.pack_planar(planes), n, m, s, x, orc.CONV_ALG1)[0]
    Ur = planes[0].astype(np.float64)
    np.testing.assert_allclose(got.real, 0.75 * (Ur @ x.real.astype(np.float64)), rtol=1e-13,
                               atol=1e-13)
    np.testing.assert_allclose(got.imag, 0.75 * (Ur @ x.imag.astype(np.float64)), rtol=1e-13,
                               atol=1e-13)


def test_conjugate_term_only():
    # U = 0, W_re = 0, x_im = 0 -> ALG1 y_re = 0, y_im = -s_w_im W_im x_re (Eq. 3)
    n, m = 17, 31
    planes, _, scales, x = _rand_layer(13, n, m)
    planes[0] = planes[1] = planes[2] = 0
    x = x.real.astype(np.float32).astype(np.complex64)
    y = orc.wl_direct(orc.pack_planar(planes), n, m, scales, x, orc.CONV_ALG1)[0]
    want = -scales[:, 3].astype(np.float64) * (planes[3].astype(np.float64) @ x.real.astype(np.float64))
    assert np.all(y.real == 0)
    np.testing.assert_allclose(y.imag, want, rtol=1e-13, atol=1e-15)
    # EQ1 has the opposite sign on that term (P:1435 expanded; R1)
    y1 = orc.wl_direct(orc.pack_planar(planes), n, m, scales, x, orc.CONV_EQ1)[0]
    np.testing.assert_allclose(y1.imag, -want, rtol=1e-13, atol=1e-15)


# ---------------------------------------------------------------- brute force

@pytest.mark.parametrize("n,m", [(1, 1), (5, 16), (16, 17), (64, 63), (33, 128)])
@pytest.mark.parametrize("conv", [orc.CONV_EQ1, orc.CONV_ALG1])
@pytest.mark.parametrize("per_row", [True, False])
def test_direct_equals_real_embedding(n, m, conv, per_row):
    # two independent evaluation paths: complex direct vs the explicit real 2n x 2m map
    planes, planar, scales, x = _rand_layer(n * 1000 + m, n, m, per_row, wi.UNIFORM3, 0.5, 2.0)
    a = orc.wl_direct(planar, n, m, scales, x, conv)
    b = orc.wl_embedding(planar, n, m, scales, x, conv)
    assert np.linalg.norm(a - b) <= 1e-12 * max(np.linalg.norm(a), 1e-30)


@pytest.mark.parametrize("n,m", [(3, 16), (9, 50), (20, 128)])
def test_alg1_literal_equals_direct_alg1(n, m):
    planes, planar, scales, x = _rand_layer(n + 17 * m, n, m)
    y, _ = orc.wl_alg1(planar, n, m, scales, x)
    d = orc.wl_direct(planar, n, m, scales, x, orc.CONV_ALG1)[0]
    assert np.linalg.norm(y - d) <= 1e-12 * np.linalg.norm(d)


def test_brute_force_all_single_codes():
    # 1x1 layers: every (plane, code) combination against the closed-form contribution
    x = np.array([0.75 - 1.5j], np.complex64)
    s = np.array([1.0, 2.0, 4.0, 8.0], np.float32)
    xc = complex(x[0])
    for p in range(4):
        for t in (-1, 1):
            planes = np.zeros((4, 1, 1), np.int8)
            planes[p, 0, 0] = t
            planar = orc.pack_planar(planes)
            unit = [1, 1j, 1, 1j][p] * float(s[p]) * t
            # EQ1: U terms hit x, W terms hit conj(x);  ALG1: (U + conj(W)) x
            eq1 = unit * (xc if p < 2 else xc.conjugate())
            alg1 = (unit if p < 2 else np.conj(unit)) * xc
            assert orc.wl_direct(planar, 1, 1, s, x, orc.CONV_EQ1)[0, 0] == eq1
            assert orc.wl_direct(planar, 1, 1, s, x, orc.CONV_ALG1)[0, 0] == alg1


# ---------------------------------------------------------------- invariants

@pytest.mark.parametrize("conv", [orc.CONV_EQ1, orc.CONV_ALG1])
def test_real_linearity(conv):
    n, m = 23, 64
    _, planar, scales, x = _rand_layer(21, n, m)
    x2 = wi.activations(22, m)[0]
    a, b = 0.5, -2.0
    y = orc.wl_direct(planar, n, m, scales, np.stack([x, x2, (a * x + b * x2).astype(np.complex64)]),
                      conv)
    combo = a * y[0] + b * y[1]
    # x3 was rounded to fp32; compare against the exact combination within that rounding
    assert np.linalg.norm(y[2] - combo) <= 1e-6 * np.linalg.norm(combo)


def test_complex_linearity_separates_conventions():
    # y(i x) = i y(x) holds for ALG1 (complex-linear) and fails for EQ1 whenever W != 0
    n, m = 19, 48
    planes, planar, scales, x = _rand_layer(31, n, m)
    ix = (1j * x).astype(np.complex64)  # exact: swaps and negates components
    for conv in (orc.CONV_ALG1, orc.CONV_EQ1):
        y = orc.wl_direct(planar, n, m, scales, np.stack([x, ix]), conv)
        diff = np.linalg.norm(y[1] - 1j * y[0]) / np.linalg.norm(y[0])
        if conv == orc.CONV_ALG1:
            assert diff <= 1e-13
        else:
            assert diff > 1e-2
    planes[2:] = 0  # W = 0: EQ1 becomes complex-linear too
    p0 = orc.pack_planar(planes)
    y = orc.wl_direct(p0, n, m, scales, np.stack([x, ix]), orc.CONV_EQ1)
    assert np.linalg.norm(y[1] - 1j * y[0]) <= 1e-13 * np.linalg.norm(y[0])


@pytest.mark.parametrize("conv", [orc.CONV_EQ1, orc.CONV_ALG1])
def test_negating_a_code_negates_its_contribution(conv):
    n, m = 8, 40
    rng = np.random.default_rng(5)
    planes, planar, scales, x = _rand_layer(41, n, m)
    y0 = orc.wl_direct(planar, n, m, scales, x, conv)[0]
    for _ in range(12):
        p, i, j = int(rng.integers(4)), int(rng.integers(n)), int(rng.integers(m))
        t = int(planes[p, i, j])
        if t == 0:
            continue
        q = planes.copy()
        q[p, i, j] = -t
        y1 = orc.wl_direct(orc.pack_planar(q), n, m, scales, x, conv)[0]
        xj = complex(x[j])
        s = float(scales[i, p])
        unit = [1, 1j, 1, 1j][p] * s * t
        if conv == orc.CONV_EQ1:
            contrib = unit * (xj if p < 2 else xj.conjugate())
        else:
            contrib = (unit if p < 2 else np.conj(unit)) * xj
        delta = y1 - y0
        assert abs(delta[i] - (-2 * contrib)) <= 1e-12 * (abs(contrib) + np.abs(y0).max())
        others = np.delete(delta, i)
        assert np.all(others == 0)


def test_scale_linearity():
    # scaling one scale by c scales exactly that sub-GEMV's contribution
    n, m = 12, 32
    planes, planar, scales, x = _rand_layer(51, n, m, per_row=False, lo=0.5, hi=2.0)
    for c in range(4):
        s1 = np.zeros(4, np.float32); s1[c] = scales[c]
        s2 = s1.copy(); s2[c] *= 4.0
        y1 = orc.wl_direct(planar, n, m, s1, x, orc.CONV_EQ1)
        y2 = orc.wl_direct(planar, n, m, s2, x, orc.CONV_EQ1)
        assert np.array_equal(y2, 4.0 * y1)


def test_padding_neutrality():
    # extra zero-code columns with zero activations change nothing (bitwise)
    n, m = 10, 20
    planes, planar, scales, x = _rand_layer(61, n, m)
    pp = np.zeros((4, n, 32), np.int8); pp[:, :, :m] = planes
    xp = np.zeros(32, np.complex64); xp[:m] = x
    for conv in (orc.CONV_EQ1, orc.CONV_ALG1):
        a = orc.wl_direct(planar, n, m, scales, x, conv)
        b = orc.wl_direct(orc.pack_planar(pp), n, 32, scales, xp, conv)
        assert np.array_equal(a, b)


def test_invalid_code_rejected_in_eval():
    n, m = 2, 16
    planar = np.zeros((4, n, 1), np.uint32)
    planar[2, 1, 0] = 0x3 << 6  # slot 3 of W_re row 1 = (1,1)
    with pytest.raises(orc.OracleError):
        orc.wl_direct(planar, n, m, np.ones(4, np.float32), np.ones(m, np.complex64))
    with pytest.raises(orc.OracleError):
        orc.wl_alg1(planar, n, m, np.ones(4, np.float32), np.ones(m, np.complex64))


def test_row_subset_matches_full():
    n, m = 50, 64
    _, planar, scales, x = _rand_layer(71, n, m)
    full = orc.wl_direct(planar, n, m, scales, x)
    rows = np.array([49, 0, 17, 17, 3])
    sub = orc.wl_direct(planar, n, m, scales, x, rows=rows)
    assert np.array_equal(sub[0], full[0, rows])


# ---------------------------------------------------------------- op counts (App. D)

def test_op_counts_paper_4096():
    # n = m = 4096 -> 134,217,728 masked add/sub, 32,768 scalar multiplies, 0.024%
    n = m = 4096
    planar = np.zeros((4, n, m // 16), np.uint32)
    y, c = orc.wl_alg1(planar, n, m, np.ones(4, np.float32), np.zeros(m, np.complex64))
    assert c["slots"] == 134_217_728
    assert c["scale_muls"] == 32_768
    assert c["inner_muls"] == 0
    assert round(100 * c["scale_muls"] / c["slots"], 3) == 0.024
    assert not y.any()


def test_op_counts_lane_split():
    # all-zero -> no lanes selected; all +1 one row -> adds only
    n, m = 1, 16
    planes = np.zeros((4, n, m), np.int8)
    planes[0] = 1
    _, c = orc.wl_alg1(orc.pack_planar(planes), n, m, np.ones(4, np.float32),
                       np.ones(m, np.complex64))
    assert c["adds"] == 32 and c["subs"] == 0  # U_re mask drives the re and im path (O1)
    assert c["slots"] == 8 * n * m and c["scale_muls"] == 8


# ---------------------------------------------------------------- two-phase dense form

def _dense(planar, n, m, scales, x, conv, omp, rows=None):
    U, Wd = orc.build_dense(planar, n, m, scales, rows, omp=omp)
    return orc.eval_dense(U, Wd, x, conv, omp=omp)


@pytest.mark.parametrize("omp", [False, True])
@pytest.mark.parametrize("ex", _golden(), ids=lambda e: e["name"])
def test_dense_form_worked_examples(ex, omp):
    # the phase-split form (CPU-baseline timing) reproduces the hand-worked values exactly
    n, m = ex["n"], ex["m"]
    planar = orc.pack_planar(np.stack([np.array(ex[p], np.int8) for p in PLANES]))
    scales = (np.array(ex["scales_per_row"], np.float32) if "scales_per_row" in ex
              else np.array(ex["scales_per_tensor"], np.float32))
    x = np.array([complex(a, b) for a, b in ex["x"]], np.complex64)
    for conv, key in ((orc.CONV_EQ1, "y_EQ1"), (orc.CONV_ALG1, "y_ALG1")):
        want = np.array([complex(a, b) for a, b in ex[key]])
        assert np.array_equal(_dense(planar, n, m, scales, x, conv, omp)[0], want)


@pytest.mark.parametrize("omp", [False, True])
def test_dense_form_w_zero_is_zgemv(omp):
    n, m = 41, 90
    planes, _, scales, x = _rand_layer(12, n, m)
    planes[2:] = 0
    U = scales[:, 0:1].astype(np.float64) * planes[0] + 1j * scales[:, 1:2] * planes[1]
    got = _dense(orc.pack_planar(planes), n, m, scales, x, orc.CONV_EQ1, omp)[0]
    np.testing.assert_allclose(got, U @ x.astype(np.complex128), rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("conv", [orc.CONV_EQ1, orc.CONV_ALG1])
def test_dense_form_bitwise_equals_direct_any_thread_count(conv):
    n, m = 203, 517
    planes, planar, scales, _ = _rand_layer(13, n, m)
    x = wi.activations(13, m, 3)
    want = orc.wl_direct(planar, n, m, scales, x, conv)
    for omp in (False, True):
        assert np.array_equal(_dense(planar, n, m, scales, x, conv, omp), want)
    rows = np.array([202, 0, 17, 17, 100])
    assert np.array_equal(_dense(planar, n, m, scales, x, conv, True, rows),
                          orc.wl_direct(planar, n, m, scales, x, conv, rows))
    assert orc.num_threads(False) == 1 and orc.num_threads(True) >= 1


def test_dense_form_rejects_invalid_encoding():
    n, m = 3, 16
    planar = orc.pack_planar(np.zeros((4, n, m), np.int8))
    planar[1, 2, 0] = 0x3  # slot 0 of row 2 = (1,1)
    with pytest.raises(orc.OracleError):
        orc.build_dense(planar, n, m, np.ones((n, 4), np.float32), omp=True)


# ---------------------------------------------------------------- decode-block ops (NEXT-3)

def test_rmsnorm_spec_examples():
    # x = [3, 4] (RMS = sqrt(12.5)), gamma = 1, eps = 0 -> [0.8485, 1.1314]
    y = orc.rmsnorm(np.array([3 + 4j]), np.ones(2), eps=0.0)
    assert abs(y[0].real - 3 / np.sqrt(12.5)) < 1e-15 and abs(y[0].imag - 4 / np.sqrt(12.5)) < 1e-15
    assert abs(y[0].real - 0.8485) < 1e-4 and abs(y[0].imag - 1.1314) < 1e-4
    # all ones, eps -> 0: unit RMS; gamma = 0 -> 0
    assert np.allclose(orc.rmsnorm(np.ones(8) * (1 + 1j), np.ones(16), 0.0), 1 + 1j)
    assert not orc.rmsnorm(np.arange(1, 5) * (1 - 2j), np.zeros(8)).any()
    # gamma applies per real component: re and im of one column get their own weights
    y = orc.rmsnorm(np.array([1 + 1j]), np.array([2.0, 0.5]), 0.0)
    assert np.isclose(y[0], 2 + 0.5j)


def test_silu_spec_examples():
    # silu(0) = 0, silu(1) = 1/(1+e^-1) = 0.7311, large x -> x
    assert orc.silu(0.0) == 0.0
    assert abs(orc.silu(1.0) - 1 / (1 + np.exp(-1.0))) < 1e-16 and abs(orc.silu(1.0) - 0.7311) < 1e-4
    assert abs(orc.silu(40.0) - 40.0) < 1e-12 and abs(orc.silu(-40.0)) < 1e-15
    z = orc.silu_c(np.array([1 - 1j]))
    assert np.isclose(z[0], orc.silu(1.0) + 1j * orc.silu(-1.0))


def test_block_zero_weights_is_identity():
    # all-zero weights -> output = x (residual-only path); every GEMV gives 0
    m, dff = 32, 48
    zero = {p: (np.zeros((n, mm), complex), np.zeros((n, mm), complex))
            for p, n, mm in (("q", m, m), ("k", m, m), ("v", m, m), ("o", m, m),
                             ("gate", dff, m), ("up", dff, m), ("down", m, dff))}
    h = wi.activations(5, m)[0].astype(np.complex128)
    g = (np.ones(2 * m), np.ones(2 * m))
    out, mid = orc.block_forward(zero, h, g)
    assert np.array_equal(out, h) and not mid["v"].any() and not mid["act"].any()


def test_block_identity_projections_closed_form():
    # U_re = I for every projection (scales 1, W = 0): q = k = v = rmsnorm(h), h1 = h + v,
    # gate = up = rmsnorm(h1), a = silu(gate) (.) up, h2 = h1 + a -- each step by hand
    m = 16
    eye = np.zeros((4, m, m), np.int8)
    eye[0] = np.eye(m, dtype=np.int8)
    U, Wd = orc.build_dense(orc.pack_planar(eye), m, m, np.ones(4, np.float32))
    assert np.array_equal(U, np.eye(m)) and not Wd.any()
    layer = {p: (U, Wd) for p in ("q", "k", "v", "o", "gate", "up", "down")}
    h = wi.activations(6, m)[0].astype(np.complex128)
    g1 = wi.scales(7, m // 2, True, 0.5, 1.5).reshape(-1).astype(np.float64)
    g2 = wi.scales(8, m // 2, True, 0.5, 1.5).reshape(-1).astype(np.float64)
    out, mid = orc.block_forward(layer, h, (g1, g2), eps=1e-5)
    v = np.stack([h.real, h.imag], -1).reshape(-1)
    xa = v * g1 / np.sqrt(np.mean(v * v) + 1e-5)
    h1 = h + (xa[0::2] + 1j * xa[1::2])
    w = np.stack([h1.real, h1.imag], -1).reshape(-1)
    xm = w * g2 / np.sqrt(np.mean(w * w) + 1e-5)
    act = xm / (1 + np.exp(-xm)) * xm
    want = h1 + (act[0::2] + 1j * act[1::2])
    assert np.allclose(mid["h1"], h1, rtol=1e-14, atol=1e-14)
    assert np.allclose(out, want, rtol=1e-14, atol=1e-14)
