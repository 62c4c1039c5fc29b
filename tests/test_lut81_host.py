"""WW_LAYOUT_LUT81 host conversion (ww_lut81_from_planar / ww_lut81_to_planar): a bijection of
the App. H bit pairs -- checked against the oracle's planar packer, by an
independent restatement of the byte rule in ww.h, and on the error cases."""
import numpy as np
import pytest

import oracle as orc
import ww_inputs as wi
import paper_2604_20913_b200 as ww


@pytest.mark.parametrize("n,m", [(1, 1), (3, 5), (7, 128), (5, 517), (2, 1025), (9, 2048)])
def test_round_trip_and_byte_rule(n, m):
    planes = wi.planes(n + m, n, m, wi.UNIFORM3)
    planar = np.asarray(orc.pack_planar(planes), dtype=np.uint32).ravel()
    lut = ww.lut81_from_planar(planar, n, m)
    T = (m + 511) // 512
    assert lut.size == ww.lut81_packed_bytes(n, m) == n * T * 512
    assert np.array_equal(ww.lut81_to_planar(lut, n, m), planar)
    # ww.h: byte 16*((i*T + t)*32 + l) + 4*p + k = sum_k' (code + 1) 3^k' of columns 512t+128k+4l..+3
    pad = np.zeros((4, n, T * 512), np.int64)
    pad[:, :, :m] = planes
    rng = np.random.default_rng(0)
    for _ in range(200):
        p, i = int(rng.integers(4)), int(rng.integers(n))
        t, k, l = int(rng.integers(T)), int(rng.integers(4)), int(rng.integers(32))
        c = pad[p, i, 512 * t + 128 * k + 4 * l:512 * t + 128 * k + 4 * l + 4]
        assert lut[16 * ((i * T + t) * 32 + l) + 4 * p + k] == sum((int(c[q]) + 1) * 3 ** q for q in range(4))
    assert np.array_equal(ww.pack_lut81(planes), lut)


def test_invalid_encodings():
    n, m = 2, 20
    planar = np.zeros(4 * n * 2, np.uint32)
    planar[3] = 0b11 << 6  # the unused (1,1) slot
    with pytest.raises(ww.WWError):
        ww.lut81_from_planar(planar, n, m)
    lut = ww.pack_lut81(np.zeros((4, n, m), np.int8))
    assert (lut == 40).all()
    bad = lut.copy()
    bad[5] = 81
    with pytest.raises(ww.WWError):
        ww.lut81_to_planar(bad, n, m)
    bad = lut.copy()
    bad[16 * 31] = 41  # lane 31 of step 0, block 0: columns 124.. are padding at m = 20
    with pytest.raises(ww.WWError):
        ww.lut81_to_planar(bad, n, m)
