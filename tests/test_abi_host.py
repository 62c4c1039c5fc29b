"""C-ABI library: loads, exports every symbol include/ww.h declares, and its host
functions (packer, unpacker, re-layout, shard planner, errors) are right.  CPU only:
no compute call needs a GPU here."""
import os
import re

import numpy as np
import pytest

import oracle as orc
import paper_2604_20913_b200 as ww
import ww_inputs as wi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "ww.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ww_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    declared = _header_functions()
    assert len(declared) >= 12
    assert set(declared) == set(ww.EXPORTS)
    for name in declared:
        assert hasattr(ww._lib, name), name


def test_version_and_status_strings():
    assert ww.version() == 1
    assert ww.status_string(0) == "WW_OK"
    assert ww.status_string(ww.ERR_INVALID_ENCODING) == "WW_ERR_INVALID_ENCODING"


def test_packed_bytes():
    assert ww.packed_bytes(2048, 2048) == 2048 * 2048
    assert ww.packed_bytes(5504, 2048) == 11_272_192
    assert ww.packed_bytes(1, 1) == 16
    assert ww.packed_bytes(3, 17) == 3 * 2 * 16


@pytest.mark.parametrize("n,m", [(1, 1), (2, 16), (3, 17), (7, 100), (16, 64)])
def test_planar_pack_matches_oracle_app_h(n, m):
    planes = wi.planes(n * 31 + m, n, m, wi.UNIFORM3)
    got = ww.pack_ternary(planes, ww.LAYOUT_PLANAR)
    want = orc.pack_planar(planes).reshape(-1)
    assert np.array_equal(got, want)


def test_worked_example_words():
    # SURVEY App. A.2 words: planar U_re [0x2,0x9] ...; the COL4 bytes are their transposition
    planes = np.array([[[1, 0], [-1, 1]], [[0, -1], [1, 0]], [[0, 1], [1, -1]], [[-1, 0], [0, 1]]],
                      np.int8)
    planar = ww.pack_ternary(planes, ww.LAYOUT_PLANAR).reshape(4, 2, 1)
    assert [int(v) for v in planar[:, :, 0].reshape(-1)] == [2, 9, 4, 2, 8, 6, 1, 8]
    col4 = ww.pack_ternary(planes, ww.LAYOUT_COL4).reshape(2, 4)
    # row 0, column 0: U_re=+1 (bit1), U_im=0, W_re=0, W_im=-1 (bit6) -> 0x42
    # row 0, column 1: U_re=0, U_im=-1 (bit2), W_re=+1 (bit5), W_im=0 -> 0x24
    assert int(col4[0, 0]) == 0x2442
    # row 1: col 0: U_re=-1 (bit0), U_im=+1 (bit3), W_re=+1 (bit5) -> 0x29;
    #        col 1: U_re=+1 (bit1), W_re=-1 (bit4), W_im=+1 (bit7) -> 0x92
    assert int(col4[1, 0]) == 0x9229
    assert not col4[:, 1:].any()


@pytest.mark.parametrize("layout", [ww.LAYOUT_PLANAR, ww.LAYOUT_COL4])
@pytest.mark.parametrize("n,m", [(1, 1), (5, 15), (4, 16), (9, 33), (33, 200)])
def test_pack_unpack_roundtrip(layout, n, m):
    planes = wi.planes(n + 1000 * m, n, m)
    packed = ww.pack_ternary(planes, layout)
    assert packed.nbytes == ww.packed_bytes(n, m)
    assert np.array_equal(ww.unpack_ternary(packed, n, m, layout), planes)


def test_repack_both_ways():
    n, m = 13, 70
    planes = wi.planes(99, n, m)
    pl = ww.pack_ternary(planes, ww.LAYOUT_PLANAR)
    c4 = ww.pack_ternary(planes, ww.LAYOUT_COL4)
    assert np.array_equal(ww.repack(pl, n, m, ww.LAYOUT_PLANAR, ww.LAYOUT_COL4), c4)
    assert np.array_equal(ww.repack(c4, n, m, ww.LAYOUT_COL4, ww.LAYOUT_PLANAR), pl)


def test_col4_matches_oracle_planar_semantics():
    # COL4 -> PLANAR through the library, then the oracle unpacks it: same planes
    n, m = 8, 50
    planes = wi.planes(5, n, m)
    pl = ww.repack(ww.pack_ternary(planes, ww.LAYOUT_COL4), n, m, ww.LAYOUT_COL4,
                   ww.LAYOUT_PLANAR).reshape(4, n, -1)
    for p in range(4):
        assert np.array_equal(orc.unpack_plane(pl[p], m), planes[p])


def test_invalid_code_rejected():
    planes = np.zeros((4, 2, 3), np.int8)
    planes[3, 1, 2] = 2
    with pytest.raises(ww.WWError) as e:
        ww.pack_ternary(planes)
    assert e.value.status == ww.ERR_INVALID_CODE
    assert "plane 3 row 1 col 2" in str(e.value)


@pytest.mark.parametrize("layout", [ww.LAYOUT_PLANAR, ww.LAYOUT_COL4])
def test_unpack_rejects_slot_11(layout):
    n, m = 2, 20
    packed = ww.pack_ternary(np.zeros((4, n, m), np.int8), layout)
    packed[3] |= 0x3 << 4  # some slot becomes (1,1)
    with pytest.raises(ww.WWError) as e:
        ww.unpack_ternary(packed, n, m, layout)
    assert e.value.status == ww.ERR_INVALID_ENCODING


def test_pack_argument_errors():
    with pytest.raises(ww.WWError) as e:
        ww._check(ww._lib.ww_pack_ternary(None, None, None, None, 1, 1, 1, 1, None))
    assert e.value.status == ww.ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("n,world", [(10, 4), (2048, 8), (5504, 8), (2048, 1), (3, 4), (7, 3)])
def test_shard_plan_partition(n, world):
    m = 2048
    shards = [ww.shard_plan(n, m, world, r) for r in range(world)]
    rpr = -(-n // world)
    covered = []
    for r, s in enumerate(shards):
        assert s.rows_per_rank == rpr and s.n_padded == rpr * world
        assert s.row_begin == min(r * rpr, n) and s.row_end == min((r + 1) * rpr, n)
        assert s.packed_offset_bytes == s.row_begin * m
        assert s.packed_bytes == (s.row_end - s.row_begin) * m
        assert s.scale_offset_floats == 4 * s.row_begin
        assert s.y_offset_complex == r * rpr
        covered.extend(range(s.row_begin, s.row_end))
    assert covered == list(range(n))  # disjoint, contiguous, complete


def test_shard_plan_spec_example_sizes():
    # n=10, t=4 -> [3,3,2,2] under the balanced split; the ceil-block plan gives
    # [3,3,3,1] (equal all-gather counts) and agrees whenever world | n.
    sizes = [ww.shard_plan(10, 16, 4, r) for r in range(4)]
    assert [s.row_end - s.row_begin for s in sizes] == [3, 3, 3, 1]
    sizes = [ww.shard_plan(2048, 16, 8, r) for r in range(8)]
    assert [s.row_end - s.row_begin for s in sizes] == [256] * 8


def test_shard_plan_errors():
    for args in ((0, 1, 1, 0), (4, 4, 0, 0), (4, 4, 2, 2), (4, 4, 2, -1)):
        with pytest.raises(ww.WWError):
            ww.shard_plan(*args)


def test_query_launch_shapes():
    for n, m in ((2048, 2048), (5504, 2048), (2048, 5504), (128, 128)):
        li = ww.query_launch(ww.Layer(n, m), 1)
        assert li["grid"] >= 1 and li["block"] % 32 == 0
        assert li["tiles"] == 1
        assert li["tile_chunks"] == -(-m // 16)
    # B > 4 runs as groups of 4 vectors: the plan of one group
    assert ww.query_launch(ww.Layer(2048, 5504), 16) == ww.query_launch(ww.Layer(2048, 5504), 4)
    li = ww.query_launch(ww.Layer(2048, 8000), 4)  # x of 4 vectors beyond one tile
    assert li["tiles"] > 1 and li["tile_chunks"] % 32 == 0
    with pytest.raises(ww.WWError) as e:
        ww.query_launch(ww.Layer(8, 8), 17)
    assert e.value.status == ww.ERR_UNSUPPORTED
    with pytest.raises(ww.WWError):
        ww.query_launch(ww.Layer(8, 8, layout=ww.LAYOUT_PLANAR), 1)


def test_launch_rows_whole_or_split_in_halves():
    # rows are never split into column parts with their own sums (ww.h ww_launch_info): a
    # row is either one warp's unit, or (B = 1, parts = 2) two halves whose lane state is
    # handed from one warp to the next, so a row's arithmetic depends on (m, B) only
    for m in (16, 1000, 1024, 2048, 4096, 5504):
        W = -(-m // 16)
        J = -(-W // 32)
        for B in (1, 4, 16):
            for n in (1, 148, 2048, 11008):
                i = ww.query_launch(ww.Layer(n, m), B)
                if i["parts"] == 1:
                    assert i["split_chunks"] == W
                else:
                    assert (B, i["parts"], i["split_chunks"]) == (1, 2, -(-J // 2) * 32)
                    assert J >= 2


def test_split_rows_planned_where_sub_partitions_are_unbalanced():
    # 148 SMs x 4 sub-partitions of 4 warps: n = 2048 gives 14 rows per CTA (4 + 4 + 3 + 3 per
    # sub-partition) -> halves, for rows with a ragged last sweep (W % 32 != 0: down); rows
    # of whole sweeps keep the stream producer; gate/up-like row counts stay whole
    shapes = ((2048, 2048), (2048, 5504), (6144, 2048), (11008, 2048), (1, 2048), (1, 5504),
              (2048, 3000), (11008, 3000))
    parts = {(n, m): ww.query_launch(ww.Layer(n, m), 1)["parts"] for n, m in shapes}
    if ww.query_launch(ww.Layer(2048, 2048), 1)["num_sms"] != 148:
        pytest.skip("planned for another SM count")
    assert parts == {(2048, 2048): 1, (2048, 5504): 2, (6144, 2048): 1, (11008, 2048): 1,
                     (1, 2048): 1, (1, 5504): 2, (2048, 3000): 2, (11008, 3000): 1}
    assert ww.query_launch(ww.Layer(2048, 5504), 2)["parts"] == 1
    assert ww.query_launch(ww.Layer(2048, 500), 1)["parts"] == 1  # one sweep per row


# ---------------------------------------------------------------- WW_LAYOUT_TILE32
def _tile32_from_app_h(planar, n, m):
    """Place the oracle's App. H words (4, n, W) at their TILE32 positions (ww.h): the
    layout is a pure permutation of App. H words, zero-padded to 32-row tiles and 4-word
    slabs."""
    W = (m + 15) // 16
    S = (W + 3) // 4
    T = (n + 31) // 32
    out = np.zeros((T, S, 32, 4, 4), np.uint32)  # tile, slab, row, plane, word-in-slab
    pw = np.zeros((4, T * 32, S * 4), np.uint32)
    pw[:, :n, :W] = planar
    pw = pw.reshape(4, T, 32, S, 4)
    out[:] = pw.transpose(1, 3, 2, 0, 4)
    return out.reshape(-1)


@pytest.mark.parametrize("n,m", [(1, 1), (3, 17), (32, 64), (33, 65), (70, 300), (64, 2048)])
def test_tile32_pack_is_app_h_words_retiled(n, m):
    planes = wi.planes(n * 7 + m, n, m, wi.UNIFORM3)
    got = ww.pack_ternary(planes, ww.LAYOUT_TILE32)
    assert got.nbytes == ww.packed_bytes(n, m, ww.LAYOUT_TILE32)
    assert got.nbytes == ((n + 31) // 32) * ((m + 63) // 64) * 2048
    want = _tile32_from_app_h(orc.pack_planar(planes), n, m)
    assert np.array_equal(got, want)
    assert np.array_equal(ww.unpack_ternary(got, n, m, ww.LAYOUT_TILE32), planes)
    for src in (ww.LAYOUT_PLANAR, ww.LAYOUT_COL4):
        other = ww.pack_ternary(planes, src)
        assert np.array_equal(ww.repack(other, n, m, src, ww.LAYOUT_TILE32), got)
        assert np.array_equal(ww.repack(got, n, m, ww.LAYOUT_TILE32, src), other)


def test_tile32_sizes_match_other_layouts_on_llama_shapes():
    for n, m in ((2048, 2048), (5504, 2048), (2048, 5504), (6144, 2048), (11008, 2048)):
        assert ww.packed_bytes(n, m, ww.LAYOUT_TILE32) == ww.packed_bytes(n, m) == n * m
    assert ww._lib.ww_packed_bytes_layout(4, 4, 9) == 0


def _tcv_maxc(n, m, sms=148):
    T, S = (n + 31) // 32, (m + 63) // 64
    U = T * S
    G = min(U, sms)
    own = lambda u: ((u + 1) * G - 1) // U  # noqa: E731
    return T, max([1] + [own((t + 1) * S - 1) - own(t * S) for t in range(T)])


def test_tcv_workspace_bytes():
    """T tiles x (most contributing CTAs of a split tile) x 128 M-rows x NB flagged 8-byte
    words; the planner assumes the device's SM count (148 without a GPU)."""
    for (n, m, B) in ((2048, 5504, 1), (2048, 2048, 2), (11008, 2048, 1), (33, 10, 3)):
        T, maxc = _tcv_maxc(n, m)
        NB = 16 if B <= 2 else 32
        assert ww.tcv_workspace_bytes(n, m, B) == T * maxc * 128 * NB * 8
    assert ww.tcv_workspace_bytes(10, 10, 5) == 0 and ww.tcv_workspace_bytes(0, 10, 1) == 0
