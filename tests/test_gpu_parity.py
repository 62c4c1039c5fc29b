"""GPU parity: the sm_100a WL-GEMV kernels (through the C ABI) against the C fp64
oracle on the same seeded inputs.  Bar (R8): rel L2 <= 1e-5 and per element
|err| <= 1e-4 * max_c s_c(i) * sum_j |x_j|.  Integer work (packing) is bit-exact."""
import numpy as np
import pytest

import oracle as orc
import ww_inputs as wi
from _wl import LayerCase, assert_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_2604_20913_b200 as ww  # noqa: E402

CONVS = [ww.CONV_EQ1, ww.CONV_ALG1]
ORC = {ww.CONV_EQ1: orc.CONV_EQ1, ww.CONV_ALG1: orc.CONV_ALG1}


@pytest.mark.parametrize("spec", [wi.C1, wi.C2, wi.C3A, wi.C3B], ids=lambda s: s.name)
@pytest.mark.parametrize("conv", CONVS)
def test_baseline_configs_full(spec, conv):
    case = LayerCase.from_spec(spec, seed=0).device(ww, torch)
    y = case.gpu(ww, torch, conv)
    assert_parity(y, case.oracle(ORC[conv]), case)


@pytest.mark.parametrize("B", wi.C5_BATCHES)
@pytest.mark.parametrize("conv", CONVS)
def test_config5_batched_full(B, conv):
    case = LayerCase.from_spec(wi.C3B, seed=5, B=B).device(ww, torch)
    y = case.gpu(ww, torch, conv)
    assert_parity(y, case.oracle(ORC[conv]), case)


SHAPES = [(1, 1), (1, 15), (15, 1), (16, 16), (17, 17), (63, 64), (64, 65), (65, 63),
          (128, 1000), (1000, 128), (149, 17), (300, 513), (2, 4097)]


@pytest.mark.parametrize("n,m", SHAPES)
@pytest.mark.parametrize("conv", CONVS)
@pytest.mark.parametrize("per_row", [True, False])
def test_small_and_ragged_shapes(n, m, conv, per_row):
    case = LayerCase(n, m, seed=n * 7919 + m, dist=wi.UNIFORM3, per_row=per_row,
                     lo=0.5, hi=2.0).device(ww, torch)
    assert_parity(case.gpu(ww, torch, conv), case.oracle(ORC[conv]), case)


@pytest.mark.parametrize("B", list(range(1, 17)))
def test_every_batch_size_and_batch_invariance(B):
    n, m = 150, 333
    case = LayerCase(n, m, seed=B, B=B).device(ww, torch)
    yb = case.gpu(ww, torch, ww.CONV_EQ1)
    assert_parity(yb, case.oracle(orc.CONV_EQ1), case)
    # a vector's accumulation order does not depend on the rest of the batch within an
    # accumulator family (B <= 2, 3 <= B <= 4, B >= 5)
    L = case.layer(ww, ww.CONV_EQ1)
    rep = 1 if B <= 2 else (3 if B <= 4 else 5)
    for b in (0, B - 1):
        X = torch.stack([case.x_d[b]] + [case.x_d[(b + k) % B] for k in range(1, rep)])
        y1 = ww.wl_gemv_batched(L, case.packed_d, case.scales_d, X)
        assert np.array_equal(y1[0].cpu().numpy(), yb[b])


@pytest.mark.parametrize("m", [1537, 3000, 5504])
def test_ragged_last_sweep_batch2(m):
    # rows whose last 32-chunk sweep is partial (idle lanes load zeros), two vectors
    case = LayerCase(300, m, seed=m, B=2).device(ww, torch)
    assert (-(-m // 16)) % 32 != 0
    for conv in CONVS:
        assert_parity(case.gpu(ww, torch, conv), case.oracle(ORC[conv]), case)


def test_multi_tile_long_rows():
    # x larger than one shared-memory tile (B=1: 184 KB = 23552 complex columns)
    case = LayerCase(40, 30000, seed=3).device(ww, torch)
    assert ww.query_launch(case.layer(ww, 0), 1)["tiles"] > 1
    for conv in CONVS:
        assert_parity(case.gpu(ww, torch, conv), case.oracle(ORC[conv]), case)


def test_batched_multi_tile_and_waves():
    # 4 vectors of 8000 columns need column tiles; 5000 rows force several row waves per CTA
    case = LayerCase(5000, 8000, seed=4, B=4).device(ww, torch)
    assert ww.query_launch(case.layer(ww, 0), 4)["tiles"] > 1
    assert_parity(case.gpu(ww, torch, ww.CONV_ALG1), case.oracle(orc.CONV_ALG1), case)


@pytest.mark.parametrize("B", [5, 6, 7, 8, 13, 16])
def test_large_batches_run_as_groups_bitwise_equal_to_group_launches(B):
    # B > 4 runs as groups of 4 vectors (the last group overlapping): every vector equals a
    # launch of its own group of 4, bitwise, and matches the oracle
    case = LayerCase(700, 2100, seed=B, B=B).device(ww, torch)
    yb = case.gpu(ww, torch, ww.CONV_EQ1)
    assert_parity(yb, case.oracle(orc.CONV_EQ1), case)
    L = case.layer(ww, ww.CONV_EQ1)
    for b in range(B):
        s0 = min(b - b % 4, B - 4)
        y4 = ww.wl_gemv_batched(L, case.packed_d, case.scales_d, case.x_d[s0:s0 + 4])
        assert np.array_equal(y4[b - s0].cpu().numpy(), yb[b])


def test_zero_and_identity_exact():
    n = m = 257
    x = wi.activations(9, m)
    planes = np.zeros((4, n, m), np.int8)
    case = LayerCase(n, m, planes=planes, scales=np.ones((n, 4), np.float32), x=x).device(ww, torch)
    assert not case.gpu(ww, torch, ww.CONV_EQ1).any()
    planes[0] = np.eye(n, dtype=np.int8)
    case = LayerCase(n, m, planes=planes, scales=np.ones(4, np.float32), x=x).device(ww, torch)
    for conv in CONVS:
        assert np.array_equal(case.gpu(ww, torch, conv)[0], x[0])


def test_conventions_differ_only_in_w_terms():
    case = LayerCase(64, 96, seed=12).device(ww, torch)
    a = case.gpu(ww, torch, ww.CONV_EQ1)
    b = case.gpu(ww, torch, ww.CONV_ALG1)
    assert np.array_equal(a.real, b.real)  # y_re is the same expression (Eq. 2)
    assert not np.array_equal(a.imag, b.imag)


def test_determinism_and_pdl_flag():
    case = LayerCase.from_spec(wi.C2, seed=1).device(ww, torch)
    ys = [case.gpu(ww, torch, ww.CONV_EQ1) for _ in range(3)]
    ys.append(case.gpu(ww, torch, ww.CONV_EQ1, flags=ww.FLAG_PDL))
    for y in ys[1:]:
        assert np.array_equal(y, ys[0])


@pytest.mark.parametrize("m", [128, 1000, 1537, 2000, 2048, 3000, 4096, 5504])
def test_row_results_independent_of_n(m):
    # a row's arithmetic depends on (m, B) only (ww.h ww_launch_info: whole rows): the
    # first n' rows of an n-row layer, launched alone, are bitwise the same for every n'
    # (different CTA row ranges and per-warp row ranges)
    n = 1500
    case = LayerCase(n, m, seed=m + 5).device(ww, torch)
    full = case.gpu(ww, torch, ww.CONV_EQ1)[0]
    assert_parity(full[None], case.oracle(orc.CONV_EQ1), case)
    for n2 in (1, 2, 7, 31, 149, 297, 1000):
        L = ww.Layer(n2, m)
        y = ww.wl_gemv(L, case.packed_d[:ww.packed_bytes(n2, m)], case.scales_d[:n2],
                       case.x_d[0])
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), full[:n2]), f"n'={n2}"


@pytest.mark.parametrize("world", [2, 4, 8])
def test_shard_invariance_emulated(world):
    # each rank's slice run on its own (n_local rows), concatenated == unsharded, bitwise
    spec = wi.C3A
    case = LayerCase.from_spec(spec, seed=2).device(ww, torch)
    full = case.gpu(ww, torch, ww.CONV_EQ1)[0]
    gathered = torch.zeros(ww.shard_plan(spec.n, spec.m, world, 0).n_padded, dtype=torch.complex64,
                           device="cuda")
    for r in range(world):
        s = ww.shard_plan(spec.n, spec.m, world, r)
        if s.row_end == s.row_begin:
            continue
        L = ww.Layer(s.row_end - s.row_begin, spec.m)
        pk = case.packed_d[s.packed_offset_bytes:s.packed_offset_bytes + s.packed_bytes]
        sc = case.scales_d.reshape(-1)[s.scale_offset_floats:s.scale_offset_floats + s.scale_count]
        out = gathered[s.y_offset_complex:s.y_offset_complex + (s.row_end - s.row_begin)]
        ww.wl_gemv(L, pk, sc, case.x_d[0], out)
    torch.cuda.synchronize()
    assert np.array_equal(gathered[:spec.n].cpu().numpy(), full)


def test_slot_11_contributes_add_then_subtract():
    # (1,1) is never packed; the kernel applies Eq. 6 then Eq. 7 (x - x), a zero contribution
    # up to rounding (R3): parity with the oracle treating those codes as 0.
    n, m = 33, 64
    case = LayerCase(n, m, seed=21).device(ww, torch)
    ref = case.oracle(orc.CONV_EQ1)
    words = ww.pack_ternary(case.planes, ww.LAYOUT_COL4).copy()
    zero_cols = np.argwhere(case.planes[1] == 0)[:50]
    for i, j in zero_cols:  # U_im code (plane 1) of column j: bits 2, 3 of byte j%16
        w = (i * ((m + 15) // 16) + j // 16) * 4 + (j % 16) // 4
        words[w] |= 0x3 << (8 * (j % 4) + 2)
    case.packed_d = torch.from_numpy(words.view(np.uint8)).cuda()
    assert_parity(case.gpu(ww, torch, ww.CONV_EQ1), ref, case)


def test_unaligned_x_path():
    # x at an 8-byte (not 16-byte) offset exercises the 8-byte cp.async staging path
    case = LayerCase(100, 77, seed=8).device(ww, torch)
    buf = torch.zeros(78, dtype=torch.complex64, device="cuda")
    buf[1:] = case.x_d[0]
    y = ww.wl_gemv(case.layer(ww, ww.CONV_EQ1), case.packed_d, case.scales_d, buf[1:])
    torch.cuda.synchronize()
    assert_parity(y.cpu().numpy()[None], case.oracle(orc.CONV_EQ1), case)


def test_device_packer_bit_exact():
    n, m = 333, 1000
    planes = wi.planes(17, n, m)
    d = torch.from_numpy(planes).cuda().contiguous()
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    got = ww.pack_ternary_device(d, bad)
    torch.cuda.synchronize()
    want = ww.pack_ternary(planes, ww.LAYOUT_COL4).view(np.uint8)
    assert np.array_equal(got.cpu().numpy(), want) and int(bad.item()) == 0
    d[2, 5, 7] = 3
    got = ww.pack_ternary_device(d, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 1
    # only the bad column packs as zero: its word-mates 4..6 keep their codes
    fixed = planes.copy()
    fixed[:, 5, 7] = 0
    want = ww.pack_ternary(fixed, ww.LAYOUT_COL4).view(np.uint8)
    assert np.array_equal(got.cpu().numpy(), want)


def test_device_generated_codes_pack_like_host():
    n, m = 512, 2048
    d = torch.empty((4, n, m), dtype=torch.int8, device="cuda")
    for p in range(4):
        wi.codes_device(77, p, n, m, d[p])
    got = ww.pack_ternary_device(d)
    torch.cuda.synchronize()
    want = ww.pack_ternary(wi.planes(77, n, m), ww.LAYOUT_COL4).view(np.uint8)
    assert np.array_equal(got.cpu().numpy(), want)


def test_argument_errors_before_launch():
    case = LayerCase(8, 32, seed=1).device(ww, torch)
    L = case.layer(ww, ww.CONV_EQ1)
    y = torch.empty(8, dtype=torch.complex64, device="cuda")
    buf = torch.zeros(case.packed_d.numel() + 16, dtype=torch.uint8, device="cuda")
    buf[1:1 + case.packed_d.numel()] = case.packed_d
    with pytest.raises(ww.WWError) as e:
        ww.wl_gemv(L, buf[1:1 + case.packed_d.numel()], case.scales_d, case.x_d[0], y)
    assert e.value.status == ww.ERR_MISALIGNED
    # marshalling checks in the binding: wrong dtype, inner stride, sizes
    with pytest.raises(TypeError):
        ww.wl_gemv(L, case.packed_d, case.scales_d, case.x_d[0].to(torch.complex128), y)
    Z = torch.zeros((2, 64), dtype=torch.complex64, device="cuda")
    with pytest.raises(ValueError):
        ww.wl_gemv_batched(L, case.packed_d, case.scales_d, Z[:, ::2])
    with pytest.raises(ValueError):
        ww.wl_gemv(L, case.packed_d[:-16], case.scales_d, case.x_d[0], y)
    with pytest.raises(ValueError):
        ww.wl_gemv(L, case.packed_d, case.scales_d[:4], case.x_d[0], y)
    X = torch.zeros((17, 32), dtype=torch.complex64, device="cuda")
    with pytest.raises(ww.WWError) as e:
        ww.wl_gemv_batched(L, case.packed_d, case.scales_d, X)
    assert e.value.status == ww.ERR_UNSUPPORTED
    with pytest.raises(ww.WWError) as e:
        ww.wl_gemv(ww.Layer(8, 32, layout=ww.LAYOUT_PLANAR), case.packed_d, case.scales_d,
                   case.x_d[0], y)
    assert e.value.status == ww.ERR_UNSUPPORTED
    with pytest.raises(ww.WWError) as e:
        ww.wl_gemv(L, case.packed_d, case.scales_d, case.x_d[0], case.x_d[0].view(torch.complex64))
    assert e.value.status == ww.ERR_INVALID_ARGUMENT


def test_aligned_inputs_take_the_tma_path():
    # the product staging path: x boxes by cp.async.bulk.tensor (128B swizzle)
    case = LayerCase.from_spec(wi.C3B, seed=3).device(ww, torch)
    case.gpu(ww, torch, ww.CONV_EQ1)
    assert ww._lib.ww_debug_last_use_tma() == 1
    case = LayerCase(100, 77, seed=8).device(ww, torch)  # 16 does not divide m: cp.async
    case.gpu(ww, torch, ww.CONV_EQ1)
    assert ww._lib.ww_debug_last_use_tma() == 0


@pytest.mark.parametrize("n,m,B", [(2048, 2048, 1), (300, 5504, 3), (77, 1000, 1)])
def test_cp_async_staging_path_matches_tma_path(n, m, B):
    # x staged by per-thread cp.async (fallback for 16 !| m, misaligned x, odd ldx) must give
    # the same bits as the TMA (cp.async.bulk.tensor, 128B swizzle) staging
    case = LayerCase(n, m, seed=n + m + B, B=B).device(ww, torch)
    y_tma = case.gpu(ww, torch, ww.CONV_EQ1)
    ww._lib.ww_debug_force_cp_async(1)
    try:
        y_cpa = case.gpu(ww, torch, ww.CONV_EQ1)
    finally:
        ww._lib.ww_debug_force_cp_async(0)
    assert np.array_equal(y_tma, y_cpa)
    assert_parity(y_cpa, case.oracle(orc.CONV_EQ1), case)


@pytest.mark.parametrize("n,m,B", [(2048, 2048, 1), (1000, 1024, 2), (7, 512, 1), (300, 4096, 4)])
def test_row_stream_kernel_matches_row_by_row_kernel(n, m, B):
    # rows of whole 32-chunk sweeps run the kStream instantiation (one contiguous weight
    # stream per warp, L2 prefetch); the row-by-row producer must give the same bits
    case = LayerCase(n, m, seed=n + m + 7 * B, B=B).device(ww, torch)
    y_stream = case.gpu(ww, torch, ww.CONV_ALG1)
    assert ww._lib.ww_debug_last_stream() == 1
    ww._lib.ww_debug_force_rows(1)
    try:
        y_rows = case.gpu(ww, torch, ww.CONV_ALG1)
        assert ww._lib.ww_debug_last_stream() == 0
    finally:
        ww._lib.ww_debug_force_rows(0)
    assert np.array_equal(y_stream, y_rows)
    assert_parity(y_stream, case.oracle(orc.CONV_ALG1), case)


@pytest.mark.parametrize("n,m", [(2048, 2048), (2048, 5504), (300, 517), (1, 16)])
@pytest.mark.parametrize("conv", CONVS)
def test_unfused_ablation_matches_oracle(n, m, conv):
    # the paper's unfused baseline (8 real ternary GEMVs + combine), NEXT-2 ablation
    case = LayerCase(n, m, seed=n + 3 * m).device(ww, torch)
    planar = torch.from_numpy(ww.pack_ternary(case.planes, ww.LAYOUT_PLANAR).view(np.uint8)).cuda()
    L = ww.Layer(n, m, ww.LAYOUT_PLANAR, ww.SCALES_PER_ROW, conv)
    y = ww.wl_gemv_unfused(L, planar, case.scales_d, case.x_d[0])
    torch.cuda.synchronize()
    assert_parity(y.cpu().numpy()[None], case.oracle(ORC[conv]), case)


@pytest.mark.parametrize("n", [200_000, 800_000])
def test_many_rows_per_cta(n):
    # 1,350 rows per CTA still fit the shared totals (one tile); 5,400 do not, and the launch
    # takes the row-wave path -- both match the oracle
    m = 24
    case = LayerCase(n, m, seed=77).device(ww, torch)
    li = ww.query_launch(case.layer(ww, 0), 1)
    assert li["path"] == (0 if n == 200_000 else 1)
    for conv in CONVS:
        assert_parity(case.gpu(ww, torch, conv), case.oracle(ORC[conv]), case)


@pytest.mark.parametrize("B", [1, 6])
@pytest.mark.parametrize("graph", [False, True])
def test_pdl_chain_reads_previous_layers_output(B, graph):
    # layer 2 reads layer 1's y as its x and layer 3 reads it as its per-row scales,
    # all launched with WW_FLAG_PDL on one stream (the next kernel starts while the previous
    # one runs).  y1 is poisoned with NaN before every run, so a read before
    # griddepcontrol.wait would show up; results must equal the same chain without PDL, bitwise.
    n2, m1 = 300, 1000
    n1 = 2 * n2  # y1 as float32 = n2 x 4 scales
    c1 = LayerCase(n1, m1, seed=31, B=B).device(ww, torch)
    c2 = LayerCase(n2, n1, seed=32, B=B).device(ww, torch)
    c3 = LayerCase(n2, m1, seed=33, B=B).device(ww, torch)
    s = torch.cuda.Stream()

    def chain(flags, Y1, Y2, Y3):
        L1, L2, L3 = c1.layer(ww, 0, flags), c2.layer(ww, 0, flags), c3.layer(ww, 0, flags)
        ww.wl_gemv_batched(L1, c1.packed_d, c1.scales_d, c1.x_d, Y1, stream=s)
        ww.wl_gemv_batched(L2, c2.packed_d, c2.scales_d, Y1, Y2, stream=s)
        sc3 = torch.view_as_real(Y1[0]).reshape(n2, 4)
        ww.wl_gemv_batched(L3, c3.packed_d, sc3, c3.x_d, Y3, stream=s)

    def bufs():
        out = [torch.empty((B, n), dtype=torch.complex64, device="cuda") for n in (n1, n2, n2)]
        for t in out:
            torch.view_as_real(t).fill_(float("nan"))  # both parts (a complex fill gives nan+0j)
        return out

    ref = bufs()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        chain(0, *ref)
    torch.cuda.synchronize()
    assert not any(torch.isnan(torch.view_as_real(r)).any() for r in ref)
    got = bufs()
    torch.cuda.synchronize()
    if graph:
        with torch.cuda.stream(s):
            chain(ww.FLAG_PDL, *got)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            chain(ww.FLAG_PDL, *got)
    for _ in range(5):
        with torch.cuda.stream(s):
            for t in got:
                torch.view_as_real(t).fill_(float("nan"))
            if graph:
                g.replay()
            else:
                chain(ww.FLAG_PDL, *got)
        torch.cuda.synchronize()
        for a, b in zip(ref, got):
            assert torch.equal(torch.view_as_real(a), torch.view_as_real(b))


def test_keep_in_l2_window_leaves_results_unchanged():
    # ww_stream_keep_in_l2 only changes caching: same bits with and without the window
    case = LayerCase.from_spec(wi.C2, seed=4).device(ww, torch)
    s = torch.cuda.Stream()
    L = case.layer(ww, ww.CONV_EQ1)
    y0 = ww.wl_gemv(L, case.packed_d, case.scales_d, case.x_d[0], stream=s)
    ww.keep_in_l2(case.x_d, s)
    y1 = ww.wl_gemv(L, case.packed_d, case.scales_d, case.x_d[0], stream=s)
    ww.keep_in_l2(None, s)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)


SPLIT_SHAPES = [(2048, 2048), (2048, 5504), (6144, 2048), (1, 2048), (2, 1000), (149, 1000),
                (300, 513), (17, 4097), (150, 1536), (37, 700), (2000, 3000)]


@pytest.mark.parametrize("n,m", SPLIT_SHAPES)
@pytest.mark.parametrize("per_row", [True, False])
def test_split_rows_bitwise_equal_whole_rows(n, m, per_row):
    # parts = 2 (ww.h ww_launch_info): halves of a row on two warps with the first half's
    # lane state handed over in shared memory -- the same bits as the whole-row kernel on
    # every shape (odd and even sweep counts, ragged last sweeps, a warp that is giver and
    # receiver, n = 1), both x-staging paths
    case = LayerCase(n, m, seed=n * 31 + m, per_row=per_row, lo=0.5, hi=2.0).device(ww, torch)
    outs = {}
    try:
        for mode in (0, 1):
            ww._lib.ww_debug_force_split(mode)
            assert ww.query_launch(case.layer(ww, 0), 1)["parts"] == (2 if mode else 1)
            outs[mode] = case.gpu(ww, torch, ww.CONV_EQ1)
        ww._lib.ww_debug_force_cp_async(1)
        outs["cpa"] = case.gpu(ww, torch, ww.CONV_EQ1)
    finally:
        ww._lib.ww_debug_force_split(-1)
        ww._lib.ww_debug_force_cp_async(0)
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], outs["cpa"])
    assert_parity(outs[1], case.oracle(orc.CONV_EQ1), case)
