"""Tensor-core WL-GEMV with the ternary operand decoded into tensor memory
(ww_wl_gemv_tc, WW_LAYOUT_TILE32, B = 1..4) against the fp64 oracle at the north-star bar:
BASELINE configs 1-3 and 5 (B <= 4) at full size for both conventions, ragged shapes
(tiles split across CTAs, n not a multiple of 32, m not a multiple of 64), per-tensor and
per-row scales, x of very different magnitudes per vector and component, zero weights and
zero x, the App. H unused slot (1,1), repeated launches on one workspace (which every call
must leave zeroed), PDL chains reading the previous launch's output, and bitwise
independence of the result from the row shard."""
import numpy as np
import pytest

import oracle as orc
import ww_inputs as wi
from _wl import LayerCase, assert_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_2604_20913_b200 as ww  # noqa: E402

ORC = {ww.CONV_EQ1: orc.CONV_EQ1, ww.CONV_ALG1: orc.CONV_ALG1}


def _dev(case):
    case.packed_d = torch.from_numpy(ww.pack_ternary(case.planes, ww.LAYOUT_TILE32).view(np.uint8)).cuda()
    case.scales_d = torch.from_numpy(np.ascontiguousarray(case.scales)).cuda()
    case.x_d = torch.from_numpy(np.ascontiguousarray(case.x)).cuda()
    return case


def _layer(case, conv, flags=0):
    return ww.Layer(case.n, case.m, ww.LAYOUT_TILE32,
                    ww.SCALES_PER_ROW if case.per_row else ww.SCALES_PER_TENSOR, conv, flags)


def _tc(case, conv, ws=None, flags=0):
    y = ww.wl_gemv_tc(_layer(case, conv, flags), case.packed_d, case.scales_d, case.x_d, workspace=ws)
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("spec", [wi.C1, wi.C2, wi.C3A, wi.C3B], ids=["C1", "C2", "C3a", "C3b"])
@pytest.mark.parametrize("conv", [ww.CONV_EQ1, ww.CONV_ALG1])
def test_configs_full_size(spec, conv):
    case = _dev(LayerCase.from_spec(spec, seed=11))
    assert_parity(_tc(case, conv), case.oracle(ORC[conv]), case)


@pytest.mark.parametrize("B", [1, 2, 3, 4])
def test_config5_batches(B):
    case = _dev(LayerCase.from_spec(wi.C3B, seed=5, B=B))
    for conv in (ww.CONV_EQ1, ww.CONV_ALG1):
        assert_parity(_tc(case, conv), case.oracle(ORC[conv]), case)


@pytest.mark.parametrize("n,m,B", [(1, 1, 1), (1, 16, 2), (31, 63, 1), (33, 65, 3), (100, 517, 2),
                                   (300, 2048, 1), (257, 4097, 4), (4000, 100, 1), (77, 11000, 1)])
def test_ragged_shapes(n, m, B):
    case = _dev(LayerCase(n, m, seed=n + 3 * m + B, dist=wi.UNIFORM3, B=B))
    for conv in (ww.CONV_EQ1, ww.CONV_ALG1):
        assert_parity(_tc(case, conv), case.oracle(ORC[conv]), case)


def test_per_tensor_scales_and_mixed_magnitudes():
    n, m, B = 200, 1000, 4
    x = wi.activations(9, m, B)
    x *= np.array([1e-3, 1e3, 1e-6, 30.0], np.float32)[:, None]  # per-vector E
    x[1].imag *= 1e-4                                         # per-component E
    case = _dev(LayerCase(n, m, seed=9, per_row=False, lo=0.5, hi=2.0, x=x, B=B))
    assert_parity(_tc(case, ww.CONV_EQ1), case.oracle(orc.CONV_EQ1), case)


def test_zero_weights_zero_x_and_unused_slot():
    n, m = 64, 256
    case = _dev(LayerCase(n, m, planes=np.zeros((4, n, m), np.int8), scales=np.ones((n, 4), np.float32)))
    assert not _tc(case, ww.CONV_EQ1).any()
    case = _dev(LayerCase(n, m, seed=3, x=np.zeros((1, m), np.complex64)))
    assert not _tc(case, ww.CONV_EQ1).any()
    # slot (1,1) (unused) contributes nothing (DESIGN R3)
    case = _dev(LayerCase(n, m, seed=4))
    ref = case.oracle(orc.CONV_EQ1)
    words = ww.pack_ternary(case.planes, ww.LAYOUT_TILE32)
    zero = (case.planes == 0)
    # turn every zero code of plane 0, row 5 into (1,1)
    W = (m + 15) // 16
    for j in np.nonzero(zero[0, 5])[0]:
        w = j // 16
        idx = ((0 * ((W + 3) // 4) + w // 4) * 128 + 4 * 5 + 0) * 4 + w % 4
        words[idx] |= np.uint32(3) << np.uint32(2 * (j % 16))
    case.packed_d = torch.from_numpy(words.view(np.uint8)).cuda()
    assert_parity(_tc(case, ww.CONV_EQ1), ref, case)


def test_workspace_stays_zero_and_results_repeat():
    case = _dev(LayerCase.from_spec(wi.C3B, seed=21))
    ws = ww.tcv_workspace(case.n, case.m, 1)
    y0 = _tc(case, ww.CONV_EQ1, ws)
    for _ in range(3):
        assert np.array_equal(_tc(case, ww.CONV_EQ1, ws), y0)
    assert not ws.any().item()
    # a different shape on the same (large enough) workspace
    small = _dev(LayerCase(300, 700, seed=2))
    ys = _tc(small, ww.CONV_ALG1, ws)
    assert_parity(ys, small.oracle(orc.CONV_ALG1), small)
    assert not ws.any().item()


def test_shard_invariance_bitwise():
    """A row shard of 32-aligned rows gives the same bits as the full layer (exact integer
    sums: the split of tiles across CTAs and the grid do not matter)."""
    case = _dev(LayerCase.from_spec(wi.C2, seed=8))
    y = _tc(case, ww.CONV_EQ1)[0]
    for r0, r1 in ((0, 1024), (1024, 2048), (96, 160), (2016, 2048)):
        sub = _dev(LayerCase(r1 - r0, case.m, planes=case.planes[:, r0:r1], scales=case.scales[r0:r1],
                             x=case.x))
        assert np.array_equal(_tc(sub, ww.CONV_EQ1)[0], y[r0:r1])


def test_matches_cuda_core_path_within_bar():
    case = LayerCase.from_spec(wi.C2, seed=3)
    ref = case.oracle(orc.CONV_EQ1)
    _dev(case)
    yt = _tc(case, ww.CONV_EQ1)
    case.device(ww, torch)
    yf = case.gpu(ww, torch, ww.CONV_EQ1)
    assert_parity(yt, ref, case)
    assert_parity(yf, ref, case)


@pytest.mark.parametrize("graph", [False, True])
def test_pdl_chain_reads_previous_output(graph):
    """y1 = L1(x), y2 = L2(y1), y3 = L3(y2) with WW_FLAG_PDL on one stream (eager and
    captured), bitwise equal to the same chain without PDL; y1 NaN-poisoned first."""
    n = m = 2048
    cases = [_dev(LayerCase(n, m, seed=40 + k)) for k in range(3)]
    x = cases[0].x_d[0]
    ws = ww.tcv_workspace(n, m, 1)

    def chain(flags, ys):
        s = torch.cuda.current_stream()
        inp = x
        for c, y in zip(cases, ys):
            ww.wl_gemv_tc(_layer(c, ww.CONV_EQ1, flags), c.packed_d, c.scales_d, inp, y, ws, stream=s)
            inp = y

    ref = [torch.empty(n, dtype=torch.complex64, device="cuda") for _ in range(3)]
    chain(0, ref)
    torch.cuda.synchronize()
    ys = [torch.full((n,), float("nan"), dtype=torch.complex64, device="cuda") for _ in range(3)]
    if graph:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            chain(ww.FLAG_PDL, ys)  # warm-up outside capture
            torch.cuda.synchronize()
            for y in ys:
                y.fill_(float("nan"))
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                chain(ww.FLAG_PDL, ys)
            g.replay()
        torch.cuda.synchronize()
    else:
        chain(ww.FLAG_PDL, ys)
        torch.cuda.synchronize()
    for a, b in zip(ys, ref):
        assert torch.equal(a.view(torch.float32), b.view(torch.float32))
    # the chain's first link against the oracle
    assert_parity(ref[0].cpu().numpy()[None], cases[0].oracle(orc.CONV_EQ1), cases[0])


def test_device_packer_tile32_matches_host():
    for n, m in ((2048, 5504), (33, 65), (300, 517)):
        planes = wi.planes(n + m, n, m, wi.LLAMA)
        want = ww.pack_ternary(planes, ww.LAYOUT_TILE32)
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        got = ww.pack_ternary_device(torch.from_numpy(planes).cuda(), bad=bad, layout=ww.LAYOUT_TILE32)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy().view(np.uint32), want)
        assert bad.item() == 0
    planes = wi.planes(1, 40, 70, wi.LLAMA)
    planes[2, 35, 20] = 5
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    got = ww.pack_ternary_device(torch.from_numpy(planes).cuda(), bad=bad, layout=ww.LAYOUT_TILE32)
    torch.cuda.synchronize()
    assert bad.item() == 1


def test_argument_errors():
    case = _dev(LayerCase(16, 32, seed=1, B=2))
    L = _layer(case, ww.CONV_EQ1)
    with pytest.raises(ValueError):
        ww.wl_gemv_tc(L, case.packed_d, case.scales_d, torch.zeros((5, 32), dtype=torch.complex64, device="cuda"))
    Lc = ww.Layer(16, 32, ww.LAYOUT_COL4)
    with pytest.raises(ValueError):
        ww.wl_gemv_tc(Lc, case.packed_d, case.scales_d, case.x_d)
