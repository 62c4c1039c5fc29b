"""WL-GEMV by ternary subset-sum lookup (ww_wl_gemv_lut, WW_LAYOUT_LUT81, B = 1) against the
fp64 oracle at the north-star bar: BASELINE configs 1-3 at full size for both conventions,
ragged shapes (m not a multiple of 4 / 128 / 512, one and several CTAs per cluster, more
clusters than rows), per-tensor scales, zero weights and zero x, PDL chains reading the
previous launch's output, determinism and independence of the row shard."""
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
    case.packed_d = torch.from_numpy(ww.pack_lut81(case.planes)).cuda()
    case.scales_d = torch.from_numpy(np.ascontiguousarray(case.scales)).cuda()
    case.x_d = torch.from_numpy(np.ascontiguousarray(case.x)).cuda()
    return case


def _layer(case, conv, flags=0):
    return ww.Layer(case.n, case.m, ww.LAYOUT_LUT81,
                    ww.SCALES_PER_ROW if case.per_row else ww.SCALES_PER_TENSOR, conv, flags)


def _lut(case, conv, flags=0):
    y = ww.wl_gemv_lut(_layer(case, conv, flags), case.packed_d, case.scales_d, case.x_d[0])
    torch.cuda.synchronize()
    return y.cpu().numpy()[None, :]


@pytest.mark.parametrize("spec", [wi.C1, wi.C2, wi.C3A, wi.C3B], ids=["C1", "C2", "C3a", "C3b"])
@pytest.mark.parametrize("conv", [ww.CONV_EQ1, ww.CONV_ALG1])
def test_configs_full_size(spec, conv):
    case = _dev(LayerCase.from_spec(spec, seed=11))
    assert_parity(_lut(case, conv), case.oracle(ORC[conv]), case)


@pytest.mark.parametrize("n,m", [(1, 1), (1, 16), (3, 5), (31, 63), (33, 129), (100, 517), (300, 1024),
                                 (300, 1025), (257, 4097), (4000, 100), (77, 8192), (150, 333),
                                 (6144, 2048), (11008, 2048)])
def test_ragged_shapes(n, m):
    case = _dev(LayerCase(n, m, seed=n + 3 * m, dist=wi.UNIFORM3))
    for conv in (ww.CONV_EQ1, ww.CONV_ALG1):
        assert_parity(_lut(case, conv), case.oracle(ORC[conv]), case)


def test_per_tensor_scales():
    case = _dev(LayerCase(200, 1000, seed=9, per_row=False, lo=0.5, hi=2.0))
    assert_parity(_lut(case, ww.CONV_EQ1), case.oracle(orc.CONV_EQ1), case)


def test_zero_weights_and_zero_x():
    n, m = 64, 1300
    case = _dev(LayerCase(n, m, planes=np.zeros((4, n, m), np.int8), scales=np.ones((n, 4), np.float32)))
    assert not _lut(case, ww.CONV_EQ1).any()
    case = _dev(LayerCase(n, m, seed=3, x=np.zeros((1, m), np.complex64)))
    assert not _lut(case, ww.CONV_EQ1).any()


def test_single_code_brute_force():
    """One nonzero code at a time: y_i is +-s x_j (or +-i s x_j) exactly -- catches a wrong
    digit weight, block or lane in the table layout."""
    n, m = 4, 1100
    x = wi.activations(1, m, 1)
    for (p, i, j, c) in [(0, 0, 0, 1), (1, 1, 3, -1), (2, 2, 517, 1), (3, 3, 1099, -1), (0, 3, 130, -1),
                         (2, 0, 1023, -1), (1, 2, 1024, 1)]:
        planes = np.zeros((4, n, m), np.int8)
        planes[p, i, j] = c
        case = _dev(LayerCase(n, m, planes=planes, scales=np.full((n, 4), 0.5, np.float32), x=x))
        y = _lut(case, ww.CONV_EQ1)
        assert_parity(y, case.oracle(orc.CONV_EQ1), case)
        assert np.count_nonzero(y) == 1


def test_deterministic_and_shard_invariant():
    case = _dev(LayerCase(1000, 2048, seed=4))
    y0 = _lut(case, ww.CONV_EQ1)
    assert np.array_equal(y0, _lut(case, ww.CONV_EQ1))
    r0, r1 = 137, 800  # a row shard is the same rows of the packed buffer
    T = (case.m + 511) // 512
    sub = LayerCase(r1 - r0, case.m, planes=case.planes[:, r0:r1], scales=case.scales[r0:r1], x=case.x)
    sub.packed_d = case.packed_d[r0 * T * 512:r1 * T * 512]
    sub.scales_d = case.scales_d[r0:r1].contiguous()
    sub.x_d = case.x_d
    assert np.array_equal(_lut(sub, ww.CONV_EQ1), y0[:, r0:r1])


@pytest.mark.parametrize("graph", [False, True])
def test_pdl_chain_reads_previous_output(graph):
    """y1 = L1(x); y2 = L2(y1) with WW_FLAG_PDL on one stream equals the chain without PDL."""
    a = _dev(LayerCase(2048, 1024, seed=21))
    b = _dev(LayerCase(700, 2048, seed=22))
    outs = []
    for flags in (0, ww.FLAG_PDL):
        y1 = torch.full((a.n,), float("nan"), dtype=torch.complex64, device="cuda")
        y2 = torch.full((b.n,), float("nan"), dtype=torch.complex64, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            def run():
                ww.wl_gemv_lut(_layer(a, ww.CONV_EQ1, flags), a.packed_d, a.scales_d, a.x_d[0], y1, stream=s)
                ww.wl_gemv_lut(_layer(b, ww.CONV_EQ1, flags), b.packed_d, b.scales_d, y1, y2, stream=s)
            if graph and flags:
                run()
                s.synchronize()
                y1.fill_(float("nan"))
                y2.fill_(float("nan"))
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    run()
                g.replay()
            else:
                run()
        s.synchronize()
        torch.cuda.synchronize()
        outs.append(y2.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    assert np.isfinite(outs[0].view(np.float32)).all()


def test_argument_errors():
    case = _dev(LayerCase(8, 64, seed=1))
    with pytest.raises(ValueError):
        ww.wl_gemv_lut(ww.Layer(8, 64, ww.LAYOUT_COL4), case.packed_d, case.scales_d, case.x_d[0])
    with pytest.raises(ww.WWError):  # unknown convention
        ww.wl_gemv_lut(ww.Layer(8, 64, ww.LAYOUT_LUT81, conv=7), case.packed_d, case.scales_d, case.x_d[0])
    big = ww.Layer(8, 9000, ww.LAYOUT_LUT81)
    with pytest.raises(ww.WWError):
        ww.wl_gemv_lut(big, torch.zeros(ww.lut81_packed_bytes(8, 9000), dtype=torch.uint8, device="cuda"),
                       torch.ones(32, device="cuda"), torch.zeros(9000, dtype=torch.complex64, device="cuda"))


@pytest.mark.parametrize("n,m", [(5, 7), (33, 517), (64, 2048), (100, 5504)])
def test_device_packer_equals_host_packer(n, m):
    planes = wi.planes(n * m, n, m, wi.UNIFORM3)
    d = ww.pack_ternary_device(torch.from_numpy(planes).cuda(), layout=ww.LAYOUT_LUT81)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ww.pack_lut81(planes))


def test_device_packer_flags_invalid_value():
    planes = np.zeros((4, 3, 40), np.int8)
    planes[2, 1, 9] = 2
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    d = ww.pack_ternary_device(torch.from_numpy(planes).cuda(), bad=bad, layout=ww.LAYOUT_LUT81)
    torch.cuda.synchronize()
    assert int(bad.item()) != 0
    assert (d.cpu().numpy() == 40).all()  # the invalid value packs as the zero code
