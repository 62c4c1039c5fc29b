"""Tensor-core path of the batched WL-GEMV (ww_wl_gemv_batched_tc, WW_LAYOUT_TILE32 weights:
tcgen05 kind::i8 MMAs on
in-kernel decoded int8 planes and 3-limb fixed-point x) against the fp64 oracle at the
north-star bar: BASELINE config 5 (down shape) for B = 8 and 16, both conventions, ragged
shapes (n not a multiple of the 32-row tile, m not a multiple of the 128-column block),
per-tensor scales, every B up to the limit, and x vectors of very different magnitudes."""
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


def _t32(case):
    """The case on the device with its weights in WW_LAYOUT_TILE32 (the layout of this path)."""
    case.device(ww, torch)
    case.packed_d = torch.from_numpy(ww.pack_ternary(case.planes, ww.LAYOUT_TILE32).view(np.uint8)).cuda()
    return case


def _layer(case, conv):
    return ww.Layer(case.n, case.m, ww.LAYOUT_TILE32,
                    ww.SCALES_PER_ROW if case.per_row else ww.SCALES_PER_TENSOR, conv)


def _tc(case, conv):
    L = _layer(case, conv)
    y = ww.wl_gemv_batched_tc(L, case.packed_d, case.scales_d, case.x_d)
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("B", [8, 16])
@pytest.mark.parametrize("conv", [ww.CONV_EQ1, ww.CONV_ALG1])
def test_config5_tensor_core_full(B, conv):
    case = _t32(LayerCase.from_spec(wi.C3B, seed=5, B=B))
    assert_parity(_tc(case, conv), case.oracle(ORC[conv]), case)


@pytest.mark.parametrize("n,m,B", [(1, 16, 1), (33, 100, 3), (300, 517, 5), (77, 2048, 7),
                                   (2048, 2048, 12), (129, 5504, 16)])
def test_ragged_shapes_and_batches(n, m, B):
    case = _t32(LayerCase(n, m, seed=n + m + B, dist=wi.UNIFORM3, B=B))
    for conv in (ww.CONV_EQ1, ww.CONV_ALG1):
        assert_parity(_tc(case, conv), case.oracle(ORC[conv]), case)


def test_per_tensor_scales_and_mixed_magnitudes():
    n, m, B = 200, 1000, 6
    x = wi.activations(9, m, B)
    x *= np.array([1e-3, 1.0, 1e3, 5.0, 1e-6, 30.0], np.float32)[:, None]  # per-vector E
    x[2].imag *= 1e-4                                                     # per-component E
    case = _t32(LayerCase(n, m, seed=9, per_row=False, lo=0.5, hi=2.0, x=x, B=B))
    assert_parity(_tc(case, ww.CONV_EQ1), case.oracle(orc.CONV_EQ1), case)


def test_zero_weights_and_zero_x():
    n, m, B = 64, 256, 8
    planes = np.zeros((4, n, m), np.int8)
    case = _t32(LayerCase(n, m, planes=planes, scales=np.ones((n, 4), np.float32), B=B))
    assert not _tc(case, ww.CONV_EQ1).any()
    case = _t32(LayerCase(n, m, seed=3, x=np.zeros((B, m), np.complex64), B=B))
    assert not _tc(case, ww.CONV_EQ1).any()


def test_argument_errors():
    case = _t32(LayerCase(16, 32, seed=1, B=2))
    L = _layer(case, ww.CONV_EQ1)
    X = torch.zeros((17, 32), dtype=torch.complex64, device="cuda")
    with pytest.raises(ValueError):
        ww.wl_gemv_batched_tc(L, case.packed_d, case.scales_d, X)
    assert ww.tc_workspace_bytes(16, 32, 17) == 0 and ww.tc_workspace_bytes(2048, 5504, 16) > 0


def test_split_k_workspace_reuse_and_repeat():
    """Config 5 splits each 32-row tile's K range over several CTAs (64 tiles < 148 SMs): the
    partial sums meet in the workspace, which every call must leave zeroed; repeated calls on
    one workspace give identical bits, and so do other batch sizes sharing it."""
    case = _t32(LayerCase.from_spec(wi.C3B, seed=17, B=16))
    L = _layer(case, ww.CONV_EQ1)
    nb = ww.tc_workspace_bytes(case.n, case.m, 16)
    ws = torch.zeros(nb + 256, dtype=torch.uint8, device="cuda")
    y0 = ww.wl_gemv_batched_tc(L, case.packed_d, case.scales_d, case.x_d, workspace=ws).cpu().numpy()
    for _ in range(2):
        y1 = ww.wl_gemv_batched_tc(L, case.packed_d, case.scales_d, case.x_d, workspace=ws).cpu().numpy()
        assert np.array_equal(y0, y1)
    assert_parity(y0, case.oracle(orc.CONV_EQ1), case)
    y8 = ww.wl_gemv_batched_tc(L, case.packed_d, case.scales_d, case.x_d[:8], workspace=ws).cpu().numpy()
    assert np.array_equal(y8, y0[:8])
