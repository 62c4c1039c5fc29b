"""NEXT-4: the paper's own CPU datapath (Algorithm 1, AVX-512F masked add/sub + BMI2 pext,
OpenMP row ranges) against the fp64 oracle at the north-star bar, both conventions, per-row
and per-tensor scales, ragged shapes; results independent of the thread count."""
import json
import os

import numpy as np
import pytest

import cpu_alg1
import oracle as orc
import ww_inputs as wi

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")

if not cpu_alg1.supported():  # pragma: no cover - depends on the host CPU
    pytest.skip("host CPU lacks AVX-512F / BMI2", allow_module_level=True)


def _case(n, m, seed, dist=wi.LLAMA, per_row=True, lo=0.01, hi=0.1):
    planes = wi.planes(seed, n, m, dist)
    sc = wi.scales(seed, n, per_row, lo, hi)
    x = wi.activations(seed, m, 1)
    return orc.pack_planar(planes), sc, x


@pytest.mark.parametrize("spec", [wi.C1, wi.C2], ids=lambda s: s.name)
@pytest.mark.parametrize("conv", [orc.CONV_EQ1, orc.CONV_ALG1])
def test_configs_match_oracle(spec, conv):
    pl, sc, x = _case(spec.n, spec.m, 3, spec.dist, spec.per_row, spec.scale_lo, spec.scale_hi)
    y = cpu_alg1.wl_gemv(pl, spec.n, spec.m, sc, x, conv)
    ok, rel, worst = orc.tolerance_check(y[None], orc.wl_direct(pl, spec.n, spec.m, sc, x, conv),
                                         sc, x)
    assert ok, (rel, worst)


@pytest.mark.parametrize("n,m", [(1, 1), (3, 15), (17, 17), (33, 100), (64, 5504)])
def test_ragged_shapes(n, m):
    pl, sc, x = _case(n, m, n + m, wi.UNIFORM3, False, 0.5, 2.0)
    for conv in (orc.CONV_EQ1, orc.CONV_ALG1):
        y = cpu_alg1.wl_gemv(pl, n, m, sc, x, conv)
        ok, rel, worst = orc.tolerance_check(y[None], orc.wl_direct(pl, n, m, sc, x, conv), sc, x)
        assert ok, (n, m, conv, rel, worst)


def test_thread_count_invariance():
    pl, sc, x = _case(517, 300, 9)
    ys = [cpu_alg1.wl_gemv(pl, 517, 300, sc, x, 0, t) for t in (1, 2, 3, 8)]
    for y in ys[1:]:
        assert np.array_equal(y, ys[0])


@pytest.mark.parametrize("ex", json.load(open(GOLDEN))["examples"], ids=lambda e: e["name"])
def test_worked_examples_exact(ex):
    # SPEC S:189 and the hand-worked 2x2 / 4x4 examples (tests/golden): dyadic, exact in fp32
    n, m = ex["n"], ex["m"]
    planes = np.stack([np.array(ex[p], np.int8) for p in ("U_re", "U_im", "W_re", "W_im")])
    sc = (np.array(ex["scales_per_row"], np.float32) if "scales_per_row" in ex
          else np.array(ex["scales_per_tensor"], np.float32))
    x = np.array([complex(a, b) for a, b in ex["x"]], np.complex64)
    for conv, key in ((0, "y_EQ1"), (1, "y_ALG1")):
        want = np.array([complex(a, b) for a, b in ex[key]], np.complex64)
        assert np.array_equal(cpu_alg1.wl_gemv(orc.pack_planar(planes), n, m, sc, x, conv), want)
