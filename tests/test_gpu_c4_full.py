"""Full-size parity of the headline configuration (only sampled rows had been
checked): every row of all 224 projections of the config-4 decode stack -- built exactly as
bench.py builds it (device-generated weights, device packer, fused q/k/v and gate/up stages,
PDL launches, one CUDA graph per token) -- against the fp64 oracle (unpack -> dense complex
rows -> Eq. 1), EQ1 on all 32 layers and ALG1 on one layer; and the persistent program
engine's plain chain bitwise equal to it.  The oracle side regenerates every code, scale and
activation on the host from the seeds (nothing flows from the GPU to the oracle)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as orc
import ww_inputs as wi

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_2604_20913_b200 as ww  # noqa: E402
from paper_2604_20913_b200.stack import PROJ_NAMES, WLStack, program_stages  # noqa: E402

THREADS = max(1, min(8, (os.cpu_count() or 1)))


def _graph_step(stack):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        stack.step(s)
    torch.cuda.synchronize()
    for y in stack.Y:
        y.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        stack.step(s)
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()


def _check_projection(args):
    st, mb, got, conv = args
    spec = mb.spec
    planes = wi.planes(mb.seed, spec.n, spec.m, spec.dist)
    sc = wi.scales(mb.seed, spec.n, True, spec.scale_lo, spec.scale_hi)
    x = wi.activations(st.x_seed, spec.m, 1)
    U, Wd = orc.build_dense(orc.pack_planar(planes), spec.n, spec.m, sc)
    ref = orc.eval_dense(U, Wd, x, conv)
    ok, rel, worst = orc.tolerance_check(got[None], ref, sc, x)
    return ok, rel, worst, f"{st.label}.{PROJ_NAMES[mb.proj]}"


def _check_stack(stack, conv):
    jobs = []
    for st in stack.stages:
        g = stack.gathered(st).cpu().numpy()
        for mb in st.members:
            jobs.append((st, mb, g[mb.row0:mb.row0 + mb.spec.n].copy(), conv))
    with ThreadPoolExecutor(THREADS) as ex:  # ctypes calls release the GIL
        res = list(ex.map(_check_projection, jobs))
    bad = [r for r in res if not r[0]]
    assert not bad, bad[:5]
    return len(res), max(r[1] for r in res), max(r[2] for r in res)


def test_c4_all_rows_all_projections_eq1():
    stack = WLStack(layers=wi.C4_LAYERS, seed=0)
    _graph_step(stack)
    nproj, rel, worst = _check_stack(stack, orc.CONV_EQ1)
    assert nproj == 224
    print(f"C4 EQ1: 224 projections, max rel L2 {rel:.2e}, max per-element ratio {worst:.3f}")
    # the persistent program engine (plain chain) computes the same bits
    prog = ww.Program([program_stages(stack, [stack], "plain")])
    ref = [y.clone() for y in stack.Y]
    for y in stack.Y:
        y.zero_()
    prog.run()
    torch.cuda.synchronize()
    for a, b in zip(ref, stack.Y):
        assert torch.equal(a, b)


def test_c4_one_layer_alg1():
    stack = WLStack(layers=1, seed=0, conv=ww.CONV_ALG1)
    _graph_step(stack)
    nproj, rel, worst = _check_stack(stack, orc.CONV_ALG1)
    assert nproj == 7


@pytest.mark.parametrize("lut,layers", [(("qkv", "gateup"), wi.C4_LAYERS), (("qkv", "o", "gateup", "down"), 2)])
def test_c4_lookup_stages_all_rows(lut, layers):
    """The stack as bench.py's default line runs it (qkv and gate/up on the lookup path,
    ww_wl_gemv_lut, the rest on the predicated-add kernel) -- and every stage on the lookup
    path -- against the oracle, every row of every projection, PDL launches in one graph."""
    stack = WLStack(layers=layers, seed=0, lut_stages=lut)
    _graph_step(stack)
    nproj, rel, worst = _check_stack(stack, orc.CONV_EQ1)
    assert nproj == 7 * layers
    print(f"C4 lookup {lut}: {nproj} projections, max rel L2 {rel:.2e}, max per-element ratio {worst:.3f}")
