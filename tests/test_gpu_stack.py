"""The config-4 decode stack exactly as bench.py times it (device-generated weights, device
packer, PDL launches): sampled rows of every projection shape against the oracle, and
row-sharded ranks (emulated on one GPU, exchange by copies) bitwise equal to one rank."""
import numpy as np
import pytest

import oracle as orc
import ww_inputs as wi

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_2604_20913_b200 as ww  # noqa: E402
from paper_2604_20913_b200.stack import WLStack  # noqa: E402


@pytest.fixture(scope="module")
def stack2():
    return WLStack(layers=2, seed=0)


def test_stack_sampled_rows_match_oracle(stack2):
    st = stack2
    with torch.cuda.stream(torch.cuda.Stream()):
        st.step(torch.cuda.current_stream())
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    for pr in st.projs:
        spec = pr.spec
        rows = np.unique(np.concatenate([[0, spec.n - 1], rng.integers(0, spec.n, 14)]))
        planes = np.stack([wi.codes(pr.seed, q, spec.n, spec.m, spec.dist, row0=int(r), nrows=1)[0]
                           for r in rows for q in range(4)]).reshape(len(rows), 4, spec.m)
        planes = np.ascontiguousarray(planes.transpose(1, 0, 2))
        sc = wi.scales(pr.seed, spec.n, True, spec.scale_lo, spec.scale_hi)[rows]
        x = wi.activations(pr.seed, spec.m, 1)
        ref = orc.wl_direct(orc.pack_planar(planes), len(rows), spec.m, sc, x, orc.CONV_EQ1)
        got = st.gathered(pr).cpu().numpy()[rows][None]
        ok, rel, worst = orc.tolerance_check(got, ref, sc, x)
        assert ok, (pr.name, rel, worst)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_stack_equals_single_rank(stack2, world):
    ranks = [WLStack(layers=2, seed=0, rank=r, world=world) for r in range(world)]
    for st in ranks:
        st.step(exchange=False)
    stack2.step()
    torch.cuda.synchronize()
    for i, pr in enumerate(stack2.projs):
        # emulated all-gather: copy every rank's slot into rank 0's gathered buffer
        y0 = ranks[0].Y[i]
        n = y0.numel() // world
        for r in range(1, world):
            y0[r * n:(r + 1) * n] = ranks[r].Y[i][r * n:(r + 1) * n]
        got = ranks[0].gathered(ranks[0].projs[i]).cpu().numpy()
        want = stack2.gathered(pr).cpu().numpy()
        assert np.array_equal(got, want), pr.name


def test_stack_graph_replay_equals_eager(stack2):
    st = stack2
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st.step(s)
    torch.cuda.synchronize()
    eager = [y.clone() for y in st.Y]
    for y in st.Y:
        y.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        st.step(s)
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, st.Y):
        assert torch.equal(a, b)
