"""The config-4 decode stack exactly as bench.py times it (device-generated weights, device
packer, fused qkv / gate-up stages, PDL launches): sampled rows of every projection against
the oracle, row-sharded ranks (emulated on one GPU, exchange by copies) bitwise equal to one
rank, fused stages bitwise equal to one launch per projection, graph replay == eager."""
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


def test_stage_structure(stack2):
    names = [st.name for st in stack2.stages]
    assert names == ["qkv", "o", "gateup", "down"] * 2
    assert [st.n for st in stack2.stages[:4]] == [6144, 2048, 11008, 2048]
    assert [st.m for st in stack2.stages[:4]] == [2048, 2048, 2048, 5504]


def test_stack_sampled_rows_match_oracle(stack2):
    st_ = stack2
    with torch.cuda.stream(torch.cuda.Stream()):
        st_.step(torch.cuda.current_stream())
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    for st in st_.stages:
        x = wi.activations(st.x_seed, st.m, 1)
        for mb in st.members:
            spec = mb.spec
            rows = np.unique(np.concatenate([[0, spec.n - 1], rng.integers(0, spec.n, 10)]))
            planes = np.stack([wi.codes(mb.seed, q, spec.n, spec.m, spec.dist, row0=int(r),
                                        nrows=1)[0] for r in rows for q in range(4)])
            planes = np.ascontiguousarray(planes.reshape(len(rows), 4, spec.m).transpose(1, 0, 2))
            sc = wi.scales(mb.seed, spec.n, True, spec.scale_lo, spec.scale_hi)[rows]
            ref = orc.wl_direct(orc.pack_planar(planes), len(rows), spec.m, sc, x, orc.CONV_EQ1)
            got = st_.member_output(st, mb).cpu().numpy()[rows][None]
            ok, rel, worst = orc.tolerance_check(got, ref, sc, x)
            assert ok, (st.label, ww.stack.PROJ_NAMES[mb.proj], rel, worst)


def test_fused_stages_equal_one_launch_per_projection(stack2):
    # a row's arithmetic depends on (m, B) only, so stacking q/k/v (gate/up) rows into one
    # launch changes nothing bitwise
    un = WLStack(layers=1, seed=0, fuse=False)
    un.step()
    stack2.step()
    torch.cuda.synchronize()
    by_proj = {st.members[0].proj: un.gathered(st) for st in un.stages}
    for st in stack2.stages[:4]:
        for mb in st.members:
            assert torch.equal(stack2.member_output(st, mb), by_proj[mb.proj]), mb.proj


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_stack_equals_single_rank(stack2, world):
    ranks = [WLStack(layers=2, seed=0, rank=r, world=world) for r in range(world)]
    for st in ranks:
        st.step(exchange=False)
    stack2.step()
    torch.cuda.synchronize()
    for i, st in enumerate(stack2.stages):
        # emulated all-gather: copy every rank's slot into rank 0's gathered buffer
        y0 = ranks[0].Y[i]
        n = y0.numel() // world
        for r in range(1, world):
            y0[r * n:(r + 1) * n] = ranks[r].Y[i][r * n:(r + 1) * n]
        got = ranks[0].gathered(ranks[0].stages[i]).cpu().numpy()
        want = stack2.gathered(st).cpu().numpy()
        assert np.array_equal(got, want), st.label


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
