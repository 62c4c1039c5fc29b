"""The persistent stage-chained program kernel (ww_program_*): plain config-4
stages bitwise equal to the per-launch kernel, the multi-rank protocol (fused all-gather by
direct stores + readiness counters) emulated as several ranks in ONE cooperative launch,
repeat launches / graph replays (epoch logic), and the NEXT-3 decode block against the fp64
oracle stage by stage."""
import numpy as np
import pytest

import oracle as orc
import ww_inputs as wi

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_2604_20913_b200 as ww  # noqa: E402
from paper_2604_20913_b200.stack import WLStack, block_gammas, program_stages  # noqa: E402


def _programs(layers, world, mode="plain", seed=0, gam=None):
    parts = [WLStack(layers=layers, seed=seed, rank=r, world=world) for r in range(world)]
    stages = [program_stages(p, parts, mode, gam) for p in parts]
    return parts, ww.Program(stages, world=world)


@pytest.fixture(scope="module")
def ref2():
    st = WLStack(layers=2, seed=0)
    st.step()
    torch.cuda.synchronize()
    return st


def test_plain_program_bitwise_equals_per_launch_stack(ref2):
    parts, prog = _programs(2, 1)
    info = prog.info()
    assert info["grid"] == torch.cuda.get_device_properties(0).multi_processor_count
    assert info["block"] == 17 * 32 and info["nslot"] >= 8
    prog.run()
    torch.cuda.synchronize()
    for i, st in enumerate(ref2.stages):
        assert torch.equal(parts[0].gathered(parts[0].stages[i]), ref2.gathered(st)), st.label


@pytest.mark.parametrize("world", [2, 3, 4])
def test_emulated_ranks_fused_allgather_bitwise(ref2, world):
    # `world` ranks' shards in one launch: every rank stores its rows into every rank's
    # gathered buffer and bumps every rank's counter; each rank's copy == the 1-rank result
    parts, prog = _programs(2, world)
    prog.run()
    torch.cuda.synchronize()
    for i, st in enumerate(ref2.stages):
        want = ref2.gathered(st)
        for g in range(world):
            assert torch.equal(parts[g].gathered(parts[g].stages[i]), want), (st.label, g)


def test_repeat_launches_and_graph_replay(ref2):
    # the readiness counters are never reset: each launch advances an epoch (ww.h)
    parts, prog = _programs(2, 2)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            prog.run(s)
    torch.cuda.synchronize()
    for y in parts[0].Y + parts[1].Y:
        y.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        prog.run(s)
    with torch.cuda.stream(s):
        for _ in range(4):
            g.replay()
    torch.cuda.synchronize()
    for i, st in enumerate(ref2.stages):
        for p in parts:
            assert torch.equal(p.gathered(p.stages[i]), ref2.gathered(st)), st.label


@pytest.mark.parametrize("n,m", [(1, 16), (100, 2048), (300, 5504), (5000, 512), (149, 11264)])
def test_single_stage_program_matches_oracle(n, m):
    # ragged CTA / warp row splits (n < #SMs, n not a multiple of 16), the widest x
    planes = wi.planes(n + m, n, m)
    scales = wi.scales(n + m, n, True, 0.01, 0.1)
    x = wi.activations(n + m, m)
    packed = torch.from_numpy(ww.pack_ternary(planes).view(np.uint8)).cuda()
    sc = torch.from_numpy(scales).cuda()
    xd = torch.from_numpy(x[0]).cuda()
    y = torch.full((n,), float("nan"), dtype=torch.complex64, device="cuda")
    for conv, oconv in ((ww.CONV_EQ1, orc.CONV_EQ1), (ww.CONV_ALG1, orc.CONV_ALG1)):
        st = ww.Stage(packed=packed, scales=sc, n_local=n, row0=0, m=m, x=xd, y=[y], conv=conv,
                      wait=0)
        ww.Program([[st]]).run()
        torch.cuda.synchronize()
        ref = orc.wl_direct(orc.pack_planar(planes), n, m, scales, x, oconv)
        ok, rel, worst = orc.tolerance_check(y.cpu().numpy()[None], ref, scales, x)
        assert ok, (rel, worst)
        y1 = ww.wl_gemv(ww.Layer(n, m, conv=conv), packed, sc, xd)
        torch.cuda.synchronize()
        assert torch.equal(y1, y)


# ---------------------------------------------------------------- NEXT-3 decode block

def _dense_layer(part, st, mb):
    spec = mb.spec
    planes = wi.planes(mb.seed, spec.n, spec.m, spec.dist)
    sc = wi.scales(mb.seed, spec.n, True, spec.scale_lo, spec.scale_hi)
    return orc.build_dense(orc.pack_planar(planes), spec.n, spec.m, sc), sc


def _check_stage(got, want, scales, x_eff, tag):
    # north-star bar (rel L2 <= 1e-5) plus the per-element bound on the effective x, with
    # 4 ulp of the output's own magnitude for the fused residual / SiLU (R11)
    err = got.astype(np.complex128) - want
    rel = np.linalg.norm(err) / max(np.linalg.norm(want), 1e-30)
    l1 = np.sum(np.abs(x_eff.real) + np.abs(x_eff.imag))
    bound = 1e-4 * scales.max(axis=1) * l1 + 4 * np.spacing(np.abs(want).astype(np.float32))
    worst = np.max(np.maximum(np.abs(err.real), np.abs(err.imag)) / bound)
    assert rel <= 1e-5 and worst <= 1.0, (tag, rel, worst)


@pytest.mark.parametrize("world,conv", [(1, 0), (2, 0), (1, 1)])
def test_decode_block_matches_oracle_stage_by_stage(world, conv):
    layers = 2
    gam_h = block_gammas(0, layers, 2048)
    gam = [tuple(torch.from_numpy(g).cuda() for g in pair) for pair in gam_h]
    parts = [WLStack(layers=layers, seed=0, rank=r, world=world, conv=conv) for r in range(world)]
    prog = ww.Program([program_stages(p, parts, "block", gam) for p in parts], world=world)
    prog.run()
    torch.cuda.synchronize()
    P = parts[0]
    Y = [P.gathered(st).cpu().numpy() for st in P.stages]
    for g in range(1, world):  # every rank holds the same gathered outputs
        for i, st in enumerate(parts[g].stages):
            assert np.array_equal(parts[g].gathered(st).cpu().numpy(), Y[i])
    h0 = P.x_of(P.stages[0])[0].cpu().numpy()
    for l in range(layers):
        dense = {}
        for st in P.stages[4 * l:4 * l + 4]:
            for mb in st.members:
                dense[ww.stack.PROJ_NAMES[mb.proj]] = (_dense_layer(P, st, mb), mb)
        h = h0 if l == 0 else Y[4 * l - 1]
        qkv, h1, gu, h2 = Y[4 * l:4 * l + 4]
        # each stage from the GPU's own input of that stage (errors do not compound)
        xa = orc.rmsnorm(h, gam_h[l][0])
        for name, lo in (("q", 0), ("k", 2048), ("v", 4096)):
            (UW, sc), _ = dense[name]
            _check_stage(qkv[lo:lo + 2048], orc.wl_dense_apply(*UW, xa, conv), sc, xa, f"L{l}.{name}")
        v = qkv[4096:6144]
        (UW, sc), _ = dense["o"]
        _check_stage(h1, orc.wl_dense_apply(*UW, v, conv) + h, sc, v, f"L{l}.o")
        xm = orc.rmsnorm(h1, gam_h[l][1])
        (UW, sc), _ = dense["gate"]
        _check_stage(gu[:5504], orc.silu_c(orc.wl_dense_apply(*UW, xm, conv)), sc, xm, f"L{l}.gate")
        (UW, sc), _ = dense["up"]
        _check_stage(gu[5504:11008], orc.wl_dense_apply(*UW, xm, conv), sc, xm, f"L{l}.up")
        a = orc.mul_c(gu[:5504], gu[5504:11008])
        (UW, sc), _ = dense["down"]
        _check_stage(h2, orc.wl_dense_apply(*UW, a, conv) + h1, sc, a, f"L{l}.down")
    # end to end over the two blocks from h0, fp64 oracle all the way (<= 1e-3)
    h = h0.astype(np.complex128)
    for l in range(layers):
        layer = {}
        for st in P.stages[4 * l:4 * l + 4]:
            for mb in st.members:
                layer[ww.stack.PROJ_NAMES[mb.proj]] = _dense_layer(P, st, mb)[0]
        h, _ = orc.block_forward(layer, h, gam_h[l], conv=conv)
    rel = np.linalg.norm(Y[-1] - h) / np.linalg.norm(h)
    assert rel <= 1e-5, rel


@pytest.mark.parametrize("world", [1, 2])
def test_per_stage_kernel_block_chain_bitwise_equals_program(world):
    # the same fused ops in the per-stage PDL kernel (ww_wl_gemv_fused) and in the program
    # kernel share their device code: the decode-block chain agrees bit for bit; at world 2
    # the per-stage ranks exchange by copies (NCCL is the product exchange, tested on >= 2 GPUs)
    layers = 2
    gam = [tuple(torch.from_numpy(g).cuda() for g in pair) for pair in block_gammas(3, layers, 2048)]
    ref = WLStack(layers=layers, seed=3)
    ww.Program([program_stages(ref, [ref], "block", gam)]).run()
    parts = [WLStack(layers=layers, seed=3, rank=r, world=world, chain="block", gammas=gam)
             for r in range(world)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(len(parts[0].stages)):
            for p in parts:
                p.launch(i, s)
            for p in parts:  # emulated all-gather of stage i
                n = p.Y[i].numel() // world
                for q in parts:
                    if q is not p:
                        q.Y[i][p.rank * n:(p.rank + 1) * n].copy_(p.Y[i][p.rank * n:(p.rank + 1) * n])
    torch.cuda.synchronize()
    for i, st in enumerate(ref.stages):
        for p in parts:
            assert torch.equal(p.gathered(p.stages[i]), ref.gathered(st)), (st.label, p.rank)


def test_fused_ops_argument_errors():
    case_n, m = 64, 2048
    packed = torch.zeros(ww.packed_bytes(case_n, m), dtype=torch.uint8, device="cuda")
    sc = torch.ones((case_n, 4), device="cuda")
    x = torch.zeros(m, dtype=torch.complex64, device="cuda")
    L = ww.Layer(case_n, m)
    with pytest.raises(ww.WWError) as e:  # MUL without its second operand
        ww.wl_gemv_fused(L, packed, sc, x, ops=ww.Ops(prologue=ww.PRO_MUL))
    assert e.value.status == ww.ERR_INVALID_ARGUMENT
    with pytest.raises(ww.WWError) as e:  # 16 does not divide m: no TMA staging
        L2 = ww.Layer(case_n, 100)
        ww.wl_gemv_fused(L2, packed, sc, x[:100], ops=ww.Ops(epilogue=ww.EPI_SILU, silu_rows=10))
    assert e.value.status == ww.ERR_MISALIGNED
    y = ww.wl_gemv_fused(L, packed, sc, x, ops=None)  # no ops == ww_wl_gemv
    torch.cuda.synchronize()
    assert not torch.view_as_real(y).any()


def test_program_per_tensor_scales_alg1_and_empty_shards():
    # per-tensor scales, ALG1, and a 3-row stage over 4 emulated ranks (rank 3 owns no rows)
    n, m, world = 3, 512, 4
    planes = wi.planes(41, n, m, wi.UNIFORM3)
    scales = wi.scales(41, n, False, 0.5, 2.0)
    x = wi.activations(41, m)
    packed = torch.from_numpy(ww.pack_ternary(planes).view(np.uint8)).cuda()
    sc = torch.from_numpy(scales).cuda()
    xd = torch.from_numpy(x[0]).cuda()
    ys = [torch.empty((4 * world,), dtype=torch.complex64, device="cuda") for _ in range(world)]
    for y in ys:
        torch.view_as_real(y).fill_(float("nan"))  # (torch.full with a complex nan: nan + 0j)
    stages = []
    for r in range(world):
        sh = ww.shard_plan(n, m, world, r)
        nl = sh.row_end - sh.row_begin
        pk = packed[sh.packed_offset_bytes:sh.packed_offset_bytes + max(sh.packed_bytes, 16)]
        stages.append([ww.Stage(packed=pk, scales=sc, n_local=nl, row0=sh.row_begin, m=m, x=xd,
                                y=ys, scale_mode=ww.SCALES_PER_TENSOR, conv=ww.CONV_ALG1, wait=0)])
    ww.Program(stages, world=world).run()
    torch.cuda.synchronize()
    ref = orc.wl_direct(orc.pack_planar(planes), n, m, scales, x, orc.CONV_ALG1)
    for g in range(world):
        got = ys[g][:n].cpu().numpy()[None]
        ok, rel, worst = orc.tolerance_check(got, ref, scales, x)
        assert ok, (g, rel, worst)
        assert torch.isnan(torch.view_as_real(ys[g][n:])).all()  # nothing written past n


def test_program_init_argument_errors():
    x = torch.zeros(2048, dtype=torch.complex64, device="cuda")
    y = torch.zeros(16, dtype=torch.complex64, device="cuda")
    pk = torch.zeros(ww.packed_bytes(16, 2048), dtype=torch.uint8, device="cuda")
    sc = torch.ones((16, 4), device="cuda")
    bad_m = ww.Stage(packed=pk, scales=sc, n_local=16, row0=0, m=100, x=x, y=[y], wait=0)
    with pytest.raises(ww.WWError) as e:
        ww.Program([[bad_m]])
    assert e.value.status == ww.ERR_INVALID_ARGUMENT
    mul_no_x2 = ww.Stage(packed=pk, scales=sc, n_local=16, row0=0, m=2048, x=x, y=[y], wait=0,
                         prologue=ww.PRO_MUL)
    with pytest.raises(ww.WWError) as e:
        ww.Program([[mul_no_x2]])
    assert e.value.status == ww.ERR_INVALID_ARGUMENT
    misaligned = ww.Stage(packed=pk[1:], scales=sc, n_local=16, row0=0, m=2048, x=x, y=[y], wait=0)
    with pytest.raises(ww.WWError) as e:
        ww.Program([[misaligned]])
    assert e.value.status == ww.ERR_MISALIGNED
