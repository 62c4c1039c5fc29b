"""The G > 1 paths on real GPUs: NCCL ranks, one process per GPU, spawned
here when >= 2 GPUs are visible (skipped below 2: a single GPU cannot host ranks that wait on
each other).  Row-sharded layers C2, C3b and C5 (B = 16) with the NCCL all-gather, the
config-4 stack (PDL launches + NCCL per stage) and the persistent program with its fused
all-gather (stores into every rank's symmetric-memory outputs + readiness counters): every
rank's gathered y is bitwise equal to the 1-GPU y, and the sharded layers pass the oracle bar."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs >= 2 CUDA devices", allow_module_level=True)
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORLD = min(torch.cuda.device_count(), 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layer_case(rank, world, spec, B, seed):
    import paper_2604_20913_b200 as ww
    import ww_inputs as wi
    from paper_2604_20913_b200.stack import exchange_shards, gathered_rows
    n, m = spec.n, spec.m
    planes = wi.planes(seed, n, m, spec.dist)
    scales = wi.scales(seed, n, True, spec.scale_lo, spec.scale_hi)
    x = wi.activations(seed, m, B)
    packed = torch.from_numpy(ww.pack_ternary(planes).view(np.uint8)).cuda()
    sc = torch.from_numpy(scales).cuda()
    X = torch.from_numpy(x).cuda()
    sh = ww.shard_plan(n, m, world, rank)
    nl = sh.row_end - sh.row_begin
    Yg = torch.zeros(sh.n_padded * B, dtype=torch.complex64, device="cuda")
    if nl:
        L = ww.Layer(nl, m)
        mine = Yg[rank * B * sh.rows_per_rank:(rank + 1) * B * sh.rows_per_rank].view(B, -1)
        ww.wl_gemv_batched(L, packed[sh.packed_offset_bytes:sh.packed_offset_bytes + sh.packed_bytes],
                           sc.reshape(-1)[sh.scale_offset_floats:sh.scale_offset_floats + sh.scale_count],
                           X, mine)
    exchange_shards(Yg, rank, world)
    got = np.stack([gathered_rows(Yg, world, B, sh.rows_per_rank, n, b).cpu().numpy()
                    for b in range(B)])
    full = ww.wl_gemv_batched(ww.Layer(n, m), packed, sc, X).cpu().numpy()
    return got, full, planes, scales, x


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        import oracle as orc
        import paper_2604_20913_b200 as ww
        import ww_inputs as wi
        from paper_2604_20913_b200.stack import WLStack, block_gammas, program_stages
        out = {}
        for name, spec, B in (("C2", wi.C2, 1), ("C3b", wi.C3B, 1), ("C5_B16", wi.C3B, 16)):
            got, full, planes, scales, x = _layer_case(rank, world, spec, B, 11)
            ok = np.array_equal(got, full)
            if rank == 0:
                ref = orc.wl_direct(orc.pack_planar(planes), spec.n, spec.m, scales, x)
                ok = ok and orc.tolerance_check(got, ref, scales, x)[0]
            out[name] = bool(ok)
        # config-4 stack, 2 layers: PDL launches + NCCL all-gather per stage
        st = WLStack(layers=2, seed=0, rank=rank, world=world)
        st.step()
        torch.cuda.synchronize()
        ref = WLStack(layers=2, seed=0)  # the 1-GPU stack on this rank's GPU
        ref.step()
        torch.cuda.synchronize()
        out["stack_nccl"] = all(torch.equal(st.gathered(a), ref.gathered(b))
                                for a, b in zip(st.stages, ref.stages))
        # persistent program, fused all-gather through symmetric memory (plain and block)
        gam = [tuple(torch.from_numpy(g).cuda() for g in p) for p in block_gammas(0, 2, 2048)]
        for chain in ("plain", "block"):
            sp = WLStack(layers=2, seed=0, rank=rank, world=world, symm=True)
            prog = ww.Program([program_stages(sp, None, chain, gam)], world=world, rank_base=rank,
                              sync=sp.symm.sync_ptrs())
            for _ in range(3):  # epochs advance per launch
                prog.run()
            torch.cuda.synchronize()
            dist.barrier()
            r1 = WLStack(layers=2, seed=0)
            ww.Program([program_stages(r1, [r1], chain, gam)]).run()
            torch.cuda.synchronize()
            out[f"program_{chain}"] = all(torch.equal(sp.gathered(a), r1.gathered(b))
                                          for a, b in zip(sp.stages, r1.stages))
        q.put((rank, out))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_multi_gpu_ranks_bitwise_equal_to_one_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in range(WORLD):
        assert isinstance(res[r], dict), res[r]
        assert all(res[r].values()), (r, res[r])
