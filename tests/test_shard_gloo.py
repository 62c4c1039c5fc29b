"""Row sharding + all-gather (the N > 1 path) with world_size 2 and 4 on CPU (gloo): each
rank computes only its ww_shard_plan rows (here with the oracle, since the CPU has no
kernel), the gathered vector equals the unsharded oracle output bitwise, for B = 1 and B > 1."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle as orc
import ww_inputs as wi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, m, B, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_2604_20913_b200 as ww
    from paper_2604_20913_b200.stack import exchange_shards, gathered_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = ww.shard_plan(n, m, world, rank)
        planes = wi.planes(9, n, m)
        scales = wi.scales(9, n, True, 0.01, 0.1)
        x = wi.activations(9, m, B)
        # this rank's rows only: COL4 slice -> planar via the library re-layout -> oracle
        nloc = sh.row_end - sh.row_begin
        y = torch.zeros(sh.n_padded * B, dtype=torch.complex128)
        if nloc:
            col4 = ww.pack_ternary(planes, ww.LAYOUT_COL4).view(np.uint8)
            local = col4[sh.packed_offset_bytes:sh.packed_offset_bytes + sh.packed_bytes].view(np.uint32)
            planar = ww.repack(local, nloc, m, ww.LAYOUT_COL4, ww.LAYOUT_PLANAR)
            sc = scales.reshape(-1)[sh.scale_offset_floats:sh.scale_offset_floats + sh.scale_count]
            yl = orc.wl_direct(planar, nloc, m, sc.reshape(nloc, 4), x, orc.CONV_EQ1)
            slot = y.view(world, B, sh.rows_per_rank)[rank]
            slot[:, :nloc] = torch.from_numpy(yl)
        exchange_shards(y, rank, world)
        full = orc.wl_direct(orc.pack_planar(planes), n, m, scales, x, orc.CONV_EQ1)
        ok = all(np.array_equal(gathered_rows(y, world, B, sh.rows_per_rank, n, b).numpy(), full[b])
                 for b in range(B))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,m,B", [(2, 37, 48, 1), (2, 64, 33, 3), (4, 10, 16, 1), (4, 3, 20, 2)])
def test_sharded_allgather_equals_unsharded(world, n, m, B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res
