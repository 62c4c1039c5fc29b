"""Host-side logic of the G > 1 exchange, on CPU: the symmetric-buffer layout and peer
addressing used by the program kernel's fused all-gather (NEXT-1), and, across gloo ranks
(world 2 and 4), that every stage's row shards tile the stage exactly once with identical
gathered offsets on every rank."""
import os
import socket

import pytest
import torch.multiprocessing as mp

import ww_inputs as wi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_symm_layout_and_peer_address():
    from paper_2604_20913_b200.stack import SYNC_BYTES, peer_address, symm_layout
    counts = [6144, 2048, 11008, 2048]
    offs, sync_off, total = symm_layout(counts)
    assert offs[0] == 0 and all(o % 256 == 0 for o in offs) and sync_off % 256 == 0
    for o, c, nxt in zip(offs, counts, offs[1:] + [sync_off]):
        assert o + 8 * c <= nxt  # no overlap
    assert total == sync_off + SYNC_BYTES
    bases = [0x7F0000000000, 0x7E0000000000, 0x7D0000000000]
    for k, o in enumerate(offs):
        ptr = bases[0] + o + 40
        assert [peer_address(ptr, bases[0], b) - b for b in bases] == [o + 40] * 3
    with pytest.raises(AssertionError):
        peer_address(bases[0] - 8, bases[0], bases[1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_20913_b200 as ww
        from paper_2604_20913_b200.stack import FUSED_STAGES, symm_layout
        mine = []
        for name, projs in FUSED_STAGES:
            n = sum(wi.C4_PROJS[p].n for p in projs)
            m = wi.C4_PROJS[projs[0]].m
            sh = ww.shard_plan(n, m, world, rank)
            mine.append((name, n, sh.row_begin, sh.row_end, sh.y_offset_complex, sh.n_padded))
        counts = [r[5] for r in mine]
        allr = [None] * world
        dist.all_gather_object(allr, (mine, symm_layout(counts)))
        ok = all(a[1] == allr[0][1] for a in allr)  # the same symmetric layout on every rank
        for k, (name, n, *_rest) in enumerate(mine):
            rows = sorted((a[0][k][2], a[0][k][3]) for a in allr)
            cover = 0
            for lo, hi in rows:  # contiguous, disjoint, complete
                ok &= lo == min(cover, n) and hi >= lo
                cover = max(cover, hi)
            ok &= cover == n
            # each rank's rows land at its own gathered offset (rank-major slots)
            ok &= all(a[0][k][4] == r * (a[0][k][5] // world) for r, a in enumerate(allr))
        q.put((rank, bool(ok)))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_stage_shards_tile_rows_on_every_rank(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v is True for v in res.values()), res
