"""Decode linear stack of BASELINE config 4: ``layers`` decoder layers x 7 widely-linear
projections (q, k, v, o: complex 2048->2048; gate, up: 2048->5504; down: 5504->2048), one
token (B vectors), output rows sharded over ``world`` GPUs with an all-gather after every
launch (north star).

Projections that read the same activation are one launch ("stage"), as a decode step runs
them: q, k and v share the normed hidden state, gate and up share the post-attention one.
A stage stacks its projections' rows (independent seeded weights and scales per projection),
so a layer is four dependent launches -- qkv (6144 x 2048), o (2048 x 2048), gate/up
(11008 x 2048), down (2048 x 5504) -- each followed by its all-gather.  ``fuse=False``
gives one stage per projection (seven launches per layer).

Host orchestration only: weights are drawn on the GPU by ``ww_inputs`` and packed by the
library's device packer; every stage runs in ``ww_wl_gemv_batched`` and every exchange is a
NCCL all-gather through ``torch.distributed``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import ww_inputs as wi

from . import (CONV_EQ1, FLAG_PDL, LAYOUT_COL4, LAYOUT_LUT81, SCALES_PER_ROW, Layer, launches_for_batch,
               packed_bytes, pack_ternary_device, shard_plan, wl_gemv_batched)

PROJ_NAMES = ("q", "k", "v", "o", "gate", "up", "down")
FUSED_STAGES = (("qkv", (0, 1, 2)), ("o", (3,)), ("gateup", (4, 5)), ("down", (6,)))
UNFUSED_STAGES = tuple((PROJ_NAMES[p], (p,)) for p in range(7))
# the projection whose seed draws a projection's input x: q, k, v read one activation and
# gate, up another, fused or not
X_GROUP = (0, 0, 0, 3, 4, 4, 6)


def exchange_shards(y, rank: int, world: int, group=None):
    """In-place all-gather of a rank-major gathered buffer y ([world][B][rows_per_rank]
    flattened): this rank's slot is the input, every rank ends with all slots (ww.h
    ww_shard_plan).  NCCL on GPUs, gloo on CPU (tests)."""
    if world == 1:
        return
    import torch.distributed as dist
    n = y.numel() // world
    dist.all_gather_into_tensor(y, y[rank * n:(rank + 1) * n], group=group)


def gathered_rows(y, world: int, B: int, rows_per_rank: int, n: int, b: int = 0):
    """Rows 0..n-1 of vector b from a rank-major gathered buffer."""
    return y.view(world, B, rows_per_rank)[:, b, :].reshape(-1)[:n]


@dataclass
class Member:
    """One projection inside a stage: its rows are [row0, row0 + spec.n) of the stage."""
    proj: int
    spec: object          # ww_inputs.LayerSpec
    seed: int             # per-projection seed (ww_inputs.layer_seed)
    row0: int


@dataclass
class Stage:
    layer: int
    name: str
    members: list
    n: int                # stacked rows of the stage
    m: int
    shard: object         # ww.Shard of this rank over the stage's n rows
    off: int = 0          # byte offset of the local packed rows in the weight buffer
    nbytes: int = 0
    soff: int = 0         # float offset of the local scales
    xoff: int = 0         # complex offset of the stage's input in X
    ylocal: int = 0       # local rows (may be 0)
    index: int = 0
    x_seed: int = 0       # seed of the stage's input activation (ww_inputs.activations)

    @property
    def label(self):
        return f"L{self.layer}.{self.name}"


SYNC_BYTES = 2048  # ww_program_sync_bytes()


def peer_address(local_ptr: int, local_base: int, peer_base: int) -> int:
    """The same byte of a symmetric buffer as mapped from another rank: buffers are laid out
    identically on every rank, so an offset from the local base is an offset from any peer's
    base."""
    assert local_ptr >= local_base
    return peer_base + (local_ptr - local_base)


def symm_layout(counts, align: int = 256):
    """Byte offsets of the per-stage gathered outputs (complex64 counts) and of the sync words
    inside one symmetric buffer; returns (offsets, sync_offset, total_bytes)."""
    offs, o = [], 0
    for c in counts:
        offs.append(o)
        o += (8 * c + align - 1) // align * align
    return offs, o, o + SYNC_BYTES


class SymmOutputs:
    """One symmetric-memory buffer per rank holding every stage's gathered output and the
    program's sync words; `bases[g]` = rank g's mapping of it (peer pointers, NVLink)."""

    def __init__(self, counts, device, group):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        offs, sync_off, total = symm_layout(counts)
        self.buf = symm_mem.empty(total, dtype=torch.uint8, device=device)
        self.buf.zero_()
        torch.cuda.synchronize(device)
        self.handle = symm_mem.rendezvous(self.buf, group if group is not None else dist.group.WORLD)
        self.bases = [int(p) for p in self.handle.buffer_ptrs]
        self.local = self.buf.data_ptr()
        self.views = [self.buf[o:o + 8 * c].view(torch.complex64) for o, c in zip(offs, counts)]
        self.sync_off = sync_off
        dist.barrier(group=group)

    def peer(self, t, g: int) -> int:
        return peer_address(t.data_ptr(), self.local, self.bases[g])

    def sync_ptrs(self):
        return [b + self.sync_off for b in self.bases]


class WLStack:
    """All stages of the stack resident in HBM on one rank (its row shard of every stage)."""

    def __init__(self, layers: int = wi.C4_LAYERS, seed: int = 0, B: int = 1, rank: int = 0,
                 world: int = 1, conv: int = CONV_EQ1, pdl: bool = True, device=None,
                 group=None, fuse: bool = True, chain: str = "plain", gammas=None,
                 symm: bool = False, lut_stages=()):
        """chain "plain": every stage reads its own seeded x; "block": the NEXT-3 decode-block
        chain (block_inputs), stage inputs are earlier stages' gathered outputs, with the
        fused RMSNorm / SiLU / (.) / residual ops of ww_wl_gemv_fused (B = 1, fuse = True).
        lut_stages: names of the stages (B = 1, plain chain) that run on the lookup path
        (ww_wl_gemv_lut, WW_LAYOUT_LUT81 weights) instead of the predicated-add kernel."""
        self.lut_stages = frozenset(lut_stages)
        if self.lut_stages:
            assert B == 1 and chain == "plain", "the lookup path is B = 1, plain chain"
        self.layers, self.seed, self.B, self.rank, self.world = layers, seed, B, rank, world
        self.conv, self.group, self.chain, self.gammas = conv, group, chain, gammas
        if chain == "block":
            assert B == 1 and fuse and gammas is not None
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.flags = FLAG_PDL if pdl else 0
        self.stages: list[Stage] = []
        off = soff = xoff = 0
        for l in range(layers):
            for name, projs in (FUSED_STAGES if fuse else UNFUSED_STAGES):
                members, r0 = [], 0
                for p in projs:
                    spec = wi.C4_PROJS[p]
                    members.append(Member(p, spec, wi.layer_seed(seed, l, p), r0))
                    r0 += spec.n
                m = members[0].spec.m
                sh = shard_plan(r0, m, world, rank)
                nloc = sh.row_end - sh.row_begin
                lay = LAYOUT_LUT81 if name in self.lut_stages else LAYOUT_COL4
                st = Stage(l, name, members, r0, m, sh, off, nloc * packed_bytes(1, m, lay), soff,
                           xoff, nloc, len(self.stages),
                           wi.layer_seed(seed, l, X_GROUP[projs[0]]))
                self.stages.append(st)
                off += st.nbytes
                soff += 4 * nloc
                xoff += B * m
        self.weight_bytes = off
        self.W = torch.empty(max(off, 16), dtype=torch.uint8, device=self.device)
        self.S = torch.empty(max(soff, 4), dtype=torch.float32, device=self.device)
        self.X = torch.empty(max(xoff, 1), dtype=torch.complex64, device=self.device)
        # gathered outputs: [world][B][rows_per_rank] per stage (rank-major, ww.h); with
        # symm=True they (and the program's readiness words) live in ONE symmetric-memory
        # buffer every rank maps (torch.distributed._symmetric_memory), so the program kernel
        # can store rows straight into every peer's copy (fused all-gather, NEXT-1)
        counts = [st.shard.n_padded * B for st in self.stages]
        self.symm = None
        if symm:
            self.symm = SymmOutputs(counts, self.device, group)
            self.Y = self.symm.views
        else:
            self.Y = [torch.zeros(c, dtype=torch.complex64, device=self.device) for c in counts]
        self._fill()

    # ------------------------------------------------------------------ inputs
    def _fill(self):
        xs_host = np.empty(self.X.numel(), dtype=np.complex64)
        for st in self.stages:
            rb, re = st.shard.row_begin, st.shard.row_end
            if st.ylocal:
                planes = torch.empty((4, st.ylocal, st.m), dtype=torch.int8, device=self.device)
                scales = np.empty((st.ylocal, 4), dtype=np.float32)
                for mb in st.members:
                    lo, hi = max(rb, mb.row0), min(re, mb.row0 + mb.spec.n)
                    if lo >= hi:
                        continue
                    for q in range(4):
                        wi.codes_device(mb.seed, q, hi - lo, st.m, planes[q, lo - rb:hi - rb],
                                        mb.spec.dist, row0=lo - mb.row0)
                    sc = wi.scales(mb.seed, mb.spec.n, mb.spec.per_row, mb.spec.scale_lo,
                                   mb.spec.scale_hi)
                    scales[lo - rb:hi - rb] = sc[lo - mb.row0:hi - mb.row0]
                pack_ternary_device(planes, out=self.W[st.off:st.off + st.nbytes],
                                    layout=LAYOUT_LUT81 if st.name in self.lut_stages else LAYOUT_COL4)
                self.S[st.soff:st.soff + 4 * st.ylocal] = torch.from_numpy(scales.reshape(-1))
            xs_host[st.xoff:st.xoff + self.B * st.m] = wi.activations(st.x_seed, st.m,
                                                                      self.B).reshape(-1)
        self.X.copy_(torch.from_numpy(xs_host))
        torch.cuda.synchronize(self.device)

    def inputs(self):
        """The step's host-fed inputs: every stage's x (plain), or h_0 alone (block chain)."""
        return self.X if self.chain == "plain" else self.X[:self.stages[0].m]

    def x_of(self, st: Stage):
        return self.X[st.xoff:st.xoff + self.B * st.m].view(self.B, st.m)

    def y_local_view(self, st: Stage):
        """This rank's [B][rows_per_rank] slot of the gathered output (first ylocal rows used)."""
        rpr = st.shard.rows_per_rank
        base = self.rank * self.B * rpr
        return self.Y[st.index][base:base + self.B * rpr].view(self.B, rpr)

    def gathered(self, st: Stage, b: int = 0):
        """Full output y[b] (all n rows of the stage) after the all-gather."""
        return gathered_rows(self.Y[st.index], self.world, self.B, st.shard.rows_per_rank, st.n, b)

    def member_output(self, st: Stage, mb: Member, b: int = 0):
        """Projection mb's output rows inside the stage's gathered output."""
        return self.gathered(st, b)[mb.row0:mb.row0 + mb.spec.n]

    # ------------------------------------------------------------------ the step
    def launch(self, i: int, stream=None):
        """Stage i on this rank: WL-GEMV of the local rows into the gathered slot."""
        st = self.stages[i]
        if not st.ylocal:
            return 0
        L = Layer(st.ylocal, st.m, LAYOUT_COL4, SCALES_PER_ROW, self.conv, self.flags)
        if self.chain == "block":
            from . import Ops, wl_gemv_fused
            kw = block_inputs(self, i, self.gammas)
            x = kw.pop("x")
            wl_gemv_fused(L, self.W[st.off:st.off + st.nbytes],
                          self.S[st.soff:st.soff + 4 * st.ylocal], x,
                          self.y_local_view(st)[0], Ops(row0=st.shard.row_begin, **kw),
                          stream=stream)
            return 1
        if st.name in self.lut_stages:
            from . import wl_gemv_lut
            L.layout = LAYOUT_LUT81
            wl_gemv_lut(L, self.W[st.off:st.off + st.nbytes], self.S[st.soff:st.soff + 4 * st.ylocal],
                        self.x_of(st)[0], self.y_local_view(st)[0][:st.ylocal], stream=stream)
            return 1
        wl_gemv_batched(L, self.W[st.off:st.off + st.nbytes],
                        self.S[st.soff:st.soff + 4 * st.ylocal], self.x_of(st),
                        self.y_local_view(st), stream=stream)
        return launches_for_batch(self.B)

    def exchange(self, i: int):
        """All-gather of stage i's y shards (NCCL over NVLink); no-op on one rank."""
        if self.world == 1:
            return 0
        exchange_shards(self.Y[i], self.rank, self.world, self.group)
        return 1

    def step(self, stream=None, exchange: bool = True):
        """One token through the whole stack; returns the number of WL-GEMV launches.
        exchange=False skips the all-gathers (tests emulating ranks on one GPU)."""
        k = 0
        for i in range(len(self.stages)):
            k += self.launch(i, stream)
            if exchange:
                self.exchange(i)
        return k

    # ------------------------------------------------------------------ accounting
    def algorithmic_bytes(self) -> int:
        """Bytes the method must move on this rank per step: packed rows + x + y + scales."""
        t = 0
        for st in self.stages:
            if st.ylocal:
                t += st.nbytes + 8 * st.m * self.B + 8 * st.ylocal * self.B + 16 * st.ylocal
        return t

    def packed_act_bytes(self) -> int:
        """North-star roofline bytes: packed weights + activation (x) bytes on this rank."""
        return sum(st.nbytes + 8 * st.m * self.B for st in self.stages if st.ylocal)

    def adds(self) -> int:
        """Algorithmic fp32 add/sub count on this rank (8 per complex column per row, App. D)."""
        return sum(8 * st.ylocal * st.m * self.B for st in self.stages)


# ------------------------------------------------------------------ persistent program
EPS = 1e-5


def block_gammas(seed: int, layers: int, m: int):
    """RMSNorm weights of the decode blocks (NEXT-3): per layer gamma_attn and gamma_mlp, each
    2m fp32 (the real 2m-vector view), seeded ~ U[0.5, 1.5] (DESIGN.md input recipe)."""
    out = []
    for l in range(layers):
        pair = []
        for k in range(2):
            s = wi.layer_seed(seed ^ 0x5EED, l, 100 + k)
            pair.append(np.ascontiguousarray(wi.scales(s, m // 2, True, 0.5, 1.5).reshape(-1)))
        out.append(tuple(pair))
    return out


def block_inputs(part: "WLStack", i: int, gammas, x0=None) -> dict:
    """Input and fused ops of stage i in the NEXT-3 decode-block chain, on this
    rank's copies of the gathered outputs (part.Y): per layer l
      qkv   x = RMSNorm(h_l; gamma_attn)            -> QKV_l
      o     x = v = QKV_l[4096:6144], + residual h_l -> H1_l   (attention = identity on v)
      gateup x = RMSNorm(H1_l; gamma_mlp), SiLU on the gate rows -> GU_l
      down  x = SiLU(gate) (.) up = GU_l[:5504] (.) GU_l[5504:], + residual H1_l -> h_{l+1}
    with h_0 = x0 (default: stage 0's seeded x).  Returns x and the ww_ops fields."""
    from . import EPI_RESIDUAL, EPI_SILU, PRO_MUL, PRO_RMSNORM
    st = part.stages[i]
    Yl = part.Y
    l = st.layer
    base = 4 * l
    h_l = (x0 if x0 is not None else part.x_of(part.stages[0])[0]) if l == 0 else Yl[base - 1]
    if st.name == "qkv":
        return dict(x=h_l, prologue=PRO_RMSNORM, gamma=gammas[l][0], eps=EPS)
    if st.name == "o":
        return dict(x=Yl[base][4096:6144], epilogue=EPI_RESIDUAL, residual=h_l)
    if st.name == "gateup":
        return dict(x=Yl[base + 1], prologue=PRO_RMSNORM, gamma=gammas[l][1], eps=EPS,
                    epilogue=EPI_SILU, silu_rows=5504)
    if st.name == "down":
        return dict(x=Yl[base + 2][:5504], x2=Yl[base + 2][5504:11008], prologue=PRO_MUL,
                    epilogue=EPI_RESIDUAL, residual=Yl[base + 1])
    raise ValueError(st.name)


def program_stages(part: "WLStack", parts: list, mode: str = "plain", gammas=None,
                   x0=None):
    """ww_stage list of one rank (`part`) for a persistent program over its WLStack; the
    gathered outputs of rank g live in parts[g].Y.  mode "plain": every stage reads its own
    seeded x (BASELINE config 4 as round 1 timed it) and waits for the previous stage;
    mode "block": the NEXT-3 decode block chain -- per layer
      qkv   x = RMSNorm(h_l; gamma_attn)            -> QKV_l
      o     x = v = QKV_l[4096:6144], + residual h_l -> H1_l
      gateup x = RMSNorm(H1_l; gamma_mlp), SiLU on the gate rows -> GU_l
      down  x = SiLU(gate) (.) up = GU_l[:5504] (.) GU_l[5504:], + residual H1_l -> h_{l+1}
    with h_0 = x0 (default: stage 0's seeded x).  gammas: block_gammas() as device tensors."""
    from . import SCALES_PER_ROW, Stage
    world = part.world
    assert part.B == 1
    st_list = []
    for i, st in enumerate(part.stages):
        if parts is None:  # one rank per process: peer-mapped symmetric outputs
            ys = [part.symm.peer(part.Y[i], g) for g in range(world)]
        else:  # every rank's buffers in this process (one-GPU emulation)
            assert len(parts) == world
            ys = [parts[g].Y[i] for g in range(world)]
        kw = dict(packed=part.W[st.off:st.off + max(st.nbytes, 16)],
                  scales=part.S[st.soff:st.soff + max(4 * st.ylocal, 4)],
                  n_local=st.ylocal, row0=st.shard.row_begin, m=st.m, y=ys,
                  scale_mode=SCALES_PER_ROW, conv=part.conv, wait=1 if i > 0 else 0)
        if mode == "plain":
            kw.update(x=part.x_of(st)[0])
        elif mode == "block":
            kw.update(block_inputs(part, i, gammas, x0))
        else:
            raise ValueError(mode)
        st_list.append(Stage(**kw))
    return st_list
