"""Decode linear stack of BASELINE config 4: ``layers`` decoder layers x 7 widely-linear
projections (q, k, v, o: complex 2048->2048; gate, up: 2048->5504; down: 5504->2048), one
token (B vectors), output rows sharded over ``world`` GPUs with an all-gather of every
projection's y (north star).

Host orchestration only: weights are drawn on the GPU by ``ww_inputs`` and packed by the
library's device packer; every projection runs in ``ww_wl_gemv`` / ``ww_wl_gemv_batched``
and every exchange is a NCCL all-gather through ``torch.distributed``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import ww_inputs as wi

from . import (CONV_EQ1, FLAG_PDL, LAYOUT_COL4, SCALES_PER_ROW, Layer, packed_bytes,
               pack_ternary_device, shard_plan, wl_gemv_batched)

PROJ_NAMES = ("q", "k", "v", "o", "gate", "up", "down")


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
class Proj:
    layer: int
    proj: int
    spec: object          # ww_inputs.LayerSpec
    seed: int             # per-projection seed (ww_inputs.layer_seed)
    shard: object         # ww.Shard of this rank
    off: int              # byte offset of the local packed rows in the weight buffer
    nbytes: int           # local packed bytes
    soff: int             # float offset of the local scales
    xoff: int             # complex offset of this projection's input in X
    ylocal: int           # local rows (may be 0)

    @property
    def name(self):
        return f"L{self.layer}.{PROJ_NAMES[self.proj]}"


class WLStack:
    """All projections of the stack resident in HBM on one rank (its row shard)."""

    def __init__(self, layers: int = wi.C4_LAYERS, seed: int = 0, B: int = 1, rank: int = 0,
                 world: int = 1, conv: int = CONV_EQ1, pdl: bool = True, device=None,
                 group=None):
        self.layers, self.seed, self.B, self.rank, self.world = layers, seed, B, rank, world
        self.conv, self.group = conv, group
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.flags = FLAG_PDL if pdl else 0
        self.projs: list[Proj] = []
        off = soff = xoff = 0
        for l in range(layers):
            for p, spec in enumerate(wi.C4_PROJS):
                sh = shard_plan(spec.n, spec.m, world, rank)
                nloc = sh.row_end - sh.row_begin
                self.projs.append(Proj(l, p, spec, wi.layer_seed(seed, l, p), sh, off,
                                       nloc * packed_bytes(1, spec.m), soff, xoff, nloc))
                off += nloc * packed_bytes(1, spec.m)
                soff += 4 * nloc
                xoff += B * spec.m
        self.weight_bytes = off
        self.W = torch.empty(max(off, 16), dtype=torch.uint8, device=self.device)
        self.S = torch.empty(max(soff, 4), dtype=torch.float32, device=self.device)
        self.X = torch.empty(max(xoff, 1), dtype=torch.complex64, device=self.device)
        # gathered outputs: [world][B][rows_per_rank] per projection (rank-major, ww.h)
        self.Y = [torch.zeros(p.shard.n_padded * B, dtype=torch.complex64, device=self.device)
                  for p in self.projs]
        self._fill()

    # ------------------------------------------------------------------ inputs
    def _fill(self):
        xs_host = np.empty(self.X.numel(), dtype=np.complex64)
        for pr in self.projs:
            n, m = pr.spec.n, pr.spec.m
            if pr.ylocal:
                planes = torch.empty((4, pr.ylocal, m), dtype=torch.int8, device=self.device)
                for q in range(4):
                    wi.codes_device(pr.seed, q, pr.ylocal, m, planes[q], pr.spec.dist,
                                    row0=pr.shard.row_begin)
                pack_ternary_device(planes, out=self.W[pr.off:pr.off + pr.nbytes])
                sc = wi.scales(pr.seed, n, pr.spec.per_row, pr.spec.scale_lo, pr.spec.scale_hi)
                self.S[pr.soff:pr.soff + 4 * pr.ylocal] = torch.from_numpy(
                    np.ascontiguousarray(sc[pr.shard.row_begin:pr.shard.row_end]).reshape(-1))
            xs_host[pr.xoff:pr.xoff + self.B * m] = wi.activations(pr.seed, m, self.B).reshape(-1)
        self.X.copy_(torch.from_numpy(xs_host))
        torch.cuda.synchronize(self.device)

    def x_of(self, pr: Proj):
        return self.X[pr.xoff:pr.xoff + self.B * pr.spec.m].view(self.B, pr.spec.m)

    def y_local_view(self, pr: Proj):
        """This rank's [B][rows_per_rank] slot of the gathered output (first ylocal rows used)."""
        rpr = pr.shard.rows_per_rank
        base = self.rank * self.B * rpr
        return self.Y[self.projs.index(pr)][base:base + self.B * rpr].view(self.B, rpr)

    def gathered(self, pr: Proj, b: int = 0):
        """Full output y[b] (n rows) of a projection after the all-gather."""
        return gathered_rows(self.Y[self.projs.index(pr)], self.world, self.B,
                             pr.shard.rows_per_rank, pr.spec.n, b)

    # ------------------------------------------------------------------ the step
    def launch(self, i: int, stream=None):
        """Projection i on this rank: WL-GEMV of the local rows into the gathered slot."""
        pr = self.projs[i]
        if not pr.ylocal:
            return 0
        L = Layer(pr.ylocal, pr.spec.m, LAYOUT_COL4, SCALES_PER_ROW, self.conv, self.flags)
        wl_gemv_batched(L, self.W[pr.off:pr.off + pr.nbytes], self.S[pr.soff:pr.soff + 4 * pr.ylocal],
                        self.x_of(pr), self.y_local_view(pr), stream=stream)
        return 1

    def exchange(self, i: int):
        """All-gather of projection i's y shards (NCCL over NVLink); no-op on one rank."""
        if self.world == 1:
            return 0
        exchange_shards(self.Y[i], self.rank, self.world, self.group)
        return 1

    def step(self, stream=None, exchange: bool = True):
        """One token through the whole stack; returns the number of WL-GEMV launches.
        exchange=False skips the all-gathers (tests emulating ranks on one GPU)."""
        k = 0
        for i in range(len(self.projs)):
            k += self.launch(i, stream)
            if exchange:
                self.exchange(i)
        return k

    # ------------------------------------------------------------------ accounting
    def algorithmic_bytes(self) -> int:
        """Bytes the method must move on this rank per step: packed rows + x + y + scales."""
        t = 0
        for pr in self.projs:
            if pr.ylocal:
                t += pr.nbytes + 8 * pr.spec.m * self.B + 8 * pr.ylocal * self.B + 16 * pr.ylocal
        return t

    def packed_act_bytes(self) -> int:
        """North-star roofline bytes: packed weights + activation (x) bytes on this rank."""
        return sum(pr.nbytes + 8 * pr.spec.m * self.B for pr in self.projs if pr.ylocal)

    def adds(self) -> int:
        """Algorithmic fp32 add/sub count on this rank (8 per complex column per row, App. D)."""
        return sum(8 * pr.ylocal * pr.spec.m * self.B for pr in self.projs)
