"""Shared helpers for the GPU parity tests: build one seeded layer on both sides.

The oracle side gets App. H planar words packed by ``oracle.pack_planar``; the CUDA
side gets COL4 words packed by the product's host packer.  Both come from the same
dense int8 planes drawn by ``ww_inputs`` (no value flows from the CUDA path to the
oracle)."""
from __future__ import annotations

import numpy as np

import oracle as orc
import ww_inputs as wi


class LayerCase:
    def __init__(self, n, m, seed=0, dist=wi.LLAMA, per_row=True, lo=0.01, hi=0.1, B=1,
                 planes=None, scales=None, x=None):
        self.n, self.m, self.B = n, m, B
        self.planes = wi.planes(seed, n, m, dist) if planes is None else planes
        self.scales = wi.scales(seed, n, per_row, lo, hi) if scales is None else scales
        self.x = wi.activations(seed, m, B) if x is None else x
        self.per_row = self.scales.ndim == 2
        self._planar = None

    @classmethod
    def from_spec(cls, spec, seed=0, B=1):
        return cls(spec.n, spec.m, seed, spec.dist, spec.per_row, spec.scale_lo, spec.scale_hi, B)

    @property
    def planar(self):
        if self._planar is None:
            self._planar = orc.pack_planar(self.planes)
        return self._planar

    def oracle(self, conv, rows=None):
        return orc.wl_direct(self.planar, self.n, self.m, self.scales, self.x, conv, rows)

    # ---- CUDA side
    def device(self, ww, torch):
        self.packed_d = torch.from_numpy(ww.pack_ternary(self.planes, ww.LAYOUT_COL4).view(np.uint8)).cuda()
        self.scales_d = torch.from_numpy(np.ascontiguousarray(self.scales)).cuda()
        self.x_d = torch.from_numpy(np.ascontiguousarray(self.x)).cuda()
        return self

    def layer(self, ww, conv, flags=0):
        return ww.Layer(self.n, self.m, ww.LAYOUT_COL4,
                        ww.SCALES_PER_ROW if self.per_row else ww.SCALES_PER_TENSOR, conv, flags)

    def gpu(self, ww, torch, conv, flags=0):
        L = self.layer(ww, conv, flags)
        if self.B == 1:
            y = ww.wl_gemv(L, self.packed_d, self.scales_d, self.x_d[0])
            out = y[None, :]
        else:
            out = ww.wl_gemv_batched(L, self.packed_d, self.scales_d, self.x_d)
        torch.cuda.synchronize()
        return out.cpu().numpy()


def assert_parity(y_gpu, y_ref, case, rows=None):
    ok, rel, worst = orc.tolerance_check(y_gpu, y_ref, case.scales, case.x, rows)
    assert ok, f"rel L2 {rel:.3e} (bar 1e-5), worst per-element ratio {worst:.3f} (bar 1)"
    return rel, worst
