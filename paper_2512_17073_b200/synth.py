"""Synthetic, directly-constructed quantized MoE layers generated on the device.

SURVEY 7.2 step 0 / 8(d): at Mixtral shape the reference's own ``compress``
costs minutes per projection, so benchmark and large-shape parity inputs are
built DIRECTLY as quantized artifacts: uniformly random packed codes (random
bytes are valid LSB-first 2/3-bit streams), fp16 scale/zero drawn in the
ranges an INT2 min-max fit of unit-Gaussian weights produces, INT3 low-rank
factors with the magnitudes of a rank-r SVD of that residual, and a gate
with unit-norm columns x router_skew (ref/moe.py:297-298).

``oracle.bridge.synth_store(layer, expert_ids)`` (test infrastructure)
downloads the same bytes into an oracle ``Store`` for the CPU parity check.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import LRCMoELayer, _Keep, build_down_tiles, build_lr_tiles, build_tiles

MIXTRAL = dict(hidden=4096, ffn=14336, num_experts=8, top_k=2)
DEEPSEEK = dict(hidden=2048, ffn=11008, num_experts=64, top_k=8)


def _qmat(keep, gen, rows, cols, bits, gs, scale_range, zero_over_scale):
    """Random quantized matrix in reference storage form, generated on the device."""
    torch = _lib.device_required()
    nbytes = (rows * cols * bits + 7) // 8
    packed = keep.add(torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda",
                                    generator=gen))
    gpr = -(-cols // gs)
    lo, hi = scale_range
    s = torch.rand((rows, gpr), device="cuda", generator=gen) * (hi - lo) + lo
    z = -zero_over_scale * s * (1.0 + 0.1 * torch.randn((rows, gpr), device="cuda", generator=gen))
    sh = keep.add(s.half().view(torch.uint16).contiguous())
    zh = keep.add(z.half().view(torch.uint16).contiguous())
    m = _lib.LrcQmat()
    m.packed, m.scales, m.zeros, m.dense = packed.data_ptr(), sh.data_ptr(), zh.data_ptr(), None
    m.rows, m.cols, m.bits, m.group_size = rows, cols, bits, gs
    return m, (packed, sh, zh)


class SynthLayer:
    """A directly-constructed quantized MoE layer resident in HBM."""

    def __init__(self, hidden, ffn, num_experts, top_k=2, num_shared=0, bits=2, rank=32,
                 factor_bits=3, seed=0, router_skew=1.4, max_tokens=64, tiles=True,
                 comp_experts=None, zero_weights=False):
        torch = _lib.device_required()
        self.hidden, self.ffn, self.E, self.S = hidden, ffn, num_experts, num_shared
        self.bits, self.rank, self.top_k = bits, rank, top_k
        self.keep = _Keep()
        gen = torch.Generator(device="cuda")
        gen.manual_seed(seed)
        rng = np.random.default_rng(seed)
        g = rng.standard_normal((hidden, num_experts))
        self.gate = g / np.linalg.norm(g, axis=0, keepdims=True) * router_skew
        qmax = (1 << bits) - 1
        wscale = (4.2 / qmax, 5.4 / qmax)  # (max-min)/qmax of a 64-sample N(0,1) group
        self.raw = []  # per expert: {name: (packed, scales, zeros, rows, cols, bits, gs)}
        experts = []
        comp_experts = range(num_experts + num_shared) if comp_experts is None else comp_experts
        for e in range(num_experts + num_shared):
            ex = _lib.LrcExpert()
            raw = {}
            for name, (r, c) in (("w1", (ffn, hidden)), ("w3", (ffn, hidden)), ("w2", (hidden, ffn))):
                m, t = _qmat(self.keep, gen, r, c, bits, 64, wscale, qmax / 2.0)
                if zero_weights:  # scale = zero = 0: only the low-rank path contributes
                    t[1].zero_()
                    t[2].zero_()
                setattr(ex, name, m)
                raw[name] = (*t, r, c, bits, 64)
            if rank > 0 and e in comp_experts:
                fq = (1 << factor_bits) - 1
                for un, vn, (r, c) in (("u1", "v1", (ffn, hidden)), ("u3", "v3", (ffn, hidden)),
                                       ("u2", "v2", (hidden, ffn))):
                    ugs, vgs = min(64, rank), 64
                    um, ut = _qmat(self.keep, gen, r, rank, factor_bits, ugs,
                                   (0.10 / fq, 0.14 / fq), fq / 2.0)
                    vm, vt = _qmat(self.keep, gen, rank, c, factor_bits, vgs,
                                   (0.20 / fq, 0.28 / fq), fq / 2.0)
                    setattr(ex, un, um)
                    setattr(ex, vn, vm)
                    raw[un] = (*ut, r, rank, factor_bits, ugs)
                    raw[vn] = (*vt, rank, c, factor_bits, vgs)
                ex.rank = rank
            if tiles and bits == 2:
                ex.up_tiles = build_tiles([ex.w1, ex.w3], self.keep).data_ptr()
                ex.down_tiles = build_down_tiles(ex.w2, self.keep).data_ptr()
                if ex.rank:
                    build_lr_tiles(ex, hidden, ffn, self.keep)
            experts.append(ex)
            self.raw.append(raw)
        self.layer = LRCMoELayer(self.gate, experts, hidden, ffn, num_experts, num_shared,
                                 self.keep, max_tokens=max_tokens, top_k=top_k)

    # ------------------------------------------------------------- bytes --
    def expert_bytes(self) -> int:
        from .quant import packed_size_bytes

        return 2 * packed_size_bytes(self.ffn, self.hidden, self.bits, True) + \
            packed_size_bytes(self.hidden, self.ffn, self.bits, True)

    def comp_bytes(self) -> int:
        from .lowrank import compensator_size_bytes

        if self.rank == 0:
            return 0
        r = self.rank
        meta = 0
        for rows, cols in ((self.ffn, self.hidden), (self.ffn, self.hidden), (self.hidden, self.ffn)):
            meta += 4 * (rows * -(-r // min(64, r)) + r * -(-cols // 64))
        return 2 * compensator_size_bytes(self.ffn, self.hidden, r) + \
            compensator_size_bytes(self.hidden, self.ffn, r) + meta
