"""Bridge device-resident synthetic layers to oracle Stores (TEST INFRASTRUCTURE ONLY).

Downloads the exact bytes a ``paper_2512_17073_b200.synth.SynthLayer`` holds in
HBM and rebuilds them as oracle records: codes unpacked from the LSB-first
stream with the oracle's own ``unpack_codes``, fp16 metadata widened to f64.
"""

from __future__ import annotations

import numpy as np

from . import lrc


def _qm(t):
    packed, sh, zh, rows, cols, bits, gs = t
    codes = lrc.unpack_codes(packed.cpu().numpy().tobytes(), rows * cols, bits)
    s = sh.cpu().numpy().view(np.float16).astype(np.float64)
    z = zh.cpu().numpy().view(np.float16).astype(np.float64)
    return lrc.QM(rows, cols, bits, gs, codes.reshape(rows, cols), s, z)


def synth_store(layer, expert_ids, layer_id=0) -> lrc.Store:
    st = lrc.Store()
    for e in expert_ids:
        raw = layer.raw[e]
        for p, (un, vn) in (("w1", ("u1", "v1")), ("w3", ("u3", "v3")), ("w2", ("u2", "v2"))):
            comp = lrc.Comp(layer.rank, _qm(raw[un]), _qm(raw[vn]), p) if un in raw else None
            st.records[(layer_id, e, p)] = lrc.Rec(_qm(raw[p]), comp)
    return st


class LazyStore(lrc.Store):
    """Store that materialises an expert's records on first access (host-built
    synthetic artifacts for the CPU reference arm; deterministic per expert)."""

    def __init__(self, make_expert):
        super().__init__()
        self._make = make_expert

    def get(self, layer, expert, proj):
        key = (layer, expert, proj)
        if key not in self.records:
            for p, rec in self._make(layer, expert).items():
                self.records[(layer, expert, p)] = rec
        return self.records[key]
