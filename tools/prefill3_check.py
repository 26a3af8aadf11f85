"""Prefill engine with 3-bit codes: parity vs the generic path and timing vs B.

    python tools/prefill3_check.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_17073_b200 import _lib  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402


def rel(a, b):
    a, b = a.double(), b.double()
    return float(((a - b).norm(dim=1) / b.norm(dim=1).clamp_min(1e-30)).max())


def timed(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


def main():
    _lib.load()
    for bits in (3, 2):
        sl = SynthLayer(4096, 14336, 8, top_k=2, bits=bits, rank=32, seed=7, max_tokens=512, tiles=(bits == 2))
        L = sl.layer
        L.set_tcd_max(0)
        print(f"{bits}-bit prefill eligible:", L.prefill_eligible, flush=True)
        for B in (16, 64, 256):
            x = torch.randn((B, 4096), device="cuda").to(torch.bfloat16)
            L.set_prefill_min(1)
            y1, i1, _ = L.forward(x, 2, 1)
            torch.cuda.synchronize()
            y1 = y1.clone()
            tp = timed(lambda: L.forward(x, 2, 1))
            L.set_prefill_min(1 << 30)
            y2, i2, _ = L.forward(x, 2, 1, generic=(bits != 2))
            torch.cuda.synchronize()
            tg = timed(lambda: L.forward(x, 2, 1, generic=(bits != 2)), iters=3)
            print(f"{bits}-bit B={B:4d}: prefill {tp:9.1f} us  {'generic' if bits != 2 else 'tiled'} {tg:9.1f} us  "
                  f"rel L2 {rel(y1, y2):.3e}  idx equal {bool(torch.equal(i1, i2))}", flush=True)
        del sl, L
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
