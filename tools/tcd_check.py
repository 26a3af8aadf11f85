"""First-light check of the tensor-core decode engine on B200: tcd vs the tiled
(mma.sync) path and the generic path on the same synthetic layers, then a
graph-replayed timing at B=1 (8 rotating Mixtral layers, like bench.py).

    python tools/tcd_check.py [--quick]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_17073_b200 import _lib  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402


def rel(a, b):
    a, b = a.double(), b.double()
    return float(((a - b).norm(dim=1) / b.norm(dim=1).clamp_min(1e-30)).max())


def compare(name, sl, B, k, n, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((B, sl.hidden), device="cuda", generator=g).to(torch.bfloat16)
    L = sl.layer
    L.set_tcd_max(8)
    y1, i1, w1 = L.forward(x, k, n)
    torch.cuda.synchronize()
    y1, i1, w1 = y1.clone(), i1.clone(), w1.clone()
    L.set_tcd_max(0)
    y2, i2, w2 = L.forward(x, k, n, generic=(sl.bits != 2))
    torch.cuda.synchronize()
    L.set_tcd_max(8)
    same_idx = bool(torch.equal(i1, i2))
    print(f"{name:34s} B={B}: rel L2 vs {'generic' if sl.bits != 2 else 'tiled'} {rel(y1, y2):.3e}  "
          f"idx equal {same_idx}  w maxdiff {float((w1 - w2).abs().max()):.2e}  |y| {float(y2.abs().max()):.3g}",
          flush=True)
    return rel(y1, y2), same_idx


def timing(B=1, layers=8, steps=400, tcd=True, bits=2):
    sls = [SynthLayer(4096, 14336, 8, top_k=2, bits=bits, rank=32, seed=100 * l, max_tokens=64, tiles=(bits == 2))
           for l in range(layers)]
    xs = [torch.randn((B, 4096), device="cuda").to(torch.bfloat16) for _ in range(2 * layers)]
    ys = [torch.empty((B, 4096), dtype=torch.float32, device="cuda") for _ in range(layers)]
    idx = [torch.empty((B, 2), dtype=torch.int32, device="cuda") for _ in range(layers)]
    wts = [torch.empty((B, 2), dtype=torch.float32, device="cuda") for _ in range(layers)]
    out = {}
    for mode in (("tcd", "tiled") if tcd else ("tiled",)):
        for sl in sls:
            sl.layer.set_tcd_max(8 if mode == "tcd" else 0)

        def step(i):
            l = i % layers
            sls[l].layer.forward(xs[i % (2 * layers)], 2, 1, y=ys[l], topk_idx=idx[l], topk_w=wts[l],
                                 generic=(bits != 2 and mode != "tcd"))

        for i in range(2 * layers):
            step(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for i in range(3):
                step(i)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            for i in range(steps):
                step(i)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out[mode] = ms * 1e3 / steps
        name = mode if bits == 2 or mode == "tcd" else "generic"
        print(f"timing {name}: {bits}-bit B={B} {out[mode]:.2f} us/step  {steps * B / (ms / 1e3):.0f} tok/s", flush=True)
    return out


def main():
    _lib.load()
    torch.manual_seed(0)
    quick = "--quick" in sys.argv
    # tiny (C1 dims) and Mixtral (C2) layers, 2-bit
    sl = SynthLayer(512, 1024, 8, top_k=2, bits=2, rank=16, seed=1, max_tokens=64)
    print("tcd eligible (C1):", sl.layer.tcd_eligible, flush=True)
    for B in (1, 4, 8):
        compare("C1 2-bit r16 top-2 n=1", sl, B, 2, 1, seed=B)
    del sl
    sl = SynthLayer(4096, 14336, 8, top_k=2, bits=2, rank=32, seed=2, max_tokens=64)
    print("tcd eligible (C2):", sl.layer.tcd_eligible, flush=True)
    for B in ((1, 8) if quick else (1, 2, 3, 4, 8)):
        compare("C2 2-bit r32 top-2 n=1", sl, B, 2, 1, seed=10 + B)
    compare("C2 2-bit r32 top-2 n=0", sl, 1, 2, 0, seed=99)
    del sl
    if not quick:
        sl = SynthLayer(4096, 14336, 8, top_k=2, bits=3, rank=32, seed=3, max_tokens=64, tiles=False)
        print("tcd eligible (C2 3-bit):", sl.layer.tcd_eligible, flush=True)
        for B in (1, 8):
            compare("C2 3-bit r32 top-2 n=1", sl, B, 2, 1, seed=20 + B)
        del sl
    torch.cuda.empty_cache()
    timing(B=1)
    if "--timing3" in sys.argv:
        timing(B=8, steps=200)
        timing(B=1, bits=3, steps=200)
        timing(B=8, bits=3, steps=100)
        timing(B=64, bits=3, steps=50, tcd=False)
    elif not quick:
        timing(B=8, steps=200)


if __name__ == "__main__":
    main()
