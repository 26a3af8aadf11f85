"""Small-shape run of every engine for compute-sanitizer:

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_run.py

C1-sized layers (d=512, ffn=1024, 8 experts top-2, rank 16): cluster router +
tiled kernels (B=1, 4), the tensor-core decode engine (INT2 forced, INT3
default; B=1, 3), the generic path, the prefill engine (2- and 3-bit), the
forward_pairs path and the EP dispatch / combine kernels.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_17073_b200 import _lib  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402


def main():
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(0)
    for bits in (2, 3):
        sl = SynthLayer(512, 1024, 8, top_k=2, bits=bits, rank=16, seed=bits, max_tokens=64, tiles=(bits == 2))
        L = sl.layer
        for B in (1, 4):
            x = torch.randn((B, 512), device="cuda", generator=g).to(torch.bfloat16)
            L.forward(x, 2, 1)                      # tiled (2-bit) / tcd (3-bit)
            L.forward(x, 2, 1, generic=True)        # generic
            L.set_tcd_max(8)
            L.forward(x, 2, 1)                      # tcd
            L.set_tcd_max(-1)
        x = torch.randn((16, 512), device="cuda", generator=g).to(torch.bfloat16)
        L.set_prefill_min(1)
        L.forward(x, 2, 1)                          # prefill engine
        L.set_prefill_min(1 << 20)
        idx = torch.tensor([0, 3, 5, 7], dtype=torch.int32, device="cuda")
        L.forward_pairs(x[:4], idx, torch.ones(4, device="cuda"), torch.tensor([1, 0, 1, 0], dtype=torch.uint8,
                                                                              device="cuda"))
        torch.cuda.synchronize()
        print(f"{bits}-bit engines ok", flush=True)
    # EP dispatch / combine kernels (world 2, capacity 8)
    B, k, W, C, d = 4, 2, 2, 8, 512
    ti = torch.tensor([[0, 5], [3, 1], [7, 6], [2, 4]], dtype=torch.int32, device="cuda")
    tw = torch.rand((B, k), device="cuda")
    x = torch.randn((B, d), device="cuda", generator=g).to(torch.bfloat16)
    xs = torch.empty((W * C, d), dtype=torch.bfloat16, device="cuda")
    meta = torch.empty((W * C, 3), dtype=torch.int32, device="cuda")
    so = torch.empty((B * k,), dtype=torch.int32, device="cuda")
    _lib.check(lib.lrc_ep_dispatch(_lib.ptr(ti), _lib.ptr(tw), _lib.ptr(x), B, k, 1, 8, W, C, d, _lib.ptr(xs),
                                   _lib.ptr(meta), _lib.ptr(so), _lib.stream_ptr()))
    back = torch.randn((W * C, d), device="cuda", generator=g)
    y = torch.empty((B, d), device="cuda")
    _lib.check(lib.lrc_ep_combine(_lib.ptr(back), _lib.ptr(so), B, k, d, _lib.ptr(y), _lib.stream_ptr()))
    torch.cuda.synchronize()
    print("ep kernels ok", flush=True)


if __name__ == "__main__":
    main()
