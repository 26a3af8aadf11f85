"""Compare the speculative (B<=8) and exact (B>8) prologue paths on one layer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_17073_b200 import _lib  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402

_lib.load()
sl = SynthLayer(256, 512, 8, top_k=2, rank=16, seed=1, max_tokens=64)
x = torch.randn((9, 256), device="cuda").to(torch.bfloat16)
for top_n in (0, 1):
    y9, i9, w9 = sl.layer.forward(x, 2, top_n)
    y9 = y9.clone()
    for generic in (False, True):
        y1, i1, w1 = sl.layer.forward(x[:1].contiguous(), 2, top_n, generic=generic)
        torch.cuda.synchronize()
        d = (y1[0] - y9[0]).abs().max().item()
        print(f"top_n={top_n} generic={generic} idx1={i1[0].tolist()} idx9={i9[0].tolist()} "
              f"w1={w1[0].tolist()} w9={w9[0].tolist()} maxdiff={d:.4g} |y9|={y9[0].abs().max().item():.4g} "
              f"|y1|={y1[0].abs().max().item():.4g}")
y0 = torch.full((1, 256), 12345.0, device="cuda")
yz, _, _ = sl.layer.forward(x[:1].contiguous(), 0, 0, y=y0)
print("top_k=0 output (should be zeros):", yz.abs().max().item())
