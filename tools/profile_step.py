"""Run a few C2 decode steps (B tokens) for ncu / launch-list capture.

    python tools/profile_step.py [--batch 1] [--steps 6]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_17073_b200 import _lib  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--layers", type=int, default=2)
a = ap.parse_args()
_lib.load()
layers = [SynthLayer(4096, 14336, 8, top_k=2, rank=32, seed=l, max_tokens=64) for l in range(a.layers)]
x = torch.randn((a.batch, 4096), device="cuda").to(torch.bfloat16)
for i in range(a.steps):
    layers[i % a.layers].layer.forward(x, 2, 1)
torch.cuda.synchronize()
print("ok")
