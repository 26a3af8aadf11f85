"""Print per-phase device times of C2 decode steps (profiling events, no host gaps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_17073_b200 import _lib  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
_lib.load()
layers = [SynthLayer(4096, 14336, 8, top_k=2, rank=32, seed=l, max_tokens=64) for l in range(4)]
x = torch.randn((B, 4096), device="cuda").to(torch.bfloat16)
for sl in layers:
    sl.layer.set_profiling(True)
ph = []
for i in range(24):
    torch.cuda._sleep(1_000_000)
    layers[i % 4].layer.forward(x, 2, 1)
    ph.append(layers[i % 4].layer.phase_ms())
ph = np.array(ph[4:]) * 1e3
print(f"B={B} debug={os.environ.get('LRC_TILED_DEBUG', '0')} route/lr_down/up/down us:",
      np.round(ph.mean(0), 2))
