"""Cold vs warm instruction/data caches: time the standalone router kernel
(lrc_route, same kernel as the layer's prologue) right after a full layer step
(cold) and immediately repeated (warm)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_17073_b200 import _lib  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402

lib = _lib.load()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
layers = [SynthLayer(4096, 14336, 8, top_k=2, rank=32, seed=l, max_tokens=64) for l in range(4)]
x = torch.randn((B, 4096), device="cuda").to(torch.bfloat16)
gate = torch.randn((8, 4096), device="cuda", dtype=torch.float64)
probs = torch.empty((B, 8), device="cuda", dtype=torch.float64)
idx = torch.empty((B, 2), device="cuda", dtype=torch.int32)
w = torch.empty((B, 2), device="cuda", dtype=torch.float32)
st = torch.cuda.current_stream().cuda_stream


def route():
    _lib.check(lib.lrc_route(ctypes.c_void_p(gate.data_ptr()), ctypes.c_void_p(x.data_ptr()), 2, B, 4096, 8, 2, 1, 0,
                             ctypes.c_void_p(probs.data_ptr()), ctypes.c_void_p(idx.data_ptr()),
                             ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(st)))


ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
cold, warm = [], []
for i in range(30):
    layers[i % 4].layer.forward(x, 2, 1)
    ev[0].record()
    route()
    ev[1].record()
    route()
    ev[2].record()
    torch.cuda.synchronize()
    if i >= 5:
        cold.append(ev[0].elapsed_time(ev[1]) * 1e3)
        warm.append(ev[1].elapsed_time(ev[2]) * 1e3)
print(f"B={B} lrc_route after a layer step: cold {np.median(cold):.2f} us, warm (repeat) {np.median(warm):.2f} us")
