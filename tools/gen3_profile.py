import sys, torch
sys.path.insert(0, '.')
from paper_2512_17073_b200 import _lib
from paper_2512_17073_b200.synth import SynthLayer
_lib.load()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
sl = SynthLayer(4096, 14336, 8, top_k=2, bits=3, rank=32, seed=5, max_tokens=64, tiles=False)
tcd = len(sys.argv) > 2 and sys.argv[2] == "tcd"
sl.layer.set_tcd_max(-1 if tcd else 0)
x = torch.randn((B, 4096), device="cuda").to(torch.bfloat16)
for _ in range(3):
    sl.layer.forward(x, 2, 1, generic=not tcd)
torch.cuda.synchronize()
