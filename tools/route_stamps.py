"""Per-CTA %globaltimer stamps of one decode layer step: router (LRC_ROUTE_STAMPS)
and tiled up/down kernels (LRC_TILED_DEBUG bit 3), relative to router entry.

usage: python tools/route_stamps.py B [extra LRC_TILED_DEBUG bits]
"""
import ctypes
import os
import sys

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
extra = int(sys.argv[2]) if len(sys.argv) > 2 else 0
os.environ.setdefault("LRC_ROUTE_STAMPS", "1")
os.environ["LRC_TILED_DEBUG"] = str(8 | extra)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_17073_b200 import _lib  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402

lib = _lib.load()
layers = [SynthLayer(4096, 14336, 8, top_k=2, rank=32, seed=l, max_tokens=64) for l in range(4)]
x = torch.randn((B, 4096), device="cuda").to(torch.bfloat16)


def grab(which, n):
    buf = np.zeros(n, dtype=np.uint64)
    _lib.check(lib.lrc_debug_stamps(which, buf.ctypes.data_as(ctypes.c_void_p), n))
    return buf.astype(np.int64)


# back-to-back steps over the 4 layers (like the bench); stamps of the last step
for rep in range(3):
    for i in range(16):
        layers[i % 4].layer.forward(x, 2, 1)
    torch.cuda.synchronize()
    r = grab(0, 1024 * 8).reshape(1024, 8)
    t = grab(1, 2 * 256 * 8).reshape(2, 256, 8)

r = r[r[:, 0] > 0]
t0 = r[:, 0].min()


def show(name, v):
    v = v[v > 0]
    if v.size:
        v = (v - t0) / 1e3
        print(f"  {name:26s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us  (n={v.size})")


print(f"B={B}  router CTAs={r.shape[0]}")
nl = r[1:8]  # non-leader logit CTAs of row 0 (x = 1..7)
for k, n in ((3, "nonleader: loads+fma done"), (4, "nonleader: reduce done"), (5, "nonleader: dsmem done")):
    show(n, nl[:, k])
for k, n in enumerate(["entry", "work done", "sel: softmax done", "select done", "plan ticket", "plan done", "logits done", "sel: top-k done"]):
    show("route " + n, r[:8, k])
ax = r[8:]  # aux CTAs (rows > 0): zeroing + speculative V.x
for k, n in ((0, "entry"), (2, "griddep passed"), (3, "x staged"), (4, "x sums"), (1, "work done")):
    show("aux " + n, ax[:, k])
for up, nm in ((1, "up"), (0, "down")):
    for k, n in enumerate(["entry", "griddep passed", "setup done", "prod first issue", "prod last issue",
                           "cons first data", "cons done", "epi done"]):
        show(f"{nm} {n}", t[up, :148, k])

# per-item stamps of CTA 0 (last step): issue / data / MMA done / epilogue done
for i in range(16):
    layers[i % 4].layer.forward(x, 2, 1)
torch.cuda.synchronize()
t = grab(1, 2 * 256 * 8 + 2 * 64 * 6)[2 * 256 * 8:].reshape(2, 64, 6)
for up, nm in ((1, "up"), (0, "down")):
    it = t[up]
    it = it[it[:, 0] > 0]
    base = it[0, 0]
    print(f"{nm} CTA0 items (us rel. to first issue): issue / cons-wait / data / mma-core / posted / epi")
    for k, row in enumerate(it[:16]):
        print("   ", k, np.round((row - base) / 1e3, 2))
