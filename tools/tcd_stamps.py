"""Per-CTA %globaltimer stamps of one tensor-core decode layer step (LRC_TCD_STAMPS=1).
Stamps: 8 gate in smem, 9 logits reduced, 10 selection done, 11 before the plan;
0 after the grid-dependency wait, 1 plan done, 2 aux V.x jobs done,
3 aux phase-U finalisation done, 4 grid barrier passed, 5 CTA end,
6 decode warp 0 enters phase D, 7 MMA warp done."""
import os
import sys

os.environ["LRC_TCD_STAMPS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_17073_b200 import _lib  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402

_lib.load()
WM = int(os.environ.get('TCD_WAIT_MODE', '0'))
_lib.check(_lib.lib().lrc_debug_stamps(4, None, WM))
print('wait mode', WM)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
sl = SynthLayer(4096, 14336, 8, top_k=2, bits=2, rank=32, seed=5, max_tokens=64)
x = torch.randn((B, 4096), device="cuda").to(torch.bfloat16)
for _ in range(3):
    sl.layer.forward(x, 2, 1)
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * (148 * 16))()
_lib.check(_lib.lib().lrc_debug_stamps(2, buf, 148 * 16))
sl.layer.forward(x, 2, 1)
torch.cuda.synchronize()
_lib.check(_lib.lib().lrc_debug_stamps(2, buf, 148 * 16))
st = np.array(buf[:], dtype=np.float64).reshape(148, 16)
t0 = st[:, 0][st[:, 0] > 0].min()
t0c = st[0, 0]
rel = np.where(st > 0, (st - t0) / 1e3, np.nan)
names = ["wait", "plan", "vx", "U fin", "gbar", "end", "dec->D", "mma end", "gate in", "logits", "select",
         "pre-plan"]
uf = rel[:, 3]
order = np.argsort(-np.nan_to_num(uf))
print("slowest U fin CTAs: cta  plan  vx  epiUdone  Ufin  gbar")
for c in order[:12]:
    print(f"  {c:4d} {rel[c, 1]:7.2f} {rel[c, 2]:7.2f} {rel[c, 12]:7.2f} {rel[c, 3]:7.2f} {rel[c, 4]:7.2f}")
eu = rel[:, 12]
print(f"epi U done  min {np.nanmin(eu):.2f} med {np.nanmedian(eu):.2f} max {np.nanmax(eu):.2f}")
print(f"U fin - epi U done: med {np.nanmedian(uf - eu):.2f} max {np.nanmax(uf - eu):.2f}")
for i, n in ((13, "x images done"), (14, "build_plan done"), (15, "build_stages done")):
    col = rel[:, i]
    print(f"{i} {n:18s} min {np.nanmin(col):8.2f}  med {np.nanmedian(col):8.2f}  max {np.nanmax(col):8.2f} us")
for i, n in enumerate(names):
    col = rel[:, i]
    print(f"{i} {n:8s} min {np.nanmin(col):8.2f}  med {np.nanmedian(col):8.2f}  max {np.nanmax(col):8.2f} us")

ws = (ctypes.c_uint64 * 192)()
_lib.check(_lib.lib().lrc_debug_stamps(5, ws, 192))
sl.layer.forward(x, 2, 1)
torch.cuda.synchronize()
_lib.check(_lib.lib().lrc_debug_stamps(5, ws, 192))
w = np.array(ws[:], dtype=np.float64).reshape(24, 8)
print("CTA 0 wait cycles: decode warps: full aempty | total;  epilogue warps: dfull tempty | total")
for i in range(8):
    print(f"  dec w{i}: {w[i][0]:9.0f} {w[i][1]:9.0f} | {w[i][7]:9.0f}")
for i in range(8, 12):
    print(f"  epi w{i}: {w[i][2]:9.0f} {w[i][3]:9.0f} | {w[i][7]:9.0f}")
print(f"  mma w12: afull {w[12][4]:9.0f} dempty {w[12][5]:9.0f} images {w[12][6]:9.0f} | issue {w[12][2]:9.0f} +commits {w[12][3]:9.0f} | total {w[12][7]:9.0f}")
tr = (ctypes.c_uint64 * 2048)()
_lib.check(_lib.lib().lrc_debug_stamps(3, tr, 2048))
sl.layer.forward(x, 2, 1)
torch.cuda.synchronize()
_lib.check(_lib.lib().lrc_debug_stamps(3, tr, 2048))
t = np.array(tr[:], dtype=np.float64).reshape(8, 256)
b = t[0][0]
def f(v):
    return f"{v - b:8.0f}" if v > 0 else "       -"
print("CTA 0, clock64 cycles from producer stage-0 issue")
print("stage: codes issued | B issued | dec w0 aempty seen | dec w0 done | MMA issued | epi dfull seen | epi D loaded | epi done")
for i in range(40):
    print(f"  {i:3d}: {f(t[0][i])} {f(t[1][i])} {f(t[7][i])} {f(t[3][i])} {f(t[2][i])} {f(t[6][i])} {f(t[4][i])} {f(t[5][i])}")
