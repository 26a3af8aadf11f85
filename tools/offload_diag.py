"""Offload variance diagnosis: per repeat, wall time vs the copy stream's busy
time (events around every expert fetch) -> bytes / copy-busy-second (link rate)
and the host-side gap.  python tools/offload_diag.py [--layers 8] [--repeats 6]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_17073_b200 import offload  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--tokens", type=int, default=16)
ap.add_argument("--repeats", type=int, default=6)
ap.add_argument("--slots", type=int, default=2)
args = ap.parse_args()
gates, host = [], []
for l in range(args.layers):
    sl = SynthLayer(4096, 14336, 8, top_k=2, rank=32, seed=100 + l, max_tokens=8)
    gates.append(sl.gate)
    host.append(offload.host_experts_from_synth(sl))
    del sl
    torch.cuda.empty_cache()
eng = offload.OffloadEngine(gates, host, 4096, 14336, top_k=2, top_n=1, n_slots=args.slots, max_tokens=8)
# wrap _fetch to time each miss's copies on the copy stream
orig = eng._fetch
marks = []


def timed_fetch(key, busy):
    hit = key in eng.lru
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(eng.copy_stream)
    slot = orig(key, busy)
    if not hit:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(eng.copy_stream)
        marks.append((e0, e1, eng.host[key[0]][key[1]].nbytes, time.perf_counter()))
    return slot


eng._fetch = timed_fetch
# per-layer host timing: routing sync (.cpu()), copy issue, descriptor updates, forward launch
orig_route = eng.route
layer_t = []


def timed_route(layer, x):
    t0 = time.perf_counter()
    idx = orig_route(layer, x)
    t1 = time.perf_counter()
    layer_t.append((layer, t1 - t0))
    return idx


eng.route = timed_route
gen = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((1, 4096), device="cuda", generator=gen).to(torch.bfloat16)
for _ in range(3):
    x = eng.forward(x, normalize=True)
torch.cuda.synchronize()
for r in range(args.repeats):
    marks.clear()
    layer_t.clear()
    t1 = time.perf_counter()
    for _ in range(args.tokens):
        x = eng.forward(x, normalize=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t1
    copy_ms = [a.elapsed_time(b) for a, b, _, _ in marks]
    nbytes = sum(m[2] for m in marks)
    busy = sum(copy_ms) / 1e3
    print(f"run {r}: {args.tokens / wall:6.2f} tok/s  wall {wall * 1e3:7.1f} ms  copies {len(marks)}  "
          f"copy-busy {busy * 1e3:7.1f} ms  link {nbytes / busy / 1e9:6.2f} GB/s  "
          f"per-copy ms min/med/max {min(copy_ms):.2f}/{sorted(copy_ms)[len(copy_ms) // 2]:.2f}/{max(copy_ms):.2f}",
          flush=True)
    rs = sorted(t for _, t in layer_t)
    print(f"    route+sync per layer ms: med {rs[len(rs) // 2] * 1e3:.2f}  max {rs[-1] * 1e3:.1f}  "
          f"sum {sum(rs) * 1e3:.1f}  top5 {[round(t * 1e3, 1) for t in rs[-5:]]}", flush=True)
