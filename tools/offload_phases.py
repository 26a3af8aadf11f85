"""Host-phase timing of the offload engine's layer step (variance diagnosis):
per repeat, summed host seconds in routing poll / copy issue / descriptor
updates / forward launch, and the largest single stall with its phase."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_17073_b200 import _lib, offload  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402

L, T, R = 8, 16, int(sys.argv[1]) if len(sys.argv) > 1 else 6
gates, host = [], []
for l in range(L):
    sl = SynthLayer(4096, 14336, 8, top_k=2, rank=32, seed=100 + l, max_tokens=8)
    gates.append(sl.gate)
    host.append(offload.host_experts_from_synth(sl))
    del sl
    torch.cuda.empty_cache()
eng = offload.OffloadEngine(gates, host, 4096, 14336, top_k=2, top_n=1, n_slots=2, max_tokens=8)
ph = {}


def tick(name, t0):
    t1 = time.perf_counter()
    d = t1 - t0
    s, mx, where = ph.get(name, (0.0, 0.0, None))
    ph[name] = (s + d, max(mx, d), where)
    return t1


def layer_step(layer, x):
    t = time.perf_counter()
    idx = eng.route(layer, x).reshape(-1)
    t = tick("route_launch", t)
    hostb = eng._idx_host[:idx.numel()]
    hostb.copy_(idx, non_blocking=True)
    eng._idx_ev.record(torch.cuda.current_stream())
    while not eng._idx_ev.query():
        pass
    t = tick("route_poll", t)
    need = sorted(set(hostb.tolist()))
    keys = {(layer, e) for e in need}
    dl = eng.layers[layer]
    slots = {e: eng._fetch((layer, e), keys) for e in need}
    t = tick("copy_issue", t)
    for e in need:
        d = eng._desc(layer, e, slots[e])
        _lib.check(_lib.lib().lrc_layer_set_expert_async(dl._handle, e, ctypes.byref(d), _lib.stream_ptr()))
        dl._experts[e] = d
        torch.cuda.current_stream().wait_event(eng.slot_ready[slots[e]])
    t = tick("desc", t)
    y, _, _ = dl.forward(x, eng.k, eng.n)
    done = torch.cuda.Event()
    done.record(torch.cuda.current_stream())
    for e in need:
        eng.slot_used[eng.lru[(layer, e)]] = done
    t = tick("forward_launch", t)
    return y


if os.environ.get("GC_FREEZE"):
    import gc

    gc.collect()
    gc.freeze()  # the pool / engine objects leave the collector's generations
gen = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((1, 4096), device="cuda", generator=gen).to(torch.bfloat16)
for r in range(R + 1):
    ph.clear()
    t1 = time.perf_counter()
    for _ in range(T):
        for l in range(L):
            y = layer_step(l, x)
            y = y * torch.rsqrt(y.pow(2).mean(dim=-1, keepdim=True) + 1e-6)
            x = y.to(torch.bfloat16)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t1
    if r == 0:
        continue
    print(f"run {r}: {T / wall:6.2f} tok/s wall {wall * 1e3:7.1f} ms | " +
          "  ".join(f"{k} {v[0] * 1e3:6.1f} (max {v[1] * 1e3:5.1f})" for k, v in ph.items()), flush=True)
