"""Offload engine (config C3): experts fetched on demand from pinned host memory
into an LRU set of GPU slots give the same layer outputs as the resident layer,
with hits, misses and evictions all exercised."""
import pytest
import torch

from paper_2512_17073_b200 import offload
from paper_2512_17073_b200.synth import SynthLayer


@pytest.mark.gpu
def test_offload_matches_resident_layers():
    hidden, ffn, E = 512, 1024, 8
    layers = [SynthLayer(hidden, ffn, E, top_k=2, rank=16, seed=20 + l, max_tokens=8) for l in range(2)]
    host = [offload.host_experts_from_synth(sl) for sl in layers]
    # 8 slots for 2 layers x 8 experts: a step needs up to B*k <= 8, so evictions occur
    eng = offload.OffloadEngine([sl.gate for sl in layers], host, hidden, ffn, top_k=2, top_n=1,
                                n_slots=8, max_tokens=8)
    gen = torch.Generator(device="cuda").manual_seed(0)
    worst = 0.0
    for step in range(6):
        B = 1 + step % 4
        x = torch.randn((B, hidden), device="cuda", generator=gen).to(torch.bfloat16)
        y = eng.forward(x)
        ref = x
        for sl in layers:
            ref = sl.layer.forward(ref, 2, 1)[0].to(torch.bfloat16)
        torch.cuda.synchronize()
        err = float((y.float() - ref.float()).norm() / ref.float().norm())
        worst = max(worst, err)
    assert worst < 1e-2, worst  # bf16 chaining of two layers; single-layer check below
    assert eng.stats["misses"] > 0 and eng.stats["hits"] > 0


@pytest.mark.gpu
def test_offload_single_layer_exact():
    hidden, ffn, E = 512, 1024, 8
    sl = SynthLayer(hidden, ffn, E, top_k=2, rank=16, seed=31, max_tokens=8)
    eng = offload.OffloadEngine([sl.gate], [offload.host_experts_from_synth(sl)], hidden, ffn,
                                top_k=2, top_n=1, n_slots=2, max_tokens=8)
    gen = torch.Generator(device="cuda").manual_seed(1)
    for step in range(8):
        x = torch.randn((1, hidden), device="cuda", generator=gen).to(torch.bfloat16)
        y = eng.forward_layer(0, x)
        ref = sl.layer.forward(x, 2, 1)[0]
        torch.cuda.synchronize()
        err = float((y - ref).norm() / ref.norm())
        assert err < 1e-5, (step, err)
    # 2 slots, top-2 routing over 8 experts: evictions must have happened
    assert eng.stats["misses"] >= 3
    per = sum(b.numel() for b in eng.host[0][0].bufs.values())
    assert eng.stats["bytes"] >= eng.stats["misses"] * per * 0.9


@pytest.mark.gpu
def test_forward_host_graph_replay():
    """lrc_layer_forward_host captures its H2D -> layer -> D2H sequence as a
    CUDA graph per shape; replays with new host buffers must match forward()."""
    sl = SynthLayer(512, 1024, 8, top_k=2, rank=16, seed=41, max_tokens=8)
    for B in (1, 1, 3, 3, 3, 1):
        x = torch.randn((B, 512), device="cuda").to(torch.bfloat16)
        xh = x.cpu().pin_memory()
        yh = torch.empty((B, 512), dtype=torch.float32).pin_memory()
        sl.layer.forward_host(xh, yh, 2, 1)
        torch.cuda.synchronize()
        ref = sl.layer.forward(x, 2, 1)[0].cpu()
        err = float((yh - ref).norm() / ref.norm())
        assert err < 1e-5, (B, err)


@pytest.mark.gpu
def test_gpu_pager_matches_resident_layers():
    """GPU-driven paging: every expert in mapped pinned memory, copied into 2
    slots by the pager kernel inside each layer forward (no host round trip);
    a 2-layer chain matches the resident chain, single layers match exactly."""
    hidden, ffn, E = 512, 1024, 8
    layers = [SynthLayer(hidden, ffn, E, top_k=2, rank=16, seed=50 + l, max_tokens=8) for l in range(2)]
    host = [offload.host_experts_from_synth(sl) for sl in layers]
    eng = offload.GpuPagerEngine([sl.gate for sl in layers], host, hidden, ffn, top_k=2, top_n=1, max_tokens=1)
    gen = torch.Generator(device="cuda").manual_seed(2)
    for step in range(6):
        x = torch.randn((1, hidden), device="cuda", generator=gen).to(torch.bfloat16)
        y0 = eng.forward_layer(0, x)
        ref0 = layers[0].layer.forward(x, 2, 1)[0]
        torch.cuda.synchronize()
        assert float((y0 - ref0).norm() / ref0.norm()) < 1e-5, step
        y = eng.forward(x)
        ref = x
        for sl in layers:
            ref = sl.layer.forward(ref, 2, 1)[0].to(torch.bfloat16)
        torch.cuda.synchronize()
        assert float((y.float() - ref.float()).norm() / ref.float().norm()) < 1e-2, step


@pytest.mark.gpu
def test_gpu_pager_graph_capture():
    """The paged layer chain of one token captured as a CUDA graph replays to the
    same result as the eager chain."""
    hidden, ffn, E = 512, 1024, 8
    layers = [SynthLayer(hidden, ffn, E, top_k=2, rank=16, seed=60 + l, max_tokens=8) for l in range(3)]
    eng = offload.GpuPagerEngine([sl.gate for sl in layers], [offload.host_experts_from_synth(sl) for sl in layers],
                                 hidden, ffn, top_k=2, top_n=1, max_tokens=1)
    x = torch.randn((1, hidden), device="cuda").to(torch.bfloat16)
    eager = eng.forward(x.clone()).float()
    xin = x.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        eng.forward(xin)  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = eng.forward(xin)
    g.replay()
    torch.cuda.synchronize()
    assert float((out.float() - eager).norm() / eager.norm()) < 1e-6


@pytest.mark.gpu
def test_gpu_pager_lru_cache_matches_resident_and_simulator():
    """Budgeted LRU in the GPU pager (lrc_pager_cache, 5 slots shared by 2
    layers x 8 experts): every step matches the resident layers, resident hits
    move nothing, and the device's hit / miss counts equal the reference cost
    model's LRU (simulate.py, cache_policy="lru") on the recorded trace."""
    from paper_2512_17073_b200 import simulate as sim

    hidden, ffn, E, L = 512, 1024, 8, 2
    layers = [SynthLayer(hidden, ffn, E, top_k=2, rank=16, seed=70 + l, max_tokens=8, router_skew=2.5)
              for l in range(L)]
    eng = offload.GpuPagerEngine([sl.gate for sl in layers], [offload.host_experts_from_synth(sl) for sl in layers],
                                 hidden, ffn, top_k=2, top_n=1, max_tokens=1, cache_slots=5)
    gen = torch.Generator(device="cuda").manual_seed(3)
    eng.start_trace()
    for step in range(24):
        x = torch.randn((1, hidden), device="cuda", generator=gen).to(torch.bfloat16)
        y = eng.forward(x)
        ref = x
        for sl in layers:
            ref = sl.layer.forward(ref, 2, 1)[0].to(torch.bfloat16)
        torch.cuda.synchronize()
        assert float((y.float() - ref.float()).norm() / ref.float().norm()) < 1e-2, step
    hits, misses = eng.cache_stats()
    assert hits + misses == 24 * L * 2 and hits > 0
    trace = eng.routing_trace()
    dims = sim.ModelDims(hidden, ffn, L, E, 2)
    plan = sim.TransferPlan(expert_bits=2, top_n=1, rank=16, cache_policy="lru",
                            cache_budget_bytes=5 * sim.expert_weight_bytes(dims, 2))
    rep = sim.simulate(trace, plan, sim.SYSTEM_PRESETS["gpu-only"], dims, include_prefill=False)
    assert abs(rep.cache_hit_rate - hits / (hits + misses)) < 1e-12, (rep.cache_hit_rate, hits, misses)
