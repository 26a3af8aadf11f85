"""tcgen05 prefill path: the grouped dequant-GEMM
with the low-rank term folded in as K augmentation, against the fp64 oracle and
against the decode (mma.sync tiled) path on the same layer.

Tolerances as tests/test_gpu_parity.py: layer output max relative L2 <= 1e-2
against the oracle fed the same bf16 tokens and fp16 metadata (the prefill
path additionally rounds dequantized weights, t vectors and activations to
bf16); the low-rank-only output within 5e-2.
"""
import math

import numpy as np
import pytest

from oracle import bridge, lrc

pytestmark = pytest.mark.gpu

TOL_Y = 1e-2
TOL_LR = 5e-2


@pytest.fixture(scope="module")
def torch():
    import torch as t

    import paper_2512_17073_b200._lib as L

    L.load()
    return t


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _toy():
    from test_gpu_parity import _toy_store

    st = _toy_store()
    layers = lrc.gen_model(7, 64, 128, 2, 8, num_shared=1, tail_dofs=(4.0, math.inf), router_skew=1.4)
    return st, layers


@pytest.mark.parametrize("B", [1, 37, 300])
def test_toy_prefill_vs_oracle(torch, B):
    """Reference-compressed toy layers (hidden 64 < one 256-row down tile: masked
    rows), forced onto the prefill path at every B, top_n 0/1/2."""
    from paper_2512_17073_b200.device import LRCMoELayer

    st, layers = _toy()
    st16 = lrc.round_store_meta(st)
    xs = lrc.to_bf16(np.random.default_rng(B).standard_normal((B, 64)))
    xb = torch.from_numpy(xs).cuda().to(torch.bfloat16)
    for l in range(2):
        dl = LRCMoELayer.from_artifacts(layers[l].gate, st, l, 8, 1, 64, 128, max_tokens=max(B, 16))
        assert dl.prefill_eligible
        dl.set_prefill_min(1)
        for top_n in (0, 1, 2):
            y, _, _ = dl.forward(xb, top_k=2, top_n=top_n)
            y = y.double().cpu().numpy()
            for t in sorted({0, B // 2, B - 1}):
                yo = lrc.forward(xs[t], layers[l].gate, None, 2, top_n, "compensated", st16, l,
                                 shared=layers[l].shared)
                assert rel_l2(y[t], yo) <= TOL_Y, (l, top_n, t, rel_l2(y[t], yo))


def test_prefill_equals_decode_path(torch):
    """Same layer, same tokens: prefill GEMM vs the tiled decode kernels."""
    from paper_2512_17073_b200.synth import SynthLayer

    B = 700
    sl = SynthLayer(512, 1024, 8, top_k=2, rank=32, seed=5, max_tokens=B)
    assert sl.layer.prefill_eligible
    xs = torch.randn((B, 512), device="cuda").to(torch.bfloat16)
    for top_n in (0, 1, 2):
        sl.layer.set_prefill_min(1)
        yp, ip, _ = sl.layer.forward(xs, top_k=2, top_n=top_n)
        yp, ip = yp.double().cpu().numpy(), ip.cpu().numpy()
        sl.layer.set_prefill_min(0)
        yd, idd, _ = sl.layer.forward(xs, top_k=2, top_n=top_n)
        yd, idd = yd.double().cpu().numpy(), idd.cpu().numpy()
        assert np.array_equal(ip, idd)
        # both within 1e-2 of the oracle; they differ by the prefill path's bf16
        # rounding of dequantized weights and of the t vectors
        errs = [rel_l2(yp[t], yd[t]) for t in range(B)]
        assert max(errs) <= TOL_Y and float(np.mean(errs)) <= 5e-3, (top_n, max(errs), np.mean(errs))


@pytest.mark.parametrize("B", [256, 600])
def test_mixtral_shape_prefill_vs_oracle(torch, B):
    """C2 dims (d=4096, ffn=14336, 8 experts top-2, INT2 + r32 top-1) at prefill
    batch sizes; the default threshold routes B >= 128 to the tcgen05 path."""
    from paper_2512_17073_b200.synth import SynthLayer

    sl = SynthLayer(4096, 14336, 8, top_k=2, rank=32, seed=11, max_tokens=B)
    xs = lrc.to_bf16(np.random.default_rng(B).standard_normal((B, 4096)))
    xb = torch.from_numpy(xs).cuda().to(torch.bfloat16)
    yc, idx, _ = sl.layer.forward(xb, top_k=2, top_n=1)
    yq, _, _ = sl.layer.forward(xb, top_k=2, top_n=0)
    yc, yq, idx = yc.double().cpu().numpy(), yq.double().cpu().numpy(), idx.cpu().numpy()
    check = [0, B - 1]
    st = bridge.synth_store(sl, sorted({int(e) for t in check for e in idx[t]}))
    for t in check:
        _, sel, _ = lrc.route(xs[t], sl.gate, 2, 1)
        assert sel == list(idx[t])
        yo_c = lrc.forward(xs[t], sl.gate, None, 2, 1, "compensated", st)
        yo_q = lrc.forward(xs[t], sl.gate, None, 2, 0, "compensated", st)
        assert rel_l2(yc[t], yo_c) <= TOL_Y
        assert rel_l2(yq[t], yo_q) <= TOL_Y
        assert np.linalg.norm((yc[t] - yq[t]) - (yo_c - yo_q)) <= TOL_Y * np.linalg.norm(yo_c)


def test_prefill_lr_only_vs_oracle(torch):
    """Weights zeroed: the output comes ONLY from the K-augmentation slabs."""
    from paper_2512_17073_b200.synth import SynthLayer

    B = 300
    sl = SynthLayer(4096, 14336, 8, top_k=2, rank=32, seed=21, max_tokens=B, zero_weights=True)
    xs = lrc.to_bf16(np.random.default_rng(7).standard_normal((B, 4096)))
    y, idx, _ = sl.layer.forward(torch.from_numpy(xs).cuda().to(torch.bfloat16), top_k=2, top_n=1)
    y, idx = y.double().cpu().numpy(), idx.cpu().numpy()
    assert np.abs(y).max() > 0
    check = [0, 1, B - 1]
    st = bridge.synth_store(sl, sorted({int(e) for t in check for e in idx[t]}))
    for t in check:
        yo = lrc.forward(xs[t], sl.gate, None, 2, 1, "compensated", st)
        assert rel_l2(y[t], yo) <= TOL_LR, rel_l2(y[t], yo)


def test_prefill_skewed_routing(torch):
    """All tokens on one expert pair (ragged: one expert with B pairs spanning
    several 256-pair tiles, the rest empty) and renormalized weights."""
    from paper_2512_17073_b200.synth import SynthLayer

    B = 777
    sl = SynthLayer(512, 1024, 8, top_k=2, rank=16, seed=3, max_tokens=B)
    x1 = torch.randn((1, 512), device="cuda")
    xs = (x1 + 0.01 * torch.randn((B, 512), device="cuda")).to(torch.bfloat16)
    sl.layer.set_prefill_min(1)
    yp, ip, _ = sl.layer.forward(xs, top_k=2, top_n=1, renormalize=True)
    sl.layer.set_prefill_min(0)
    yd, idd, _ = sl.layer.forward(xs, top_k=2, top_n=1, renormalize=True)
    ip = ip.cpu().numpy()
    assert len({tuple(r) for r in ip}) <= 3
    assert np.array_equal(ip, idd.cpu().numpy())
    yp, yd = yp.double().cpu().numpy(), yd.double().cpu().numpy()
    assert max(rel_l2(yp[t], yd[t]) for t in range(B)) <= TOL_Y


@pytest.mark.parametrize("prefill", [False, True])
def test_parallel_plan_matches_serial_plan(torch, prefill):
    """B * (k + S) > 2048 pairs builds the pair plan with the parallel counting
    sort; the same tokens in two halves use the serial plan.  Same routing and
    the same per-token outputs (decode tiled path and prefill path), with
    compensated shared experts (S = 1)."""
    from paper_2512_17073_b200.synth import SynthLayer

    B = 1100  # 3300 pairs
    sl = SynthLayer(512, 1024, 8, top_k=2, num_shared=1, rank=16, seed=9, max_tokens=B)
    sl.layer.set_prefill_min(1 if prefill else 0)
    xs = torch.randn((B, 512), device="cuda").to(torch.bfloat16)
    yb, ib, _ = sl.layer.forward(xs, top_k=2, top_n=1)
    yb, ib = yb.double().cpu().numpy(), ib.cpu().numpy()
    h = B // 2
    y1, i1, _ = sl.layer.forward(xs[:h].contiguous(), top_k=2, top_n=1)
    y1, i1 = y1.double().cpu().numpy(), i1.cpu().numpy()
    y2, i2, _ = sl.layer.forward(xs[h:].contiguous(), top_k=2, top_n=1)
    y2, i2 = y2.double().cpu().numpy(), i2.cpu().numpy()
    assert np.array_equal(ib, np.concatenate([i1, i2]))
    ys = np.concatenate([y1, y2])
    assert max(rel_l2(yb[t], ys[t]) for t in range(B)) <= 1e-3


def test_pairs_mode_prefill_matches_decode(torch):
    """Expert-parallel receive side (lrc_layer_forward_pairs: routing given per
    row, k = 1, per-row compensation flag) on the prefill path (B >= 128) vs the
    decode kernels."""
    from paper_2512_17073_b200.synth import SynthLayer

    B = 400
    sl = SynthLayer(512, 1024, 8, top_k=2, rank=16, seed=13, max_tokens=B)
    g = torch.Generator(device="cpu").manual_seed(3)
    xs = torch.randn((B, 512), device="cuda").to(torch.bfloat16)
    ex = torch.randint(0, 8, (B,), generator=g, dtype=torch.int32)
    w = torch.rand((B,), generator=g)
    comp = (torch.rand((B,), generator=g) < 0.5).to(torch.uint8)
    sl.layer.set_prefill_min(1)
    yp = sl.layer.forward_pairs(xs, ex, w, comp).double().cpu().numpy()
    sl.layer.set_prefill_min(0)
    yd = sl.layer.forward_pairs(xs, ex, w, comp).double().cpu().numpy()
    assert np.abs(yd).max() > 0
    assert max(rel_l2(yp[t], yd[t]) for t in range(B)) <= TOL_Y


def test_deepseek_shape_prefill(torch):
    """C5 shape (64 experts top-8, top-2 restore, d=2048, ffn=11008 = 43 x 256)
    on the prefill path: many small per-expert tiles; vs the decode path and
    the oracle."""
    from paper_2512_17073_b200.synth import SynthLayer

    B = 300
    sl = SynthLayer(2048, 11008, 64, top_k=8, rank=32, seed=2, max_tokens=B)
    assert sl.layer.prefill_eligible
    xs = lrc.to_bf16(np.random.default_rng(5).standard_normal((B, 2048)))
    xb = torch.from_numpy(xs).cuda().to(torch.bfloat16)
    sl.layer.set_prefill_min(1)
    yp, ip, _ = sl.layer.forward(xb, top_k=8, top_n=2)
    sl.layer.set_prefill_min(0)
    yd, idd, _ = sl.layer.forward(xb, top_k=8, top_n=2)
    yp, yd, ip = yp.double().cpu().numpy(), yd.double().cpu().numpy(), ip.cpu().numpy()
    assert np.array_equal(ip, idd.cpu().numpy())
    assert max(rel_l2(yp[t], yd[t]) for t in range(B)) <= TOL_Y
    st = bridge.synth_store(sl, sorted({int(e) for t in (0, B - 1) for e in ip[t]}))
    for t in (0, B - 1):
        yo = lrc.forward(xs[t], sl.gate, None, 8, 2, "compensated", st)
        assert rel_l2(yp[t], yo) <= TOL_Y, rel_l2(yp[t], yo)


def test_bulk_router_indices_bit_exact(torch):
    """Large batches route with the bulk router (routing only) + parallel plan:
    every token's top-k indices bit-exact against the fp64 oracle router."""
    from paper_2512_17073_b200.synth import SynthLayer

    B = 3000  # 6000 pairs > the serial-plan limit
    sl = SynthLayer(4096, 14336, 8, top_k=2, rank=32, seed=17, max_tokens=B)
    xs = lrc.to_bf16(np.random.default_rng(17).standard_normal((B, 4096)))
    _, idx, w = sl.layer.forward(torch.from_numpy(xs).cuda().to(torch.bfloat16), top_k=2, top_n=1)
    idx, w = idx.cpu().numpy(), w.cpu().numpy()
    for t in range(B):
        wo, sel, _ = lrc.route(xs[t], sl.gate, 2, 1)
        assert sel == list(idx[t]), (t, sel, idx[t])
    assert np.all(np.isfinite(w)) and np.all(w > 0)
