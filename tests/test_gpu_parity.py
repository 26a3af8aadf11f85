"""GPU parity: every CUDA entry point of liblrc against the oracle / golden vectors.

Contracts: codes, packed bytes, routing indices and the T2 tile
repack are bit-exact; fp64 dequantize is bit-exact; layer outputs are within
max relative L2 <= 1e-2 of the fp64 oracle fed the same bf16 tokens and fp16
scale/zero (and the LR delta y_comp - y_quant within 5e-2).
"""

import math
import os

import numpy as np
import pytest

from oracle import bridge, lrc

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))
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


# ------------------------------------------------------------------ codes --
@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("n", [1, 7, 8, 64, 1000, 4099])
def test_pack_unpack_bit_exact(torch, bits, n):
    from paper_2512_17073_b200 import quant

    c = G[f"packrand_{bits}_{n}_codes"]
    b = bytes(G[f"packrand_{bits}_{n}_bytes"])
    assert quant.pack_codes(c, bits) == b
    np.testing.assert_array_equal(quant.unpack_codes(b, n, bits), c)


def test_pack_examples(torch):
    from paper_2512_17073_b200 import quant

    assert quant.pack_codes(np.array([0, 1, 2, 3, 3, 2, 1, 0]), 2) == bytes([228, 27])
    assert quant.pack_codes(np.array([1, 2, 3, 4, 5, 6, 7, 0]), 3) == bytes(G["pack_3"])
    assert quant.pack_codes(np.array([1, 2, 3, 15]), 4) == bytes([0x21, 0xF3])


@pytest.mark.parametrize("case", range(12))
def test_dequantize_bit_exact(torch, case):
    from paper_2512_17073_b200 import quant

    i, bits, gs, hqq = G["qcases"][case]
    codes = G[f"q{i}_codes"]
    qm = quant.QuantizedMatrix(codes.shape[0], codes.shape[1], int(bits), int(gs), codes,
                               G[f"q{i}_scales"], G[f"q{i}_zeros"])
    np.testing.assert_array_equal(quant.dequantize(qm), G[f"q{i}_deq"])


@pytest.mark.parametrize("case", range(12))
def test_quantize_vs_reference(torch, case):
    from paper_2512_17073_b200 import quant

    i, bits, gs, hqq = (int(v) for v in G["qcases"][case])
    qm = quant.quantize(G[f"q{i}_w"], quant.QuantConfig(bits=bits, group_size=gs, hqq_iters=hqq))
    np.testing.assert_array_equal(qm.scales, G[f"q{i}_scales"])
    if hqq == 0:
        np.testing.assert_array_equal(qm.codes, G[f"q{i}_codes"])
        np.testing.assert_array_equal(qm.zero_points, G[f"q{i}_zeros"])
    else:
        # HQQ: CUDA pow() may differ from glibc's in the last ulp; codes must agree
        # on >= 99.5% and zero points to 1e-9 relative.
        agree = float(np.mean(qm.codes == G[f"q{i}_codes"]))
        assert agree >= 0.995, agree
        np.testing.assert_allclose(qm.zero_points, G[f"q{i}_zeros"], rtol=1e-9, atol=1e-12)


# ------------------------------------------------------------------ tiles --
@pytest.mark.parametrize("rows,cols", [(16, 128), (37, 200), (14336 // 8, 4096 // 4), (64, 64), (5, 33)])
@pytest.mark.parametrize("ni", [1, 2])
def test_tiles_round_trip_bit_exact(torch, rows, cols, ni):
    import paper_2512_17073_b200._lib as L
    from paper_2512_17073_b200 import device, quant

    rng = np.random.default_rng(rows * cols + ni)
    keep = device._Keep()
    mats, codes = [], []
    for i in range(ni):
        c = rng.integers(0, 4, (rows, cols), dtype=np.uint8)
        qm = quant.QuantizedMatrix(rows, cols, 2, 64, c, rng.random((rows, -(-cols // 64))),
                                   rng.random((rows, -(-cols // 64))))
        mats.append(device._qm_to_device(qm, keep))
        codes.append(c)
    tiles = device.build_tiles(mats, keep)
    lib = L.lib()
    for i in range(ni):
        out = torch.empty((rows, cols), dtype=torch.uint8, device="cuda")
        L.check(lib.lrc_tiles_unpack(L.ptr(tiles), rows, cols, ni, i, L.ptr(out), L.stream_ptr()))
        np.testing.assert_array_equal(out.cpu().numpy(), codes[i])


# ---------------------------------------------------------------- routing --
def test_route_tie_break(torch):
    from paper_2512_17073_b200 import moe

    layer = moe.MoELayer(gate=np.zeros((4, 4)), experts=[None] * 4)
    rr = moe.route(np.ones(4), layer, moe.ForwardConfig(top_k=2))
    assert rr.selected == [0, 1]
    np.testing.assert_allclose(rr.weights, [0.25] * 4)


def test_route_known_softmax(torch):
    from paper_2512_17073_b200 import moe

    layer = moe.MoELayer(gate=np.array([[math.log(2.0), 0.0]]), experts=[None] * 2)
    rr = moe.route(np.ones(1), layer, moe.ForwardConfig(top_k=2))
    np.testing.assert_allclose(rr.weights, [2 / 3, 1 / 3], rtol=1e-12)


@pytest.mark.parametrize("case,k,n", [(0, 2, 1), (1, 2, 1), (2, 8, 2), (3, 8, 2)])
def test_route_golden_indices_bit_exact(torch, case, k, n):
    from paper_2512_17073_b200 import moe

    gate, xs = G[f"route{case}_gate"], G[f"route{case}_x"]
    layer = moe.MoELayer(gate=gate, experts=[None] * gate.shape[1])
    for t, x in enumerate(xs):
        rr = moe.route(x, layer, moe.ForwardConfig(top_k=k, top_n=n))
        assert rr.selected == list(G[f"route{case}_sel"][t])
        assert rr.compensated == rr.selected[:n]
        np.testing.assert_allclose(rr.weights, G[f"route{case}_w"][t], rtol=1e-12, atol=1e-15)


def test_router_bf16_batch_matches_oracle(torch):
    """The fused layer router on bf16 tokens == oracle route on the same rounded tokens."""
    from paper_2512_17073_b200.synth import SynthLayer

    sl = SynthLayer(512, 256, 64, top_k=8, rank=0, seed=3, max_tokens=256)
    xs = lrc.to_bf16(np.random.default_rng(0).standard_normal((256, 512)))
    xb = torch.from_numpy(xs).cuda().to(torch.bfloat16)
    _, idx, w = sl.layer.forward(xb, top_k=8, top_n=2)
    idx = idx.cpu().numpy()
    flips = 0
    for t in range(256):
        probs, sel, _ = lrc.route(xs[t], sl.gate, 8, 2)
        flips += list(idx[t]) != sel
    assert flips == 0


# ------------------------------------------------------- layer forward -----
def _toy_store():
    st = lrc.Store()
    for key in G.files:
        if key.startswith("toy_l") and key.endswith("_codes") and "_u_" not in key and "_v_" not in key:
            base = key[: -len("_codes")]
            _, l, e, p = base.split("_")
            l, e = int(l[1:]), int(e[1:])
            qm = lrc.QM(*G[key].shape, 2, 64, G[key], G[base + "_scales"], G[base + "_zeros"])
            f = {}
            for fn in ("u", "v"):
                c = G[f"{base}_{fn}_codes"]
                f[fn] = lrc.QM(*c.shape, 3, min(64, c.shape[1]), c, G[f"{base}_{fn}_scales"],
                               G[f"{base}_{fn}_zeros"])
            st.records[(l, e, p)] = lrc.Rec(qm, lrc.Comp(16, f["u"], f["v"], p))
    return st


def _toy_layers():
    return lrc.gen_model(7, 64, 128, 2, 8, num_shared=1, tail_dofs=(4.0, math.inf), router_skew=1.4)


@pytest.mark.parametrize("generic", [False, True])
def test_toy_layer_vs_oracle(torch, generic):
    """Reference-compressed toy model (golden artifacts): device forward vs oracle."""
    from paper_2512_17073_b200.device import LRCMoELayer

    st = _toy_store()
    st16 = lrc.round_store_meta(st)
    layers = _toy_layers()
    xs = lrc.to_bf16(G["toy_x"])
    for l in range(2):
        dl = LRCMoELayer.from_artifacts(layers[l].gate, st, l, 8, 1, 64, 128)
        assert dl.tiled
        xb = torch.from_numpy(xs).cuda().to(torch.bfloat16)
        for top_n in (0, 1, 2):
            y, _, _ = dl.forward(xb, top_k=2, top_n=top_n, generic=generic)
            y = y.double().cpu().numpy()
            for t in range(len(xs)):
                yo = lrc.forward(xs[t], layers[l].gate, None, 2, top_n, "compensated", st16, l,
                                 shared=layers[l].shared)
                assert rel_l2(y[t], yo) <= TOL_Y, (l, top_n, t, rel_l2(y[t], yo))


def test_toy_api_forward_vs_reference_golden(torch):
    """moe.forward (numpy API) against the REFERENCE's own outputs (fp64 meta, fp64 x)."""
    from paper_2512_17073_b200 import moe

    st = _toy_store()
    model_layers = _toy_layers()
    for l in range(2):
        ml = moe.MoELayer(gate=model_layers[l].gate,
                          experts=[moe.Expert(*e) for e in model_layers[l].experts],
                          shared_experts=[moe.Expert(*e) for e in model_layers[l].shared])
        cfg = moe.ForwardConfig(top_k=2, top_n=1)
        for t, x in enumerate(G["toy_x"]):
            for mode in ("reference", "quantized", "compensated"):
                y = moe.forward(x, ml, cfg, mode, None if mode == "reference" else st, l)
                want = G[f"toy_y_{mode}_l{l}"][t]
                tol = 1e-12 if mode == "reference" else TOL_Y
                assert rel_l2(y, want) <= tol, (mode, l, t, rel_l2(y, want))


def test_fidelity_matches_reference(torch):
    from paper_2512_17073_b200 import moe

    st = _toy_store()
    layers = _toy_layers()
    model = moe.MoEModel(64, 128, [moe.MoELayer(l.gate, [moe.Expert(*e) for e in l.experts],
                                                [moe.Expert(*e) for e in l.shared]) for l in layers],
                         top_k=2)
    rep = moe.evaluate_fidelity(model, st, G["toy_x"], moe.ForwardConfig(top_k=2, top_n=1))
    q, c, wr = G["toy_fidelity"]
    assert abs(rep.mean_rel_err["quantized"] - q) < 5e-3 * q + 1e-4
    assert abs(rep.mean_rel_err["compensated"] - c) < 5e-3 * c + 1e-4
    assert rep.mean_rel_err["compensated"] < rep.mean_rel_err["quantized"]


@pytest.mark.parametrize("B", [1, 3, 8, 16, 40])
def test_mixtral_shape_layer_vs_oracle(torch, B):
    """C2: d=4096, ffn=14336, 8 experts top-2, INT2 + rank-32 top-1, decode batch B."""
    from paper_2512_17073_b200.synth import SynthLayer

    sl = SynthLayer(4096, 14336, 8, top_k=2, rank=32, seed=11, max_tokens=64)
    xs = lrc.to_bf16(np.random.default_rng(B).standard_normal((B, 4096)))
    xb = torch.from_numpy(xs).cuda().to(torch.bfloat16)
    yc, idx, _ = sl.layer.forward(xb, top_k=2, top_n=1)
    yq, _, _ = sl.layer.forward(xb, top_k=2, top_n=0)
    yc, yq, idx = yc.double().cpu().numpy(), yq.double().cpu().numpy(), idx.cpu().numpy()
    check = range(B) if B <= 3 else [0, B - 1]
    used = sorted({int(e) for t in check for e in idx[t]})
    st = bridge.synth_store(sl, used)
    for t in check:
        _, sel, _ = lrc.route(xs[t], sl.gate, 2, 1)
        assert sel == list(idx[t])
        yo_c = lrc.forward(xs[t], sl.gate, None, 2, 1, "compensated", st)
        yo_q = lrc.forward(xs[t], sl.gate, None, 2, 0, "compensated", st)
        assert rel_l2(yc[t], yo_c) <= TOL_Y
        assert rel_l2(yq[t], yo_q) <= TOL_Y
        # the LR delta agrees to the same absolute accuracy as the layer output
        assert np.linalg.norm((yc[t] - yq[t]) - (yo_c - yo_q)) <= TOL_Y * np.linalg.norm(yo_c)


@pytest.mark.parametrize("B", [1, 5, 16])
def test_lr_path_only_vs_oracle(torch, B):
    """Weights zeroed: the output is produced ONLY by the fused low-rank path
    w * U2.(V2.(silu(U1.(V1.x)) * U3.(V3.x))) -- checks the LR fusion at LR_TOL."""
    from paper_2512_17073_b200.synth import SynthLayer

    sl = SynthLayer(4096, 14336, 8, top_k=2, rank=32, seed=21, max_tokens=64, zero_weights=True)
    xs = lrc.to_bf16(np.random.default_rng(100 + B).standard_normal((B, 4096)))
    y, idx, _ = sl.layer.forward(torch.from_numpy(xs).cuda().to(torch.bfloat16), top_k=2, top_n=1)
    y, idx = y.double().cpu().numpy(), idx.cpu().numpy()
    assert np.abs(y).max() > 0
    st = bridge.synth_store(sl, sorted({int(e) for e in idx.ravel()}))
    for t in range(B):
        yo = lrc.forward(xs[t], sl.gate, None, 2, 1, "compensated", st)
        assert rel_l2(y[t], yo) <= TOL_LR, rel_l2(y[t], yo)
        assert rel_l2(y[t], yo) <= TOL_Y, rel_l2(y[t], yo)


def test_tiled_equals_generic_path(torch):
    from paper_2512_17073_b200.synth import SynthLayer

    sl = SynthLayer(1024, 2048, 8, top_k=2, rank=16, seed=5, max_tokens=64)
    xs = torch.randn((24, 1024), device="cuda").to(torch.bfloat16)
    yt, _, _ = sl.layer.forward(xs, top_k=2, top_n=1)
    yg, _, _ = sl.layer.forward(xs, top_k=2, top_n=1, generic=True)
    yt, yg = yt.double().cpu().numpy(), yg.double().cpu().numpy()
    for t in range(24):
        assert rel_l2(yt[t], yg[t]) <= 5e-3


def test_deepseek_shape_vs_oracle(torch):
    """C5 shape on one GPU: 64 experts top-8, top-2 restore, d=2048, ffn=11008."""
    from paper_2512_17073_b200.synth import SynthLayer

    sl = SynthLayer(2048, 11008, 64, top_k=8, rank=32, seed=2, max_tokens=16)
    xs = lrc.to_bf16(np.random.default_rng(9).standard_normal((2, 2048)))
    y, idx, _ = sl.layer.forward(torch.from_numpy(xs).cuda().to(torch.bfloat16), top_k=8, top_n=2)
    y, idx = y.double().cpu().numpy(), idx.cpu().numpy()
    st = bridge.synth_store(sl, sorted({int(e) for e in idx.ravel()}))
    for t in range(2):
        yo = lrc.forward(xs[t], sl.gate, None, 8, 2, "compensated", st)
        assert rel_l2(y[t], yo) <= TOL_Y


# ------------------------------------------------ reference API behaviour --
def _api_model(seed, hidden=32, ffn=64, layers=2, experts=4, top_k=2, shared=0, skew=1.4):
    from paper_2512_17073_b200 import moe

    return moe.gen_synthetic_model(seed=seed, hidden=hidden, ffn=ffn, num_layers=layers,
                                   num_experts=experts, top_k=top_k, num_shared=shared,
                                   router_skew=skew)


def _api_compress(model, rank, bits=2, hqq=0, quantize_factors=True, seed=0):
    """compress_model (ref/pipeline.py:125-173) through the GPU quantizer/compensator."""
    from paper_2512_17073_b200 import lowrank, quant

    st = lrc.Store()
    qcfg = quant.QuantConfig(bits=bits, group_size=64, hqq_iters=hqq)
    for l, e, p, w in model.iter_projections():
        qm = quant.quantize(w, qcfg)
        r = min(rank, min(w.shape))
        comp = None
        if r > 0:
            s = int(np.random.SeedSequence([seed, l, e, ("w1", "w2", "w3").index(p)]).generate_state(1)[0])
            comp = lowrank.build_compensator(w, qm, r, projection_id=p, seed=s,
                                             quantize_factors=quantize_factors)
        st.records[(l, e, p)] = lrc.Rec(qm, comp)
    return st


def test_api_top_n_zero_equals_quantized_bit_exact(torch):
    from paper_2512_17073_b200 import moe

    model = _api_model(5)
    st = _api_compress(model, 16)
    x = moe.gen_tokens(1, 32, 1)[0]
    cfg = moe.ForwardConfig(top_k=2, top_n=0)
    yq = moe.forward(x, model.layers[0], cfg, "quantized", st, 0)
    yc = moe.forward(x, model.layers[0], cfg, "compensated", st, 0)
    np.testing.assert_array_equal(yq, yc)


def test_api_compensated_beats_quantized(torch):
    from paper_2512_17073_b200 import moe

    model = _api_model(7, hidden=64, ffn=128, experts=8)
    st = _api_compress(model, 32)
    cfg = moe.ForwardConfig(top_k=2, top_n=1)
    toks = moe.gen_tokens(3, 64, 100)
    wins = total = 0
    for lid, layer in enumerate(model.layers):
        yr = moe.forward_batch(toks, layer, cfg, "reference")
        yq = moe.forward_batch(toks, layer, cfg, "quantized", st, lid)
        yc = moe.forward_batch(toks, layer, cfg, "compensated", st, lid)
        wins += int(np.sum(np.linalg.norm(yc - yr, axis=1) < np.linalg.norm(yq - yr, axis=1)))
        total += len(toks)
    assert wins / total >= 0.95


def test_api_full_rank_raw_factors_recover_reference(torch):
    """ref tests/test_moe.py:96-103 at the device precision contract (bf16 tokens)."""
    from paper_2512_17073_b200 import moe

    model = _api_model(6)
    st = _api_compress(model, 64, quantize_factors=False)
    cfg = moe.ForwardConfig(top_k=2, top_n=2)
    for x in moe.gen_tokens(2, 32, 5):
        yr = moe.forward(x, model.layers[0], cfg, "reference")
        yc = moe.forward(x, model.layers[0], cfg, "compensated", st, 0)
        assert np.linalg.norm(yc - yr) <= TOL_Y * np.linalg.norm(yr)


def test_api_shared_expert_toggle(torch):
    from paper_2512_17073_b200 import moe

    model = _api_model(30, experts=4, shared=1)
    st = _api_compress(model, 16)
    x = moe.gen_tokens(31, 32, 1)[0]
    on = moe.ForwardConfig(top_k=2, top_n=1, compensate_shared=True)
    off = moe.ForwardConfig(top_k=2, top_n=1, compensate_shared=False)
    y_ref = moe.forward(x, model.layers[0], on, "reference")
    y_on = moe.forward(x, model.layers[0], on, "compensated", st, 0)
    y_off = moe.forward(x, model.layers[0], off, "compensated", st, 0)
    assert np.linalg.norm(y_on - y_off) > 0
    assert np.linalg.norm(y_on - y_ref) < np.linalg.norm(y_off - y_ref)


def test_api_renormalize(torch):
    from paper_2512_17073_b200 import moe

    model = _api_model(10, experts=4)
    st = _api_compress(model, 16)
    x = moe.gen_tokens(5, 32, 1)[0]
    for mode, art in (("reference", None), ("compensated", st)):
        # every mode routes the fp64 token, as the reference does (ADVICE r1:
        # the quantized / compensated device path used to route its bf16 copy)
        rr = moe.route(x, model.layers[0], moe.ForwardConfig(top_k=2))
        scale = rr.weights[rr.selected].sum()
        y_plain = moe.forward(x, model.layers[0], moe.ForwardConfig(top_k=2), mode, art, 0)
        y_ren = moe.forward(x, model.layers[0], moe.ForwardConfig(top_k=2, renormalize_topk=True),
                            mode, art, 0)
        np.testing.assert_allclose(y_ren * scale, y_plain, rtol=1e-5 if art else 1e-10,
                                   atol=1e-6 * np.abs(y_plain).max())


def test_api_missing_artifact(torch):
    from paper_2512_17073_b200 import moe

    model = _api_model(8)
    with pytest.raises(moe.MissingArtifactError):
        moe.forward(np.ones(32), model.layers[0], moe.ForwardConfig(top_k=1), "quantized", None)
    st = _api_compress(model, 0)
    sel = moe.route(np.ones(32), model.layers[0], moe.ForwardConfig(top_k=1)).selected[0]
    for p in ("w1", "w2", "w3"):
        del st.records[(0, sel, p)]
    with pytest.raises(moe.MissingArtifactError):
        moe.forward(np.ones(32), model.layers[0], moe.ForwardConfig(top_k=1), "quantized", st, 0)


def test_api_router_band_c7(torch):
    """Acceptance c7 (ref tests/test_acceptance.py:220-229) through the device router."""
    from paper_2512_17073_b200 import moe

    model = moe.gen_synthetic_model(seed=12, hidden=64, ffn=64, num_layers=1, num_experts=8,
                                    top_k=2, router_skew=1.4)
    trace = moe.build_trace(model, moe.ForwardConfig(top_k=2), num_tokens=10_000, seed=13)
    stats = moe.routing_stats(trace)
    assert stats.num_tokens >= 10_000
    assert 0.41 <= stats.aggregate[0] <= 0.48
    assert 0.15 <= stats.aggregate[1] <= 0.22


def test_api_uniform_router(torch):
    from paper_2512_17073_b200 import moe

    model = moe.gen_synthetic_model(seed=16, hidden=32, ffn=32, num_layers=1, num_experts=4,
                                    top_k=2, router_skew=0.0)
    stats = moe.routing_stats(moe.build_trace(model, moe.ForwardConfig(top_k=2), 50, 17))
    np.testing.assert_allclose(stats.aggregate, [0.25] * 4, atol=1e-12)


def test_lowrank_api(torch):
    from paper_2512_17073_b200 import lowrank, quant

    rng = np.random.default_rng(7)
    w = rng.standard_normal((24, 36))
    qm = quant.quantize(w, quant.QuantConfig(bits=2, group_size=64, hqq_iters=0))
    comp = lowrank.build_compensator(w, qm, 24, quantize_factors=False)
    assert np.linalg.norm(w - lowrank.apply_compensation(qm, comp)) <= 1e-6 * np.linalg.norm(w)
    np.testing.assert_array_equal(lowrank.apply_compensation(qm, None), quant.dequantize(qm))
    for i in range(4):
        cs = G["svdcases"][i]
        e = G[f"svd{i}_e"]
        r = int(cs[1])
        u, s, vt = lowrank.truncated_svd(e, r, int(cs[2]))
        # SPEC.md:120 invariants: orthonormal factors (1e-8) and Eckart-Young tail (1e-6 rel)
        np.testing.assert_allclose(u.T @ u, np.eye(r), atol=1e-8)
        np.testing.assert_allclose(vt @ vt.T, np.eye(r), atol=1e-8)
        opt = float(np.sqrt(np.sum(np.linalg.svd(e, compute_uv=False)[r:] ** 2)))
        assert abs(np.linalg.norm(e - u @ np.diag(s) @ vt) - opt) <= 1e-6 * opt
        np.testing.assert_allclose(s, G[f"svd{i}_s"], rtol=1e-6)
    c = lowrank.build_compensator(w, qm, 8)
    assert c.u.bits == 3 and c.u.shape == (24, 8) and c.v.shape == (8, 36)


@pytest.fixture(scope="module")
def c1_setup():
    """C1 (BASELINE configs[0]): the reference's tiny model and its compressed
    artifacts, rebuilt by the oracle -- bit-exact with the reference's own
    compress_model (every record's SHA in c1.json is checked here)."""
    import hashlib
    import json

    c1 = json.load(open(os.path.join(HERE, "golden", "c1.json")))
    layers = lrc.gen_model(0, 512, 1024, 1, 8, router_skew=1.4)
    st = lrc.compress(layers, bits=2, group_size=64, hqq_iters=20, rank=16, factor_bits=3, seed=0)

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]

    for (l, e, p), rec in st.records.items():
        r = c1["records"][f"{e}_{p}"]
        assert sha(rec.qm.codes) == r["codes"] and sha(rec.comp.u.codes) == r["u_codes"], (e, p)
    return c1, layers, st


@pytest.mark.parametrize("mode", ["compensated", "quantized"])
def test_c1_gpu_forward_vs_reference_outputs(torch, c1_setup, mode):
    """The GPU path (moe.forward -> lrc_route + lrc_layer_forward_pairs) on the
    reference's own C1 artifacts against the REFERENCE's outputs in c1.json
    (ref/moe.py:217-259 run in the build container): routes identical, layer
    outputs within 1e-2 relative L2 (bf16 tokens / fp16 metadata on the device)."""
    from paper_2512_17073_b200 import moe

    c1, layers, st = c1_setup
    ml = moe.MoELayer(gate=layers[0].gate, experts=[moe.Expert(*e) for e in layers[0].experts])
    cfg = moe.ForwardConfig(top_k=2, top_n=1)
    for t, x in enumerate(lrc.gen_tokens(1, 512, 4)):
        assert moe.route(x, ml, cfg).selected == c1["routes"][t]
        y = moe.forward(x, ml, cfg, mode, st, 0)
        want = np.asarray(c1[f"y_{mode}"][t])
        assert rel_l2(y, want) <= TOL_Y, (t, rel_l2(y, want))
