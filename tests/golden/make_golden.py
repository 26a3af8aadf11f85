"""Generate golden vectors by importing the REAL reference (build container only).

    python tests/golden/make_golden.py            # needs /root/reference

Writes ``tests/golden/golden.npz`` (small arrays) and ``tests/golden/c1.json``
(checksums + outputs at the reference's tiny config C1).  The fixtures pin
``oracle/lrc.py`` (tests/test_oracle_golden.py) and are the reference-side
ground truth for the GPU parity tests; nothing at run time on the GPU box
reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()[:32]


def main():
    sys.path.insert(0, REF)
    from moe_lrc import lowrank, moe, quant
    from moe_lrc.pipeline import compress_model, uniform_allocation
    from moe_lrc.ranks import kurtosis_profile

    G: dict[str, np.ndarray] = {}

    # ---- pack / unpack (ref/quant.py:243-262) -------------------------------
    G["pack_2"] = np.frombuffer(quant.pack_codes(np.array([0, 1, 2, 3, 3, 2, 1, 0]), 2), np.uint8)
    G["pack_3"] = np.frombuffer(quant.pack_codes(np.array([1, 2, 3, 4, 5, 6, 7, 0]), 3), np.uint8)
    G["pack_4"] = np.frombuffer(quant.pack_codes(np.array([1, 2, 3, 15]), 4), np.uint8)
    for bits in (2, 3, 4):
        for n in (1, 7, 8, 64, 1000, 4099):
            c = np.random.default_rng(n * 10 + bits).integers(0, 1 << bits, n, dtype=np.uint8)
            G[f"packrand_{bits}_{n}_codes"] = c
            G[f"packrand_{bits}_{n}_bytes"] = np.frombuffer(quant.pack_codes(c, bits), np.uint8)

    # ---- quantize (ref/quant.py:146-213) ------------------------------------
    qcases = []
    for i, (shape, bits, gs, hqq, dist) in enumerate([
        ((8, 32), 2, 8, 0, "n"), ((5, 17), 3, 4, 0, "n"), ((3, 7), 4, 16, 0, "n"),
        ((4, 70), 2, 32, 0, "n"), ((16, 64), 2, 32, 20, "t3"), ((8, 64), 2, 64, 20, "t4"),
        ((32, 128), 3, 64, 20, "n"), ((24, 200), 2, 64, 20, "n"), ((12, 64), 4, 64, 20, "t3"),
        ((4, 8), 2, 4, 0, "zero"), ((64, 256), 2, 64, 20, "n"), ((40, 16), 3, 16, 20, "n"),
    ]):
        rng = np.random.default_rng(100 + i)
        if dist == "n":
            w = rng.standard_normal(shape)
        elif dist == "zero":
            w = np.zeros(shape)
        else:
            w = rng.standard_t(int(dist[1:]), size=shape)
        qm = quant.quantize(w, quant.QuantConfig(bits=bits, group_size=gs, hqq_iters=hqq))
        G[f"q{i}_w"] = w
        G[f"q{i}_codes"] = qm.codes
        G[f"q{i}_scales"] = qm.scales
        G[f"q{i}_zeros"] = qm.zero_points
        G[f"q{i}_deq"] = quant.dequantize(qm)
        qcases.append([i, bits, gs, hqq])
    G["qcases"] = np.array(qcases)

    # ---- truncated SVD + compensator (ref/lowrank.py:72-165) -----------------
    scases = []
    for i, (shape, r, seed) in enumerate([((64, 64), 8, 3), ((96, 48), 12, 0), ((40, 60), 6, 11),
                                          ((128, 64), 16, 5)]):
        e = np.random.default_rng(200 + i).standard_normal(shape)
        u, s, vt = lowrank.truncated_svd(e, r, seed=seed)
        G[f"svd{i}_e"], G[f"svd{i}_u"], G[f"svd{i}_s"], G[f"svd{i}_vt"] = e, u, s, vt
        scases.append([i, r, seed])
    G["svdcases"] = np.array(scases)
    ccases = []
    for i, (shape, r, bits) in enumerate([((32, 48), 8, 2), ((64, 64), 16, 2), ((128, 64), 32, 3)]):
        w = np.random.default_rng(300 + i).standard_normal(shape)
        qm = quant.quantize(w, quant.QuantConfig(bits=bits, group_size=64, hqq_iters=0))
        c = lowrank.build_compensator(w, qm, r, seed=7)
        G[f"comp{i}_w"] = w
        for f in ("u", "v"):
            fq = getattr(c, f)
            G[f"comp{i}_{f}_codes"] = fq.codes
            G[f"comp{i}_{f}_scales"] = fq.scales
            G[f"comp{i}_{f}_zeros"] = fq.zero_points
        G[f"comp{i}_applied"] = lowrank.apply_compensation(qm, c)
        ccases.append([i, r, bits])
    G["compcases"] = np.array(ccases)

    # ---- routing (ref/moe.py:183-193) ---------------------------------------
    G["route_tie_sel"] = np.array(moe.route(
        np.ones(4), moe.MoELayer(gate=np.zeros((4, 4)), experts=[None] * 4),
        moe.ForwardConfig(top_k=2)).selected)
    for i, (d, E, k, n) in enumerate([(64, 8, 2, 1), (512, 8, 2, 1), (256, 64, 8, 2), (128, 128, 8, 2)]):
        m = moe.gen_synthetic_model(seed=400 + i, hidden=d, ffn=16, num_layers=1, num_experts=E,
                                    top_k=k, router_skew=1.4)
        toks = moe.gen_tokens(500 + i, d, 64)
        sel, wts = [], []
        for x in toks:
            rr = moe.route(x, m.layers[0], moe.ForwardConfig(top_k=k, top_n=n))
            sel.append(rr.selected)
            wts.append(rr.weights)
        G[f"route{i}_gate"] = m.layers[0].gate
        G[f"route{i}_x"] = toks
        G[f"route{i}_sel"] = np.array(sel)
        G[f"route{i}_w"] = np.array(wts)

    # ---- toy model end to end (gen -> compress -> forward, 3 modes) ----------
    m = moe.gen_synthetic_model(seed=7, hidden=64, ffn=128, num_layers=2, num_experts=8, top_k=2,
                                num_shared=1, tail_dofs=(4.0, math.inf), router_skew=1.4)
    prof = kurtosis_profile(m)
    cm = compress_model(m, quant.QuantConfig(bits=2, group_size=64, hqq_iters=20),
                        uniform_allocation(prof, 16), prof, seed=3)
    G["toy_sha"] = np.array([sha(m.layers[0].gate), sha(m.layers[1].experts[3].w2),
                             sha(m.layers[1].shared_experts[0].w1)])
    for (l, e, p), rec in sorted(cm.records.items()):
        key = f"toy_l{l}_e{e}_{p}"
        G[key + "_codes"] = rec.qm.codes
        G[key + "_scales"] = rec.qm.scales
        G[key + "_zeros"] = rec.qm.zero_points
        for f in ("u", "v"):
            fq = getattr(rec.comp, f)
            G[f"{key}_{f}_codes"] = fq.codes
            G[f"{key}_{f}_scales"] = fq.scales
            G[f"{key}_{f}_zeros"] = fq.zero_points
    toks = moe.gen_tokens(11, 64, 6)
    G["toy_x"] = toks
    for mode in ("reference", "quantized", "compensated"):
        for l in range(2):
            ys = [moe.forward(x, m.layers[l], moe.ForwardConfig(top_k=2, top_n=1), mode,
                              None if mode == "reference" else cm, layer_id=l) for x in toks]
            G[f"toy_y_{mode}_l{l}"] = np.array(ys)
    rep = moe.evaluate_fidelity(m, cm, toks, moe.ForwardConfig(top_k=2, top_n=1))
    G["toy_fidelity"] = np.array([rep.mean_rel_err["quantized"], rep.mean_rel_err["compensated"],
                                  rep.win_rate])

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **G)

    # ---- C1: the reference's tiny config, as checksums + outputs ---------------
    t0 = time.time()
    m = moe.gen_synthetic_model(seed=0, hidden=512, ffn=1024, num_layers=1, num_experts=8,
                                top_k=2, router_skew=1.4)
    prof = kurtosis_profile(m)
    cm = compress_model(m, quant.QuantConfig(bits=2, group_size=64, hqq_iters=20),
                        uniform_allocation(prof, 16), prof, seed=0)
    c1 = {"config": "gen_synthetic_model(seed=0, hidden=512, ffn=1024, num_layers=1, "
                    "num_experts=8, top_k=2, router_skew=1.4); compress_model(QuantConfig(2,64,20), "
                    "uniform_allocation(16), seed=0); ForwardConfig(top_k=2, top_n=1); "
                    "gen_tokens(1, 512, 4)",
          "model_sha": {"gate": sha(m.layers[0].gate), "e0_w1": sha(m.layers[0].experts[0].w1),
                        "e7_w2": sha(m.layers[0].experts[7].w2)},
          "records": {}}
    for (l, e, p), rec in sorted(cm.records.items()):
        c1["records"][f"{e}_{p}"] = {
            "codes": sha(rec.qm.codes), "scales": sha(rec.qm.scales), "zeros": sha(rec.qm.zero_points),
            "u_codes": sha(rec.comp.u.codes), "v_codes": sha(rec.comp.v.codes),
            "u_scales": sha(rec.comp.u.scales), "v_scales": sha(rec.comp.v.scales)}
    toks = moe.gen_tokens(1, 512, 4)
    cfg = moe.ForwardConfig(top_k=2, top_n=1)
    c1["routes"] = [moe.route(x, m.layers[0], cfg).selected for x in toks]
    c1["y_compensated"] = [moe.forward(x, m.layers[0], cfg, "compensated", cm).tolist() for x in toks]
    c1["y_quantized"] = [moe.forward(x, m.layers[0], cfg, "quantized", cm).tolist() for x in toks]
    c1["y_reference"] = [moe.forward(x, m.layers[0], cfg, "reference").tolist() for x in toks]
    c1["seconds_compress"] = time.time() - t0
    with open(os.path.join(HERE, "c1.json"), "w") as f:
        json.dump(c1, f)
    print("wrote golden.npz and c1.json")


if __name__ == "__main__":
    main()
