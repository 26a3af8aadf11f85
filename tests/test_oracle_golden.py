"""Pin the CPU oracle (oracle/lrc.py) against golden vectors from the real reference.

The fixtures come from tests/golden/make_golden.py, which imports the
reference package; these tests only read the committed fixtures.
"""

import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle import lrc

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def test_pack_examples():
    assert lrc.pack_codes(np.array([0, 1, 2, 3, 3, 2, 1, 0]), 2) == bytes(G["pack_2"]) == bytes([228, 27])
    assert lrc.pack_codes(np.array([1, 2, 3, 4, 5, 6, 7, 0]), 3) == bytes(G["pack_3"]) == \
        bytes([0b11010001, 0b01011000, 0b00011111])
    assert lrc.pack_codes(np.array([1, 2, 3, 15]), 4) == bytes(G["pack_4"]) == bytes([0x21, 0xF3])


@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("n", [1, 7, 8, 64, 1000, 4099])
def test_pack_unpack_golden(bits, n):
    c = G[f"packrand_{bits}_{n}_codes"]
    b = G[f"packrand_{bits}_{n}_bytes"]
    assert lrc.pack_codes(c, bits) == bytes(b)
    np.testing.assert_array_equal(lrc.unpack_codes(bytes(b), n, bits), c)


@pytest.mark.parametrize("case", range(12))
def test_quantize_golden_bit_exact(case):
    i, bits, gs, hqq = G["qcases"][case]
    qm = lrc.quantize(G[f"q{i}_w"], int(bits), int(gs), int(hqq))
    np.testing.assert_array_equal(qm.codes, G[f"q{i}_codes"])
    np.testing.assert_array_equal(qm.scales, G[f"q{i}_scales"])
    np.testing.assert_array_equal(qm.zero_points, G[f"q{i}_zeros"])
    np.testing.assert_array_equal(lrc.dequantize(qm), G[f"q{i}_deq"])


@pytest.mark.parametrize("case", range(4))
def test_truncated_svd_golden(case):
    i, r, seed = G["svdcases"][case]
    u, s, vt = lrc.truncated_svd(G[f"svd{i}_e"], int(r), int(seed))
    np.testing.assert_array_equal(s, G[f"svd{i}_s"])
    np.testing.assert_array_equal(u, G[f"svd{i}_u"])
    np.testing.assert_array_equal(vt, G[f"svd{i}_vt"])


@pytest.mark.parametrize("case", range(3))
def test_build_compensator_golden(case):
    i, r, bits = G["compcases"][case]
    w = G[f"comp{i}_w"]
    qm = lrc.quantize(w, int(bits), 64, 0)
    c = lrc.build_compensator(w, qm, int(r), seed=7)
    for f in ("u", "v"):
        np.testing.assert_array_equal(getattr(c, f).codes, G[f"comp{i}_{f}_codes"])
        np.testing.assert_array_equal(getattr(c, f).scales, G[f"comp{i}_{f}_scales"])
        np.testing.assert_array_equal(getattr(c, f).zero_points, G[f"comp{i}_{f}_zeros"])
    np.testing.assert_array_equal(lrc.apply_compensation(qm, c), G[f"comp{i}_applied"])


def test_route_tie_break():
    _, sel, _ = lrc.route(np.ones(4), np.zeros((4, 4)), 2, 0)
    assert sel == list(G["route_tie_sel"]) == [0, 1]


@pytest.mark.parametrize("case,k,n", [(0, 2, 1), (1, 2, 1), (2, 8, 2), (3, 8, 2)])
def test_route_golden(case, k, n):
    gate, xs = G[f"route{case}_gate"], G[f"route{case}_x"]
    for t, x in enumerate(xs):
        w, sel, comp = lrc.route(x, gate, k, n)
        assert sel == list(G[f"route{case}_sel"][t])
        assert comp == sel[:n]
        np.testing.assert_array_equal(w, G[f"route{case}_w"][t])


def _toy():
    layers = lrc.gen_model(7, 64, 128, 2, 8, num_shared=1, tail_dofs=(4.0, math.inf),
                           router_skew=1.4)
    return layers


def test_toy_model_generation_bit_exact():
    layers = _toy()
    want = list(G["toy_sha"])
    assert [sha(layers[0].gate), sha(layers[1].experts[3][2]), sha(layers[1].shared[0][0])] == want


def test_toy_compress_and_forward_bit_exact():
    layers = _toy()
    st = lrc.compress(layers, bits=2, group_size=64, hqq_iters=20, rank=16, seed=3)
    for (l, e, p), rec in st.records.items():
        key = f"toy_l{l}_e{e}_{p}"
        np.testing.assert_array_equal(rec.qm.codes, G[key + "_codes"])
        np.testing.assert_array_equal(rec.qm.scales, G[key + "_scales"])
        np.testing.assert_array_equal(rec.qm.zero_points, G[key + "_zeros"])
        for f in ("u", "v"):
            np.testing.assert_array_equal(getattr(rec.comp, f).codes, G[f"{key}_{f}_codes"])
            np.testing.assert_array_equal(getattr(rec.comp, f).scales, G[f"{key}_{f}_scales"])
    for mode in ("reference", "quantized", "compensated"):
        for l in range(2):
            ys = np.array([lrc.forward(x, layers[l].gate, layers[l].experts, 2, 1, mode, st, l,
                                       shared=layers[l].shared) for x in G["toy_x"]])
            np.testing.assert_allclose(ys, G[f"toy_y_{mode}_l{l}"], rtol=1e-12, atol=1e-9)


def test_c1_model_generation_and_routes():
    c1 = json.load(open(os.path.join(HERE, "golden", "c1.json")))
    layers = lrc.gen_model(0, 512, 1024, 1, 8, router_skew=1.4)
    assert sha(layers[0].gate) == c1["model_sha"]["gate"]
    assert sha(layers[0].experts[0][0]) == c1["model_sha"]["e0_w1"]
    assert sha(layers[0].experts[7][2]) == c1["model_sha"]["e7_w2"]
    toks = lrc.gen_tokens(1, 512, 4)
    for x, want in zip(toks, c1["routes"]):
        assert lrc.route(x, layers[0].gate, 2, 1)[1] == want
    # quantizer (HQQ-20) checksums on three C1 projections
    for e, p, w in [(0, "w1", layers[0].experts[0][0]), (3, "w2", layers[0].experts[3][2]),
                    (7, "w3", layers[0].experts[7][1])]:
        qm = lrc.quantize(w, 2, 64, 20)
        rec = c1["records"][f"{e}_{p}"]
        assert sha(qm.codes) == rec["codes"]
        assert sha(qm.scales) == rec["scales"]
        assert sha(qm.zero_points) == rec["zeros"]


def test_c1_reference_forward_consistent():
    """The reference-mode outputs stored in c1.json are reproduced by the oracle."""
    c1 = json.load(open(os.path.join(HERE, "golden", "c1.json")))
    layers = lrc.gen_model(0, 512, 1024, 1, 8, router_skew=1.4)
    toks = lrc.gen_tokens(1, 512, 4)
    for x, want in zip(toks, c1["y_reference"]):
        y = lrc.forward(x, layers[0].gate, layers[0].experts, 2, 1, "reference")
        np.testing.assert_allclose(y, want, rtol=1e-12, atol=1e-9)
