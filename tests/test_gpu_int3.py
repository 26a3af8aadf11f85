"""GPU parity of the code-width / batch / expert-count corners (SURVEY 8(c), C2 + C5):
INT3 experts at decode batches 1, 8 and 64 (tensor-core decode engine for
B <= 8, prefill engine above), the tensor-core decode engine on INT2, INT2 at
B = 64, and a 128-expert top-8 layer with top-2 restore and two shared
experts.  EVERY token of every batch is checked against the fp64 oracle
(oracle/lrc.py) fed the same bf16 tokens and fp16 metadata:
max relative L2 <= 1e-2, routing indices bit-exact.
"""

import numpy as np
import pytest

from oracle import bridge, lrc

pytestmark = pytest.mark.gpu

TOL_Y = 1e-2


@pytest.fixture(scope="module")
def torch():
    import torch as t

    import paper_2512_17073_b200._lib as L

    L.load()
    return t


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def oracle_batch(xs, gate, store, k, n, n_shared=0, comp_shared=True):
    """lrc.forward for every token, resolving each (expert, compensated) pair's
    dense weights once (ref/moe.py:217-259 per token)."""
    E = gate.shape[1]
    routes = [lrc.route(x, gate, k, n) for x in xs]
    jobs = {}
    for t, (wts, sel, comp) in enumerate(routes):
        for e in sel:
            jobs.setdefault((int(e), int(e) in set(comp)), []).append((t, float(wts[e])))
        for j in range(n_shared):
            jobs.setdefault((E + j, bool(comp_shared)), []).append((t, 1.0))
    y = np.zeros((len(xs), gate.shape[0]))
    for (e, flag), lst in jobs.items():
        w1, w3, w2 = lrc.resolve(store, 0, e, flag)
        for t, wgt in lst:
            y[t] += wgt * lrc.expert_forward(w1, w3, w2, xs[t])
    return y, routes


def check_layer(torch, sl, B, k, n, seed, n_shared=0, **fwd):
    xs = lrc.to_bf16(np.random.default_rng(seed).standard_normal((B, sl.hidden)))
    y, idx, _ = sl.layer.forward(torch.from_numpy(xs).cuda().to(torch.bfloat16), top_k=k, top_n=n, **fwd)
    y, idx = y.double().cpu().numpy(), idx.cpu().numpy()
    st = bridge.synth_store(sl, sorted({int(e) for e in idx.ravel()} | set(range(sl.E, sl.E + n_shared))))
    yo, routes = oracle_batch(xs, sl.gate, st, k, n, n_shared)
    worst = 0.0
    for t in range(B):
        assert list(routes[t][1]) == list(idx[t]), (t, routes[t][1], idx[t])
        worst = max(worst, rel_l2(y[t], yo[t]))
    assert worst <= TOL_Y, worst
    return worst


@pytest.fixture(scope="module")
def int3_layer(torch):
    from paper_2512_17073_b200.synth import SynthLayer

    return SynthLayer(4096, 14336, 8, top_k=2, bits=3, rank=32, seed=31, max_tokens=64, tiles=False)


@pytest.mark.parametrize("B", [1, 8, 64])
def test_int3_mixtral_layer_all_tokens(torch, int3_layer, B):
    """C2 at INT3 + rank-32 top-1: B <= 8 runs the tensor-core decode engine, B = 64 the prefill engine."""
    L = int3_layer.layer
    assert L.tcd_eligible and L.prefill_eligible
    check_layer(torch, int3_layer, B, 2, 1, seed=300 + B)


def test_int3_generic_path_all_tokens(torch, int3_layer):
    """The CUDA-core generic path (group-vectorised decode) on INT3 codes."""
    check_layer(torch, int3_layer, 5, 2, 1, seed=77, generic=True)


@pytest.fixture(scope="module")
def int2_layer(torch):
    from paper_2512_17073_b200.synth import SynthLayer

    return SynthLayer(4096, 14336, 8, top_k=2, bits=2, rank=32, seed=41, max_tokens=64)


def test_int2_b64_all_tokens(torch, int2_layer):
    check_layer(torch, int2_layer, 64, 2, 1, seed=64)


@pytest.mark.parametrize("B", [1, 8])
def test_tcd_int2_all_tokens(torch, int2_layer, B):
    """The tensor-core decode engine forced on an INT2 layer (default: tiled kernels)."""
    L = int2_layer.layer
    assert L.tcd_eligible
    L.set_tcd_max(8)
    try:
        check_layer(torch, int2_layer, B, 2, 1, seed=500 + B)
        check_layer(torch, int2_layer, B, 2, 0, seed=600 + B)
    finally:
        L.set_tcd_max(-1)


def test_e128_top8_two_shared_all_tokens(torch):
    """C5-like routing on one GPU: 128 experts top-8, top-2 restore, 2 shared
    experts (always on, compensated), router skew 0.8."""
    from paper_2512_17073_b200.synth import SynthLayer

    sl = SynthLayer(2048, 1408, 128, top_k=8, num_shared=2, bits=2, rank=32, seed=5, router_skew=0.8,
                    max_tokens=32)
    for B in (1, 16):
        check_layer(torch, sl, B, 8, 2, seed=900 + B, n_shared=2)


@pytest.mark.parametrize("B", [16, 64])
def test_int2_small_batch_prefill_all_tokens(torch, int2_layer, B):
    """The tensor-core grouped GEMM at batch sizes below the default prefill
    threshold (MMA N = 64 tiles), every token vs the oracle."""
    L = int2_layer.layer
    assert L.prefill_eligible
    L.set_prefill_min(1)
    try:
        check_layer(torch, int2_layer, B, 2, 1, seed=700 + B)
    finally:
        L.set_prefill_min(128)
