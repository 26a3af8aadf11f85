"""Offline compression pipeline (row a10): rank allocation semantics on CPU, and
the GPU compress_model of the toy model against the reference-compressed
goldens (same model, quant config, ranks and seeds as make_golden.py)."""
import math
import os

import numpy as np
import pytest

from paper_2512_17073_b200 import pipeline

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))


def _prof(kappas):
    return pipeline.KurtosisProfile([pipeline.KurtosisEntry(0, i, "w1", k) for i, k in enumerate(kappas)], 1)


def test_allocate_ranks_greedy():
    # descending kurtosis takes the largest bucket that fits the remaining budget
    a = pipeline.allocate_ranks(_prof([5.0, 3.0, 4.0]), 16, buckets=(0, 16, 32))
    assert a.ranks == {(0, 0, "w1"): 32, (0, 2, "w1"): 16, (0, 1, "w1"): 0}
    assert a.total() == 48
    # ties break by key ascending
    b = pipeline.allocate_ranks(_prof([3.0, 3.0]), 16, buckets=(0, 16, 32))
    assert b.ranks[(0, 0, "w1")] == 32 and b.ranks[(0, 1, "w1")] == 0
    with pytest.raises(pipeline.AllocationError):
        pipeline.allocate_ranks(_prof([1.0]), 8, buckets=(8, 16))
    with pytest.raises(pipeline.AllocationError):
        pipeline.allocate_ranks(_prof([1.0]), -1)
    u = pipeline.uniform_allocation(_prof([1.0, 2.0]), 16)
    assert u.buckets == (0, 16) and set(u.ranks.values()) == {16}


@pytest.mark.gpu
def test_compress_model_toy_vs_reference_goldens():
    from paper_2512_17073_b200 import moe, quant

    m = moe.gen_synthetic_model(seed=7, hidden=64, ffn=128, num_layers=2, num_experts=8, top_k=2,
                                num_shared=1, tail_dofs=(4.0, math.inf), router_skew=1.4)
    prof = pipeline.kurtosis_profile(m)
    # kurtosis: fp64 on the GPU vs numpy
    for e in prof.entries[:6]:
        w = np.asarray(getattr((list(m.layers[e.layer_id].experts) + list(m.layers[e.layer_id].shared_experts))
                               [e.expert_id], e.projection_id), dtype=np.float64)
        d = w - w.mean()
        ref = np.mean(d ** 4) / np.mean(d * d) ** 2
        assert abs(e.kurtosis - ref) <= 1e-9 * ref
    st = pipeline.compress_model(m, quant.QuantConfig(bits=2, group_size=64, hqq_iters=20),
                                 pipeline.uniform_allocation(prof, 16), prof, seed=3)
    agree, total = 0, 0
    for (l, e, p), rec in st.records.items():
        gc = G[f"toy_l{l}_e{e}_{p}_codes"]
        agree += int((np.asarray(rec.qm.codes) == gc).sum())
        total += gc.size
        assert rec.rank == 16 and rec.comp is not None and rec.comp.rank == 16
    assert agree / total >= 0.995, agree / total  # HQQ on the GPU vs numpy order
    xs = G["toy_x"]
    rep = moe.evaluate_fidelity(m, st, xs, moe.ForwardConfig(top_k=2, top_n=1))
    q_ref, c_ref, _ = G["toy_fidelity"]
    assert rep.mean_rel_err["compensated"] < rep.mean_rel_err["quantized"]
    assert abs(rep.mean_rel_err["quantized"] - q_ref) <= 0.05 * q_ref
    assert rep.mean_rel_err["compensated"] <= 1.25 * c_ref  # same ranks, different SVD sketch draws
