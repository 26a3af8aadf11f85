"""Golden reports of the REAL reference simulator (build container only).

    python tests/golden/make_sim_golden.py        # needs /root/reference

Routes 12 tokens through a small 4-layer, 8-expert synthetic model with the
reference's own build_trace, then runs the reference's simulate() for a grid
of plans x systems at Mixtral-8x7B expert shapes (4 layers).  Writes
tests/golden/sim_trace.jsonl and tests/golden/sim_reports.json; the CPU test
tests/test_simulate.py replays the trace through paper_2512_17073_b200.simulate.
"""

from __future__ import annotations

import json
import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def plans_and_systems(sim):
    plans = [
        dict(name="fp16", expert_bits=16),
        dict(name="int2-n1-r32", expert_bits=2, top_n=1, rank=32),
        dict(name="int3-n2-r16", expert_bits=3, top_n=2, rank=16, factor_bits=4),
        dict(name="int2-lru", expert_bits=2, top_n=1, rank=32, cache_policy="lru", cache_budget_bytes=5 * 44040192),
    ]
    systems = [
        dict(name="gpu-only", pcie_bw=25e9, gpu_flops=989.4e12, gpu_hbm_bw=3.35e12, gpu_mem_capacity=80e9,
             ndp_enabled=False, overlap=False),
        dict(name="gpu-only-overlap", pcie_bw=25e9, gpu_flops=989.4e12, gpu_hbm_bw=3.35e12, gpu_mem_capacity=80e9,
             ndp_enabled=False, overlap=True),
        dict(name="b200-like", pcie_bw=55.3e9, gpu_flops=1644e12, gpu_hbm_bw=6.55e12, gpu_mem_capacity=180e9,
             ndp_enabled=False, overlap=False),
        dict(name="gpu-ndp", pcie_bw=25e9, gpu_flops=989.4e12, gpu_hbm_bw=3.35e12, gpu_mem_capacity=80e9,
             ndp_enabled=True, ndp_bw=512e9, ndp_capacity=512e9, ndp_flops=16e12, overlap=True),
    ]
    return plans, systems


def main():
    sys.path.insert(0, REF)
    from moe_lrc import moe, simulate as sim

    model = moe.gen_synthetic_model(seed=3, hidden=64, ffn=128, num_layers=4, num_experts=8, top_k=2,
                                    router_skew=1.4)
    trace = moe.build_trace(model, moe.ForwardConfig(top_k=2, top_n=2), num_tokens=12, seed=5)
    trace.to_jsonl(os.path.join(HERE, "sim_trace.jsonl"))
    dims = sim.ModelDims(hidden=4096, ffn=14336, num_layers=4, num_experts=8, top_k=2, num_shared=0)
    plans, systems = plans_and_systems(sim)
    out = []
    for s in systems:
        for p in plans:
            for n in (None, 5):
                for pre in (True, False):
                    r = sim.simulate(trace, sim.TransferPlan(**p), sim.SystemConfig(**s), dims, input_len=64,
                                     output_len=n, include_prefill=pre)
                    out.append({"plan": p, "system": s, "output_len": n, "include_prefill": pre, "report": r.as_row()})
    with open(os.path.join(HERE, "sim_reports.json"), "w") as f:
        json.dump({"dims": dict(hidden=4096, ffn=14336, num_layers=4, num_experts=8, top_k=2, num_shared=0),
                   "input_len": 64, "cells": out}, f, indent=0)
    print(len(out), "cells")


if __name__ == "__main__":
    main()
