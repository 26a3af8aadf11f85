"""Offload simulator against the REAL reference's simulate():
the reference's own routing trace (tests/golden/sim_trace.jsonl) replayed for
a grid of plans x systems (fp16 / INT2 / INT3, LRU cache, overlap, NDP) must
reproduce the reference's reports (tests/golden/sim_reports.json, made by
tests/golden/make_sim_golden.py).  Host-only: no GPU, no /root/reference."""
import json
import os

import pytest

from paper_2512_17073_b200 import simulate as sim
from paper_2512_17073_b200.moe import RoutingTrace

HERE = os.path.dirname(os.path.abspath(__file__))
G = json.load(open(os.path.join(HERE, "golden", "sim_reports.json")))
TRACE = RoutingTrace.from_jsonl(os.path.join(HERE, "golden", "sim_trace.jsonl"))


@pytest.mark.parametrize("i", range(len(G["cells"])))
def test_simulate_matches_reference(i):
    c = G["cells"][i]
    dims = sim.ModelDims(**G["dims"])
    r = sim.simulate(TRACE, sim.TransferPlan(**c["plan"]), sim.SystemConfig(**c["system"]), dims,
                     input_len=G["input_len"], output_len=c["output_len"], include_prefill=c["include_prefill"])
    got, want = r.as_row(), c["report"]
    assert got.keys() == want.keys()
    for k, v in want.items():
        if isinstance(v, float):
            assert got[k] == pytest.approx(v, rel=1e-12, abs=0.0), (k, got[k], v)
        else:
            assert got[k] == v, (k, got[k], v)


def test_simulate_errors():
    dims = sim.ModelDims(4096, 14336, 4, 8, 2)
    with pytest.raises(sim.SimulationError):
        sim.simulate(TRACE, sim.TransferPlan(expert_bits=5), sim.SYSTEM_PRESETS["gpu-only"], dims)
    with pytest.raises(sim.SimulationError):  # trace covers 4 layers, dims expect 8
        sim.simulate(TRACE, sim.TransferPlan(), sim.SYSTEM_PRESETS["gpu-only"], sim.ModelDims(4096, 14336, 8, 8, 2))
    with pytest.raises(sim.SimulationError):  # budget below one expert
        sim.simulate(TRACE, sim.TransferPlan(expert_bits=2, cache_policy="lru", cache_budget_bytes=10),
                     sim.SYSTEM_PRESETS["gpu-only"], dims)
    with pytest.raises(sim.SimulationError):
        sim.simulate(TRACE, sim.TransferPlan(), sim.SYSTEM_PRESETS["gpu-only"], dims, output_len=100)


def test_b200_system():
    s = sim.b200_system(55.3, 6546.9, 1644.0, overlap=True)
    assert s.pcie_bw == 55.3e9 and s.overlap and s.gpu_mem_capacity == 180e9
