"""Offline compression pipeline on the GPU.

Mirrors ref/ranks.py (kurtosis profile, greedy bucketed rank allocation) and
ref/pipeline.py:114-173 (``uniform_allocation``, ``compress_model``): every
projection is quantized (``quant.quantize``: fused min-max + HQQ kernel) and,
at its allocated rank clamped to min(m, n), gets a compensator
(``lowrank.build_compensator``: residual + randomized SVD + INT3 factor
quantization on the GPU).  Per-record seeds derive from the global seed as in
the reference (SeedSequence([seed, layer, expert, projection index])), so the
result does not depend on the processing order.  The returned store follows
the reference's artifact protocol (``get(layer, expert, projection)`` ->
record with ``.qm`` / ``.comp``) and feeds ``moe.forward`` / ``device_layer``
directly.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .lowrank import build_compensator
from .quant import QuantConfig, quantize

PROJECTIONS = ("w1", "w3", "w2")
DEFAULT_BUCKETS = (0, 16, 32, 128, 256, 512, 1024)  # ref/ranks.py:18


class AllocationError(ValueError):
    """Invalid allocation inputs (ref/ranks.py:23-24)."""


def kurtosis(w) -> float:
    """Population kurtosis over all elements (no excess-3 subtraction), fp64 on
    the GPU; constant matrices return 0.0 (ref/ranks.py:27-41)."""
    torch = _lib.device_required()
    t = torch.as_tensor(np.asarray(w, dtype=np.float64)).cuda().reshape(-1)
    if t.numel() == 0:
        raise AllocationError("kurtosis of an empty matrix")
    dev = t - t.mean()
    var = (dev * dev).mean()
    if float(var) == 0.0:
        return 0.0
    return float((dev.pow(4)).mean() / (var * var))


@dataclass(frozen=True)
class KurtosisEntry:
    layer_id: int
    expert_id: int
    projection_id: str
    kurtosis: float


@dataclass
class KurtosisProfile:
    entries: list
    d: int = 0

    def __len__(self) -> int:
        return len(self.entries)


@dataclass
class RankAllocation:
    buckets: tuple
    avg_budget: int
    ranks: dict = field(default_factory=dict)

    def total(self) -> int:
        return sum(self.ranks.values())

    def rank_of(self, layer_id: int, expert_id: int, projection_id: str) -> int:
        return self.ranks[(layer_id, expert_id, projection_id)]


def iter_projections(model):
    """(layer, expert, projection, matrix); shared experts get ids >= num_experts."""
    for layer_id, layer in enumerate(model.layers):
        for expert_id, expert in enumerate(list(layer.experts) + list(layer.shared_experts)):
            for proj in PROJECTIONS:
                yield layer_id, expert_id, proj, getattr(expert, proj)


def kurtosis_profile(model) -> KurtosisProfile:
    entries, d = [], 0
    for layer_id, expert_id, proj, w in iter_projections(model):
        entries.append(KurtosisEntry(layer_id, expert_id, proj, kurtosis(w)))
        d = np.asarray(w).size
    return KurtosisProfile(entries, d)


def allocate_ranks(profile: KurtosisProfile, avg_budget: int, buckets=DEFAULT_BUCKETS,
                   per_layer: bool = False) -> RankAllocation:
    """Greedy bucketed allocation under a total budget of N * avg_budget:
    entries in descending kurtosis (ties by key) take the largest bucket that
    keeps the running total within budget (ref/ranks.py:106-152)."""
    if avg_budget < 0:
        raise AllocationError(f"avg_budget must be >= 0, got {avg_budget}")
    bucket_set = tuple(sorted(set(int(b) for b in buckets)))
    if not bucket_set or bucket_set[0] != 0:
        raise AllocationError("buckets must contain 0")
    if any(b < 0 for b in bucket_set):
        raise AllocationError("buckets must be non-negative")
    keys = [(e.layer_id, e.expert_id, e.projection_id) for e in profile.entries]
    if len(set(keys)) != len(keys):
        raise AllocationError("duplicate profile entry")
    alloc = RankAllocation(bucket_set, avg_budget)

    def fill(entries):
        remaining = len(entries) * avg_budget
        for e in sorted(entries, key=lambda e: (-e.kurtosis, e.layer_id, e.expert_id, e.projection_id)):
            r = max(b for b in bucket_set if b <= remaining)
            alloc.ranks[(e.layer_id, e.expert_id, e.projection_id)] = r
            remaining -= r

    if per_layer:
        for layer_id in sorted({e.layer_id for e in profile.entries}):
            fill([e for e in profile.entries if e.layer_id == layer_id])
    else:
        fill(profile.entries)
    return alloc


def uniform_allocation(model_or_profile, rank: int) -> RankAllocation:
    """Every projection at the same rank (ref/pipeline.py:114-122)."""
    prof = model_or_profile if isinstance(model_or_profile, KurtosisProfile) else kurtosis_profile(model_or_profile)
    return RankAllocation(tuple(sorted({0, rank})), rank,
                          {(e.layer_id, e.expert_id, e.projection_id): rank for e in prof.entries})


@dataclass
class ProjRecord:
    layer: int
    expert: int
    projection: str
    qm: object
    comp: object
    kurtosis: float
    rank: int


class CompressedStore:
    """Records keyed (layer, expert, projection); the artifact protocol."""

    def __init__(self, header: dict):
        self.header = header
        self.records = {}

    def add(self, rec: ProjRecord) -> None:
        key = (rec.layer, rec.expert, rec.projection)
        if key in self.records:
            raise AllocationError(f"duplicate record {key}")
        self.records[key] = rec

    def get(self, layer: int, expert: int, projection: str) -> ProjRecord:
        return self.records[(layer, expert, projection)]


def compress_model(model, qcfg: QuantConfig, allocation: RankAllocation, profile: KurtosisProfile,
                   factor_bits: int = 3, seed: int = 0, quantize_factors: bool = True) -> CompressedStore:
    """Quantize every projection and attach its allocated-rank compensator
    (ref/pipeline.py:125-173), all on the GPU."""
    kappa = {(e.layer_id, e.expert_id, e.projection_id): e.kurtosis for e in profile.entries}
    store = CompressedStore({"hidden": model.hidden, "ffn": model.ffn, "num_layers": model.num_layers,
                             "num_experts": model.num_experts, "num_shared": model.num_shared,
                             "top_k": model.top_k, "quant": qcfg, "buckets": allocation.buckets,
                             "avg_budget": allocation.avg_budget, "seed": seed})
    for layer_id, expert_id, proj, w in iter_projections(model):
        key = (layer_id, expert_id, proj)
        qm = quantize(w, qcfg)
        rank = min(allocation.ranks[key], min(np.asarray(w).shape))
        comp = None
        if rank > 0:
            rec_seed = int(np.random.SeedSequence([seed, layer_id, expert_id, PROJECTIONS.index(proj)])
                           .generate_state(1)[0])
            comp = build_compensator(w, qm, rank, factor_bits=factor_bits, projection_id=proj, seed=rec_seed,
                                     quantize_factors=quantize_factors)
        store.add(ProjRecord(layer_id, expert_id, proj, qm, comp, kappa[key], rank))
    expected = model.num_layers * (model.num_experts + model.num_shared) * len(PROJECTIONS)
    if len(store.records) != expected:
        raise AllocationError(f"expected {expected} projection records, found {len(store.records)}")
    return store


__all__ = ["AllocationError", "KurtosisEntry", "KurtosisProfile", "RankAllocation", "ProjRecord",
           "CompressedStore", "kurtosis", "kurtosis_profile", "allocate_ranks", "uniform_allocation",
           "compress_model", "iter_projections", "DEFAULT_BUCKETS"]
