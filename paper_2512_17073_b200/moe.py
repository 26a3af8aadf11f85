"""MoE layer API of ref/moe.py, executed on the B200 through liblrc.

Drop-in names and semantics (``/root/reference/pkg/src/moe_lrc/moe.py``):
``route`` (ref :183-193), ``forward`` (ref :217-259), ``expert_forward``
(ref :171-173), ``ForwardConfig`` (ref :91-102), ``evaluate_fidelity``
(ref :382-432), ``build_trace`` / ``RoutingTrace`` / ``routing_stats``
(ref :105-158, :321-356), ``gen_synthetic_model`` / ``gen_tokens``
(ref :262-318, seeded numpy generators -- the path's INPUTS, reproduced
bit-exactly so the same seed gives the same model).

Compute placement:
* routing -> ``lrc_route`` (fp64 gate GEMV + softmax + stable top-k, CUDA)
* mode "quantized"/"compensated" -> ``lrc_layer_forward``: fused router,
  tiled 2-bit dequant-GEMV experts with the low-rank term U.(V.x) applied in
  the expert kernels for each token's top-n experts only; bf16 activations,
  fp16 scale/zero, fp32 accumulation (contract: rel. L2 <= 1e-2 vs fp64).
* mode "reference" -> ``lrc_dense_expert_f64`` (dense fp64 CUDA kernel).
"""

from __future__ import annotations

import json
import math
import weakref
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from .device import LRCMoELayer

MODES = ("reference", "quantized", "compensated")
PROJECTIONS = ("w1", "w2", "w3")


class MoEError(ValueError):
    """Invalid model, config or trace inputs (ref/moe.py:27-28)."""


class MissingArtifactError(KeyError):
    """A selected expert has no quantized weights (ref/moe.py:31-32)."""


@dataclass
class Expert:
    w1: np.ndarray  # (ffn, hidden)
    w3: np.ndarray  # (ffn, hidden)
    w2: np.ndarray  # (hidden, ffn)


@dataclass
class MoELayer:
    gate: np.ndarray  # (hidden, num_experts); logits = gate.T @ x
    experts: list
    shared_experts: list = field(default_factory=list)

    @property
    def num_experts(self) -> int:
        return len(self.experts)

    @property
    def num_shared(self) -> int:
        return len(self.shared_experts)


@dataclass
class MoEModel:
    hidden: int
    ffn: int
    layers: list
    top_k: int
    seed: int = 0
    router_skew: float = 1.0
    tail_dofs: tuple = ()

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    @property
    def num_experts(self) -> int:
        return self.layers[0].num_experts

    @property
    def num_shared(self) -> int:
        return self.layers[0].num_shared

    def iter_projections(self):
        for layer_id, layer in enumerate(self.layers):
            for expert_id, expert in enumerate(list(layer.experts) + list(layer.shared_experts)):
                for proj in PROJECTIONS:
                    yield layer_id, expert_id, proj, getattr(expert, proj)


@dataclass(frozen=True)
class ForwardConfig:
    top_k: int
    top_n: int = 0
    renormalize_topk: bool = False
    compensate_shared: bool = True

    def __post_init__(self) -> None:
        if self.top_k < 0 or self.top_n < 0:
            raise MoEError("top_k and top_n must be >= 0")
        if self.top_n > self.top_k:
            raise MoEError(f"top_n ({self.top_n}) must be <= top_k ({self.top_k})")


@dataclass
class TraceRecord:
    token: int
    layer: int
    scores: np.ndarray
    selected: list
    compensated: list


@dataclass
class RoutingTrace:
    records: list

    def num_tokens(self) -> int:
        return len({r.token for r in self.records})

    def num_layers(self) -> int:
        return len({r.layer for r in self.records})

    def to_jsonl(self, path) -> None:
        with open(path, "w") as f:
            for r in self.records:
                f.write(json.dumps({"token": r.token, "layer": r.layer,
                                    "scores": [float(s) for s in r.scores],
                                    "selected": [int(i) for i in r.selected],
                                    "compensated": [int(i) for i in r.compensated]}) + "\n")

    @classmethod
    def from_jsonl(cls, path) -> "RoutingTrace":
        recs = []
        with open(path) as f:
            for line in f:
                line = line.strip()
                if line:
                    d = json.loads(line)
                    recs.append(TraceRecord(int(d["token"]), int(d["layer"]),
                                            np.asarray(d["scores"], dtype=np.float64),
                                            [int(i) for i in d["selected"]],
                                            [int(i) for i in d["compensated"]]))
        return cls(records=recs)


@dataclass
class RouteResult:
    weights: np.ndarray
    selected: list
    compensated: list


# ---------------------------------------------------------------- helpers --
def _torch():
    return _lib.device_required()


def silu(x):
    """x / (1 + e^-x), evaluated on the device in fp64 (ref/moe.py:161-162)."""
    torch = _torch()
    t = torch.from_numpy(np.asarray(x, dtype=np.float64)).cuda()
    return (t / (1.0 + torch.exp(-t))).cpu().numpy()


def softmax(logits):
    """ref/moe.py:165-168, on the device in fp64."""
    torch = _torch()
    t = torch.from_numpy(np.asarray(logits, dtype=np.float64)).cuda()
    e = torch.exp(t - t.max())
    return (e / e.sum()).cpu().numpy()


class _DenseCache:
    """fp64 copies of full-precision expert weights in HBM (mode="reference")."""

    def __init__(self):
        self._c = {}

    def get(self, w):
        key = id(w)
        hit = self._c.get(key)
        if hit is not None and hit[0] is w:
            return hit[1]
        t = _torch().from_numpy(np.ascontiguousarray(w, dtype=np.float64)).cuda()
        self._c[key] = (w, t)
        return t


_dense = _DenseCache()


def _dense_expert_accum(expert, x_dev, mix_dev, y_dev):
    """y += mix * w2 @ (silu(w1 @ x) * (w3 @ x)) for all B rows of x_dev (fp64 CUDA)."""
    w1, w3, w2 = (_dense.get(expert.w1), _dense.get(expert.w3), _dense.get(expert.w2))
    ffn, hidden = w1.shape
    _lib.check(_lib.lib().lrc_dense_expert_f64(
        _lib.ptr(w1), _lib.ptr(w3), _lib.ptr(w2), hidden, ffn, _lib.ptr(x_dev),
        _lib.ptr(mix_dev), int(x_dev.shape[0]), _lib.ptr(y_dev), _lib.stream_ptr()))


def expert_forward(expert_w1, expert_w3, expert_w2, x):
    """w2 @ (silu(w1 @ x) * (w3 @ x)) in fp64 on the device (ref/moe.py:171-173)."""
    torch = _torch()
    x = np.asarray(x, dtype=np.float64)
    xd = torch.from_numpy(np.ascontiguousarray(x.reshape(1, -1))).cuda()
    y = torch.zeros((1, np.asarray(expert_w2).shape[0]), dtype=torch.float64, device="cuda")
    _dense_expert_accum(Expert(expert_w1, expert_w3, expert_w2), xd, None, y)
    return y.cpu().numpy().reshape(-1)


# ---------------------------------------------------------------- routing --
class _GateCache:
    def __init__(self):
        self._c = {}

    def get(self, gate):
        key = id(gate)
        hit = self._c.get(key)
        if hit is not None and hit[0] is gate:
            return hit[1]
        t = _torch().from_numpy(np.ascontiguousarray(np.asarray(gate, np.float64).T)).cuda()
        self._c[key] = (gate, t)
        return t


_gates = _GateCache()


def _route_batch(xs_dev, gate, top_k, top_n, renorm):
    """Device routing for (B, d) fp64 tokens -> probs (B,E) f64, idx (B,k), mix (B,k)."""
    torch = _torch()
    gt = _gates.get(gate)
    E, d = gt.shape
    B = int(xs_dev.shape[0])
    probs = torch.empty((B, E), dtype=torch.float64, device="cuda")
    kk = max(top_k, 1)
    idx = torch.empty((B, kk), dtype=torch.int32, device="cuda")
    mix = torch.empty((B, kk), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().lrc_route(_lib.ptr(gt), _lib.ptr(xs_dev), _lib.DTYPE_F64, B, d, E, top_k,
                                    top_n, int(bool(renorm)), _lib.ptr(probs), _lib.ptr(idx),
                                    _lib.ptr(mix), _lib.stream_ptr()), {_lib.LRC_ERR_INVALID: MoEError})
    return probs, idx, mix


def route(x: np.ndarray, layer: MoELayer, cfg: ForwardConfig) -> RouteResult:
    """Softmax routing with lower-index tie-breaking (ref/moe.py:183-193)."""
    if x.shape != (layer.gate.shape[0],):
        raise MoEError(f"token dim {x.shape} does not match gate {layer.gate.shape}")
    if cfg.top_k > layer.num_experts:
        raise MoEError(f"top_k {cfg.top_k} exceeds {layer.num_experts} experts")
    torch = _torch()
    xd = torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.float64).reshape(1, -1))).cuda()
    probs, idx, _ = _route_batch(xd, layer.gate, cfg.top_k, cfg.top_n, False)
    sel = [int(i) for i in idx.cpu().numpy()[0][: cfg.top_k]]
    return RouteResult(weights=probs.cpu().numpy()[0], selected=sel, compensated=sel[: cfg.top_n])


# ------------------------------------------------------------ device layers --
_layer_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_layer_cache_strong: dict = {}


def device_layer(artifacts, layer_id: int, layer: MoELayer, max_tokens: int = 64,
                 top_k: int = 2) -> LRCMoELayer:
    """Cached HBM copy of one layer's artifacts (uploaded once per store/layer)."""
    key = (layer_id, id(layer.gate), layer.num_experts, layer.num_shared)
    try:
        per = _layer_cache.setdefault(artifacts, {})
    except TypeError:  # not weak-referenceable
        per = _layer_cache_strong.setdefault(id(artifacts), {})
    dl = per.get(key)
    if dl is None:
        hidden = layer.gate.shape[0]
        probe = None
        for eid in range(layer.num_experts + layer.num_shared):
            try:
                probe = artifacts.get(layer_id, eid, "w1")
            except (KeyError, AttributeError):
                continue
            if probe is not None:
                break
        if probe is None:
            raise MissingArtifactError(f"no artifact for layer {layer_id}")
        ffn = probe.qm.rows
        dl = LRCMoELayer.from_artifacts(layer.gate, artifacts, layer_id, layer.num_experts,
                                        layer.num_shared, hidden, ffn, max_tokens=max_tokens,
                                        top_k=max(top_k, 1))
        per[key] = dl
    return dl


def _check_missing(dl: LRCMoELayer, idx_host, top_k, layer_id, num_experts, num_shared):
    if not dl.missing:
        return
    for row in np.atleast_2d(idx_host):
        for e in row[:top_k]:
            if int(e) in dl.missing:
                raise MissingArtifactError(
                    f"no artifact for layer {layer_id}, expert {int(e)}, w1")
    for j in range(num_shared):
        if num_experts + j in dl.missing:
            raise MissingArtifactError(f"no artifact for layer {layer_id}, expert {num_experts + j}")


def _forward_batch(xs: np.ndarray, layer: MoELayer, cfg: ForwardConfig, mode: str, artifacts,
                   layer_id: int) -> np.ndarray:
    torch = _torch()
    B = xs.shape[0]
    if mode == "reference":
        xd = torch.from_numpy(np.ascontiguousarray(xs, dtype=np.float64)).cuda()
        probs, idx, mix = _route_batch(xd, layer.gate, cfg.top_k, cfg.top_n,
                                       cfg.renormalize_topk)
        y = torch.zeros((B, layer.gate.shape[0]), dtype=torch.float64, device="cuda")
        idx_h = idx.cpu().numpy()
        sel = idx[:, : cfg.top_k].long()
        mix_d = torch.gather(probs, 1, sel)  # fp64 mixing weights (ref/moe.py:234)
        if cfg.renormalize_topk:
            tot = mix_d.sum(dim=1, keepdim=True)
            mix_d = torch.where(tot > 0, mix_d / tot, mix_d)
        for e in sorted({int(v) for v in idx_h[:, : cfg.top_k].ravel()}):
            m = ((sel == e).double() * mix_d).sum(dim=1).contiguous()
            _dense_expert_accum(layer.experts[e], xd, m, y)
        for s in layer.shared_experts:
            _dense_expert_accum(s, xd, None, y)
        return y.cpu().numpy()
    # Routing runs on the fp64 tokens, exactly as the reference's forward
    # (ref/moe.py:221-233 routes x itself): lrc_route in fp64, then the expert
    # kernels take that selection as explicit (token, expert) pairs
    # (lrc_layer_forward_pairs).  Only the expert compute sees the bf16 tokens.
    P = cfg.top_k + layer.num_shared
    dl = device_layer(artifacts, layer_id, layer, max_tokens=max(64, B * P), top_k=cfg.top_k)
    xd = torch.from_numpy(np.ascontiguousarray(xs, dtype=np.float64)).cuda()
    _, idx, mix = _route_batch(xd, layer.gate, cfg.top_k, 0, cfg.renormalize_topk)
    if dl.missing:
        _check_missing(dl, idx.cpu().numpy(), cfg.top_k, layer_id, layer.num_experts,
                       layer.num_shared)
    xb = xd.to(torch.bfloat16)
    top_n = cfg.top_n if mode == "compensated" else 0
    comp_shared = cfg.compensate_shared and mode == "compensated"
    k, S = cfg.top_k, layer.num_shared
    ex = torch.empty((B, P), dtype=torch.int32, device="cuda")
    wt = torch.ones((B, P), dtype=torch.float32, device="cuda")
    cp = torch.zeros((B, P), dtype=torch.uint8, device="cuda")
    if k:
        ex[:, :k] = idx[:, :k]
        wt[:, :k] = mix[:, :k]
        cp[:, :min(top_n, k)] = 1
    if S:
        ex[:, k:] = torch.arange(layer.num_experts, layer.num_experts + S, dtype=torch.int32, device="cuda")
        cp[:, k:] = int(comp_shared)
    rows = xb.repeat_interleave(P, dim=0)
    y = dl.forward_pairs(rows, ex.reshape(-1), wt.reshape(-1), cp.reshape(-1), validate=False)
    return y.reshape(B, P, -1).sum(1).double().cpu().numpy()


def forward(x: np.ndarray, layer: MoELayer, cfg: ForwardConfig, mode: str = "reference",
            artifacts=None, layer_id: int = 0) -> np.ndarray:
    """One MoE layer forward for a single token (ref/moe.py:217-259)."""
    if mode not in MODES:
        raise MoEError(f"unknown mode {mode!r}; expected one of {MODES}")
    if mode != "reference" and artifacts is None:
        raise MissingArtifactError(f"mode {mode!r} requires artifacts")
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (layer.gate.shape[0],):
        raise MoEError(f"token dim {x.shape} does not match gate {layer.gate.shape}")
    if cfg.top_k > layer.num_experts:
        raise MoEError(f"top_k {cfg.top_k} exceeds {layer.num_experts} experts")
    return _forward_batch(x.reshape(1, -1), layer, cfg, mode, artifacts, layer_id)[0]


def forward_batch(xs: np.ndarray, layer: MoELayer, cfg: ForwardConfig, mode: str = "compensated",
                  artifacts=None, layer_id: int = 0) -> np.ndarray:
    """Batched variant of ``forward`` over (B, hidden) tokens (one device pass)."""
    if mode not in MODES:
        raise MoEError(f"unknown mode {mode!r}; expected one of {MODES}")
    if mode != "reference" and artifacts is None:
        raise MissingArtifactError(f"mode {mode!r} requires artifacts")
    xs = np.asarray(xs, dtype=np.float64)
    if xs.ndim != 2 or xs.shape[1] != layer.gate.shape[0]:
        raise MoEError(f"tokens {xs.shape} do not match gate {layer.gate.shape}")
    if cfg.top_k > layer.num_experts:
        raise MoEError(f"top_k {cfg.top_k} exceeds {layer.num_experts} experts")
    return _forward_batch(xs, layer, cfg, mode, artifacts, layer_id)


# ------------------------------------------------------- synthetic inputs --
def _draw_tail(rng: np.random.Generator, dof: float, size) -> np.ndarray:
    if math.isinf(dof):
        return rng.standard_normal(size)
    return rng.standard_t(dof, size) / math.sqrt(dof / (dof - 2.0))


def gen_synthetic_model(seed: int, hidden: int, ffn: int, num_layers: int, num_experts: int,
                        top_k: int = 2, num_shared: int = 0, tail_dofs=None,
                        router_skew: float = 1.0) -> MoEModel:
    """Deterministic synthetic model, same draw order as ref/moe.py:269-314."""
    if hidden <= 0 or ffn <= 0 or num_layers <= 0 or num_experts <= 0:
        raise MoEError("hidden, ffn, num_layers and num_experts must be positive")
    if not 0 <= top_k <= num_experts:
        raise MoEError(f"top_k {top_k} outside [0, {num_experts}]")
    if num_shared < 0:
        raise MoEError("num_shared must be >= 0")
    if router_skew < 0:
        raise MoEError("router_skew must be >= 0")
    dofs = tuple(float(d) for d in (tail_dofs or (math.inf,)))
    for d in dofs:
        if not d > 2.0:
            raise MoEError(f"tail dof must be > 2 (got {d}); variance is undefined below")
    rng = np.random.default_rng(seed)
    layers = []
    for _ in range(num_layers):
        gate = rng.standard_normal((hidden, num_experts))
        gate = gate / np.linalg.norm(gate, axis=0, keepdims=True) * router_skew
        experts = []
        for e in range(num_experts + num_shared):
            dof = dofs[e % len(dofs)]
            experts.append(Expert(w1=_draw_tail(rng, dof, (ffn, hidden)),
                                  w3=_draw_tail(rng, dof, (ffn, hidden)),
                                  w2=_draw_tail(rng, dof, (hidden, ffn))))
        layers.append(MoELayer(gate=gate, experts=experts[:num_experts],
                               shared_experts=experts[num_experts:]))
    return MoEModel(hidden=hidden, ffn=ffn, layers=layers, top_k=top_k, seed=seed,
                    router_skew=router_skew, tail_dofs=dofs)


def gen_tokens(seed: int, hidden: int, count: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal((count, hidden))


# ------------------------------------------------------ traces and stats --
def build_trace(model: MoEModel, cfg: ForwardConfig, num_tokens: int, seed: int) -> RoutingTrace:
    """Route num_tokens tokens through every layer, batched on the device (ref/moe.py:321-333)."""
    torch = _torch()
    tokens = gen_tokens(seed, model.hidden, num_tokens)
    xd = torch.from_numpy(np.ascontiguousarray(tokens)).cuda()
    per_layer = []
    for layer in model.layers:
        if cfg.top_k > layer.num_experts:
            raise MoEError(f"top_k {cfg.top_k} exceeds {layer.num_experts} experts")
        probs, idx, _ = _route_batch(xd, layer.gate, cfg.top_k, cfg.top_n, False)
        per_layer.append((probs.cpu().numpy(), idx.cpu().numpy()))
    recs = []
    for t in range(num_tokens):
        for lid, (probs, idx) in enumerate(per_layer):
            sel = [int(i) for i in idx[t][: cfg.top_k]]
            recs.append(TraceRecord(t, lid, probs[t], sel, sel[: cfg.top_n]))
    return RoutingTrace(records=recs)


@dataclass
class RoutingStatsReport:
    aggregate: np.ndarray
    per_layer: dict
    num_tokens: int


def routing_stats(trace: RoutingTrace) -> RoutingStatsReport:
    """Mean i-th largest routing score (host statistics over a trace; ref/moe.py:345-356)."""
    if not trace.records:
        raise MoEError("empty trace")
    by_layer: dict = {}
    for r in trace.records:
        by_layer.setdefault(r.layer, []).append(np.sort(r.scores)[::-1])
    per_layer = {lid: np.mean(np.stack(rows), axis=0) for lid, rows in sorted(by_layer.items())}
    aggregate = np.mean(np.stack([np.sort(r.scores)[::-1] for r in trace.records]), axis=0)
    return RoutingStatsReport(aggregate=aggregate, per_layer=per_layer,
                              num_tokens=trace.num_tokens())


@dataclass
class FidelityReport:
    mean_rel_err: dict
    win_rate: float
    per_token: dict
    num_tokens: int


def evaluate_fidelity(model: MoEModel, artifacts, tokens: np.ndarray,
                      cfg: ForwardConfig) -> FidelityReport:
    """Relative output error of quantized / compensated vs reference, all tokens
    of a layer in one device pass per mode (ref/moe.py:382-432)."""
    tokens = np.asarray(tokens, dtype=np.float64)
    if tokens.size == 0:
        raise MoEError("tokens must be non-empty")
    errs = {"quantized": [], "compensated": []}
    for lid, layer in enumerate(model.layers):
        y = {m: _forward_batch(tokens, layer, cfg, m, None if m == "reference" else artifacts, lid)
             for m in MODES}
        ref_norm = np.linalg.norm(y["reference"], axis=1)
        for m in ("quantized", "compensated"):
            err = np.linalg.norm(y[m] - y["reference"], axis=1)
            errs[m].append(np.where(ref_norm > 0, err / np.where(ref_norm > 0, ref_norm, 1), 0.0))
    pt = {m: np.mean(np.stack(v), axis=0) for m, v in errs.items()}
    wins = float(np.mean(pt["compensated"] < pt["quantized"]))
    mean_rel = {m: float(v.mean()) for m, v in pt.items()}
    mean_rel["reference"] = 0.0
    return FidelityReport(mean_rel_err=mean_rel, win_rate=wins, per_token=pt,
                          num_tokens=len(tokens))
