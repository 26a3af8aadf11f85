"""numpy restatement of the reference CPU path (TEST INFRASTRUCTURE ONLY).

Reference = ``moe-lrc`` 0.1.0, abbreviated ``ref/`` = ``pkg/src/moe_lrc/``.
The arithmetic below repeats the reference's numpy operation order exactly
(same fp64 ops, same LAPACK calls, same RNG draws) so that integer outputs
(codes, packed bytes, routing indices) are bit-identical and float outputs
agree to the last few ulps.  The restatement is pinned by
``tests/test_oracle_golden.py`` against fixtures generated from the real
reference (``tests/golden/make_golden.py``).

Layout of this module: one flat namespace of small functions plus three
plain containers (``QM``, ``Comp``, ``Rec``) that duck-type the reference's
``QuantizedMatrix`` / ``Compensator`` / ``ProjRecord`` fields used on the
path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

PROJ_NAMES = ("w1", "w2", "w3")  # ref/ranks.py:20
HQQ_BETA0, HQQ_KAPPA = 10.0, 1.01  # ref/quant.py:22-23
SVD_OVERSAMPLE, SVD_MIN_PASSES, SVD_MAX_PASSES, SVD_STALL = 8, 8, 600, 1e-14  # ref/lowrank.py:19-24


# --------------------------------------------------------------------------
# containers
# --------------------------------------------------------------------------
@dataclass
class QM:
    """Fields of ref/quant.py:59-102 QuantizedMatrix."""

    rows: int
    cols: int
    bits: int
    group_size: int
    codes: np.ndarray        # uint8 (rows, cols)
    scales: np.ndarray       # f64 (rows, ceil(cols/gs))
    zero_points: np.ndarray  # f64 (rows, ceil(cols/gs))

    @property
    def groups_per_row(self) -> int:
        return -(-self.cols // self.group_size)


@dataclass
class Comp:
    """Fields of ref/lowrank.py:33-49 Compensator (u/v: QM or raw ndarray)."""

    rank: int
    u: object
    v: object
    projection_id: str = ""
    factor_bits: int = 3


@dataclass
class Rec:
    """The two attributes ref/moe.py:210-213 reads from an artifact record."""

    qm: QM
    comp: Comp | None = None


class Store:
    """Duck-typed artifact store: ``get(layer, expert, proj)`` as ref/artifact.py:83-84."""

    def __init__(self):
        self.records: dict = {}

    def get(self, layer, expert, proj):
        return self.records[(layer, expert, proj)]


# --------------------------------------------------------------------------
# bit packing -- ref/quant.py:243-262
# --------------------------------------------------------------------------
def pack_codes(codes, bits: int) -> bytes:
    """LSB-first continuous bitstream: code i occupies bits [i*b, i*b+b)."""
    c = np.ascontiguousarray(codes, dtype=np.uint8).ravel()
    if c.size == 0:
        return b""
    planes = (c[:, None] >> np.arange(bits, dtype=np.uint8)) & 1
    return np.packbits(planes.astype(np.uint8).ravel(), bitorder="little").tobytes()


def unpack_codes(buf: bytes, count: int, bits: int) -> np.ndarray:
    if count == 0:
        return np.zeros(0, dtype=np.uint8)
    if len(buf) < (count * bits + 7) // 8:
        raise ValueError("packed buffer too short")
    stream = np.unpackbits(np.frombuffer(buf, dtype=np.uint8), bitorder="little")
    planes = stream[: count * bits].reshape(count, bits)
    return (planes * (1 << np.arange(bits)).astype(np.uint8)).sum(axis=1).astype(np.uint8)


def packed_size_bytes(rows, cols, bits, include_metadata=False, group_size=64) -> int:
    """ref/quant.py:227-240."""
    n = (rows * cols * bits + 7) // 8
    if include_metadata:
        n += rows * (-(-cols // group_size)) * 4
    return n


def compensator_size_bytes(m, n, r, factor_bits=3) -> int:
    """ref/lowrank.py:168-172."""
    return ((m + n) * r * factor_bits + 7) // 8


# --------------------------------------------------------------------------
# quantizer -- ref/quant.py:105-224
# --------------------------------------------------------------------------
def round_half_away(v):
    """ref/quant.py:105-107."""
    return np.copysign(np.floor(np.abs(v) + 0.5), v)


def _grouped(w, gs):
    """(rows, cols) -> NaN-padded (rows, groups, gs); ref/quant.py:121-128."""
    r, c = w.shape
    g = -(-c // gs)
    out = np.full((r, g * gs), np.nan)
    out[:, :c] = w
    return out.reshape(r, g, gs)


def _codes_for(wg, s, z, qmax):
    """ref/quant.py:131-135."""
    with np.errstate(invalid="ignore"):
        return np.clip(round_half_away((wg - z) / s), 0.0, float(qmax))


def _lp_obj(wg, q, s, z, p):
    """ref/quant.py:138-143: nanmean |w - deq|^p per group."""
    with np.errstate(invalid="ignore"):
        return np.nanmean(np.abs(wg - (q * s + z)) ** p, axis=2)


def _shrink(v, beta, p):
    """ref/quant.py:110-118."""
    a = np.abs(v)
    if p == 1.0:
        t = 1.0 / beta
    else:
        with np.errstate(divide="ignore"):
            t = (1.0 / beta) * np.power(a, p - 1.0)
    return np.sign(v) * np.maximum(a - t, 0.0)


def _hqq_zero(wg, s, z, qmax, iters, p):
    """Best-objective zero points over ``iters`` proximal rounds; ref/quant.py:188-213."""
    q = _codes_for(wg, s, z, qmax)
    best = _lp_obj(wg, q, s, z, p)
    zbest = z.copy()
    beta = HQQ_BETA0
    for _ in range(iters):
        err = _shrink(np.nan_to_num(wg - (q * s + z)), beta, p)
        z = np.nanmean(wg - err - q * s, axis=2, keepdims=True)
        q = _codes_for(wg, s, z, qmax)
        obj = _lp_obj(wg, q, s, z, p)
        win = obj < best
        best = np.where(win, obj, best)
        zbest = np.where(win[:, :, None], z, zbest)
        beta *= HQQ_KAPPA
    return zbest


def quantize(w, bits=2, group_size=64, hqq_iters=20, hqq_shrink_p=0.7) -> QM:
    """Min-max affine fit per group (+ optional HQQ zero refinement); ref/quant.py:146-185."""
    w = np.asarray(w, dtype=np.float64)
    if w.ndim != 2 or w.size == 0 or not np.all(np.isfinite(w)):
        raise ValueError("quantize expects a finite non-empty 2-D matrix")
    qmax = (1 << bits) - 1
    rows, cols = w.shape
    wg = _grouped(w, group_size)
    lo = np.nanmin(wg, axis=2, keepdims=True)
    hi = np.nanmax(wg, axis=2, keepdims=True)
    s = np.where(hi == lo, 1.0, (hi - lo) / qmax)
    z = lo.copy()
    if hqq_iters > 0:
        z = _hqq_zero(wg, s, z, qmax, hqq_iters, hqq_shrink_p)
    q = _codes_for(wg, s, z, qmax).reshape(rows, -1)[:, :cols].astype(np.uint8)
    return QM(rows, cols, bits, group_size, q, s[:, :, 0].copy(), z[:, :, 0].copy())


def dequantize(qm: QM) -> np.ndarray:
    """code*scale + zero, two roundings (no FMA); ref/quant.py:216-224."""
    g = qm.groups_per_row
    buf = np.zeros((qm.rows, g * qm.group_size))
    buf[:, : qm.cols] = qm.codes.astype(np.float64)
    out = buf.reshape(qm.rows, g, qm.group_size) * qm.scales[:, :, None] + qm.zero_points[:, :, None]
    return out.reshape(qm.rows, -1)[:, : qm.cols]


# --------------------------------------------------------------------------
# low-rank compensator -- ref/lowrank.py:64-165
# --------------------------------------------------------------------------
def truncated_svd(e, r, seed=0):
    """Randomized subspace iteration with stall test; ref/lowrank.py:72-115."""
    e = np.asarray(e, dtype=np.float64)
    m, n = e.shape
    if r == 0:
        return np.zeros((m, 0)), np.zeros(0), np.zeros((0, n))
    p = min(r + SVD_OVERSAMPLE, min(m, n))
    rng = np.random.default_rng(seed)
    qb, _ = np.linalg.qr(e @ rng.standard_normal((n, p)))
    energy = float(np.sum(e * e))
    if p != min(m, n) and energy > 0.0:
        prev, stalls = -1.0, 0
        for it in range(SVD_MAX_PASSES):
            qb, _ = np.linalg.qr(e @ (e.T @ qb))
            cap = float(np.sum(np.linalg.svd(qb.T @ e, compute_uv=False)[:r] ** 2))
            if it + 1 >= SVD_MIN_PASSES:
                if abs(cap - prev) <= SVD_STALL * energy:
                    stalls += 1
                    if stalls >= 2:
                        break
                else:
                    stalls = 0
            prev = cap
    ub, sv, vt = np.linalg.svd(qb.T @ e, full_matrices=False)
    return qb @ ub[:, :r], sv[:r], vt[:r]


def build_compensator(w, qm: QM, r, factor_bits=3, projection_id="", quantize_factors=True,
                      seed=0) -> Comp:
    """sqrt(S) folded into both factors, factors quantized at 3 bits with the
    default (HQQ-20) config and group = min(64, row length); ref/lowrank.py:118-146."""
    if r == 0:
        return Comp(0, None, None, projection_id, factor_bits)
    resid = np.asarray(w, dtype=np.float64) - dequantize(qm)
    u, sv, vt = truncated_svd(resid, r, seed=seed)
    rs = np.sqrt(sv)
    uw, vw = u * rs[None, :], rs[:, None] * vt
    if not quantize_factors:
        return Comp(r, uw, vw, projection_id, factor_bits)
    uq = quantize(uw, factor_bits, min(64, max(1, uw.shape[1])))
    vq = quantize(vw, factor_bits, min(64, max(1, vw.shape[1])))
    return Comp(r, uq, vq, projection_id, factor_bits)


def factor_dense(f):
    return dequantize(f) if isinstance(f, QM) else f


def apply_compensation(qm: QM, comp: Comp | None) -> np.ndarray:
    """deq + U@V materialized; ref/lowrank.py:153-165."""
    d = dequantize(qm)
    if comp is None or comp.rank == 0:
        return d
    return d + factor_dense(comp.u) @ factor_dense(comp.v)


# --------------------------------------------------------------------------
# MoE layer -- ref/moe.py:161-259
# --------------------------------------------------------------------------
def silu(v):
    return v / (1.0 + np.exp(-v))  # ref/moe.py:161-162


def softmax(logits):
    t = np.exp(logits - logits.max())  # ref/moe.py:165-168
    return t / t.sum()


def expert_forward(w1, w3, w2, x):
    return w2 @ (silu(w1 @ x) * (w3 @ x))  # ref/moe.py:171-173


def route(x, gate, top_k, top_n):
    """(weights, selected, compensated); stable argsort => ties to lower index.
    ref/moe.py:183-193."""
    wts = softmax(gate.T @ x)
    order = np.argsort(-wts, kind="stable")
    sel = [int(i) for i in order[:top_k]]
    return wts, sel, sel[:top_n]


def resolve(store, layer_id, expert_id, compensate):
    """(w1, w3, w2) dense; ref/moe.py:196-214."""
    out = {}
    for p in PROJ_NAMES:
        rec = store.get(layer_id, expert_id, p)
        out[p] = apply_compensation(rec.qm, rec.comp) if compensate else dequantize(rec.qm)
    return out["w1"], out["w3"], out["w2"]


def forward(x, gate, experts, top_k, top_n=0, mode="compensated", store=None, layer_id=0,
            renormalize_topk=False, shared=(), compensate_shared=True):
    """One token through one layer; ref/moe.py:217-259.  ``experts``/``shared``
    are lists of (w1, w3, w2) dense triples used by mode="reference"."""
    wts, sel, comp = route(x, gate, top_k, top_n)
    mix = wts[sel]
    if renormalize_topk and mix.sum() > 0:
        mix = mix / mix.sum()
    comp = set(comp)
    y = np.zeros(gate.shape[0])
    for wgt, e in zip(mix, sel):
        if mode == "reference":
            w1, w3, w2 = experts[e]
        else:
            w1, w3, w2 = resolve(store, layer_id, e, mode == "compensated" and e in comp)
        y += wgt * expert_forward(w1, w3, w2, x)
    n_routed = gate.shape[1]
    for j in range(len(shared)):
        if mode == "reference":
            w1, w3, w2 = shared[j]
        else:
            w1, w3, w2 = resolve(store, layer_id, n_routed + j,
                                 mode == "compensated" and compensate_shared)
        y += expert_forward(w1, w3, w2, x)
    return y


# --------------------------------------------------------------------------
# synthetic inputs -- ref/moe.py:262-318, ref/pipeline.py:114-173
# --------------------------------------------------------------------------
def _tail(rng, dof, size):
    """ref/moe.py:262-266."""
    if math.isinf(dof):
        return rng.standard_normal(size)
    return rng.standard_t(dof, size) / math.sqrt(dof / (dof - 2.0))


@dataclass
class Layer:
    gate: np.ndarray                     # (hidden, E)
    experts: list = field(default_factory=list)   # [(w1, w3, w2)]
    shared: list = field(default_factory=list)


def gen_model(seed, hidden, ffn, num_layers, num_experts, num_shared=0, tail_dofs=None,
              router_skew=1.0):
    """Same single-generator draw order as ref/moe.py:269-314."""
    dofs = tuple(float(d) for d in (tail_dofs or (math.inf,)))
    rng = np.random.default_rng(seed)
    layers = []
    for _ in range(num_layers):
        g = rng.standard_normal((hidden, num_experts))
        g = g / np.linalg.norm(g, axis=0, keepdims=True) * router_skew
        ex = []
        for e in range(num_experts + num_shared):
            d = dofs[e % len(dofs)]
            w1 = _tail(rng, d, (ffn, hidden))
            w3 = _tail(rng, d, (ffn, hidden))
            w2 = _tail(rng, d, (hidden, ffn))
            ex.append((w1, w3, w2))
        layers.append(Layer(g, ex[:num_experts], ex[num_experts:]))
    return layers


def gen_tokens(seed, hidden, count):
    return np.random.default_rng(seed).standard_normal((count, hidden))  # ref/moe.py:317-318


def compress(layers, bits=2, group_size=64, hqq_iters=20, rank=16, factor_bits=3, seed=0,
             quantize_factors=True) -> Store:
    """Uniform-rank compress of every projection (ref/pipeline.py:114-173):
    rank clamped to min(shape); per-record SVD seed from
    SeedSequence([seed, layer, expert, proj_index])."""
    st = Store()
    for li, layer in enumerate(layers):
        for ei, (w1, w3, w2) in enumerate(list(layer.experts) + list(layer.shared)):
            for p, w in zip(("w1", "w3", "w2"), (w1, w3, w2)):
                qm = quantize(w, bits, group_size, hqq_iters)
                r = min(rank, min(w.shape))
                comp = None
                if r > 0:
                    rs = int(np.random.SeedSequence([seed, li, ei, PROJ_NAMES.index(p)])
                             .generate_state(1)[0])
                    comp = build_compensator(w, qm, r, factor_bits, p, quantize_factors, rs)
                st.records[(li, ei, p)] = Rec(qm, comp)
    return st


# --------------------------------------------------------------------------
# parity-protocol helpers: round inputs to the device storage formats
# --------------------------------------------------------------------------
def to_bf16(a):
    """Round-to-nearest-even fp64 -> bf16 -> fp64 (via fp32, as torch does)."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def to_fp16(a):
    return np.asarray(a, dtype=np.float16).astype(np.float64)


def round_qm_meta(qm: QM) -> QM:
    return QM(qm.rows, qm.cols, qm.bits, qm.group_size, qm.codes,
              to_fp16(qm.scales), to_fp16(qm.zero_points))


def round_store_meta(st: Store) -> Store:
    """Copy of ``st`` with every scale/zero (weights and factors) rounded to fp16."""
    out = Store()
    for k, rec in st.records.items():
        comp = rec.comp
        if comp is not None and comp.rank > 0 and isinstance(comp.u, QM):
            comp = Comp(comp.rank, round_qm_meta(comp.u), round_qm_meta(comp.v),
                        comp.projection_id, comp.factor_bits)
        out.records[k] = Rec(round_qm_meta(rec.qm), comp)
    return out
