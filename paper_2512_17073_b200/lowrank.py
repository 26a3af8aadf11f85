"""Low-rank residual compensators -- API of ref/lowrank.py, computed on the GPU.

* ``residual``            W - deq(Q(W)) with the bit-exact device dequantizer
* ``truncated_svd``       same randomized subspace iteration as ref/lowrank.py:72-115
                          (sketch r+8, 8..600 passes, 1e-14 stall test, same seeded
                          Gaussian sketch), with the QR/SVD/GEMM steps on the device
                          in fp64 (cuSOLVER/cuBLAS through torch.linalg -- library
                          linear algebra on the offline producer, not the hot path)
* ``build_compensator``   sqrt(S) fold + 3-bit factor quantization with the GPU
                          quantizer (ref/lowrank.py:118-146)
* ``apply_compensation``  deq + U@V materialised for API parity (ref/lowrank.py:153-165);
                          the MoE forward never calls it -- the fused kernels apply
                          U.(V.x) per token instead.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Union

import numpy as np

from . import _lib
from .quant import QuantConfig, QuantizedMatrix, dequantize_device, quantize

SVD_OVERSAMPLE = 8
SVD_MIN_ITERS = 8
SVD_MAX_ITERS = 600
SVD_STALL_REL = 1e-14

Factor = Union[QuantizedMatrix, np.ndarray]


class CompensatorError(ValueError):
    """Raised for shape or rank violations (ref/lowrank.py:29)."""


@dataclass
class Compensator:
    """Rank-r factor pair (ref/lowrank.py:33-49)."""

    rank: int
    u: Factor | None
    v: Factor | None
    projection_id: str = ""
    factor_bits: int = 3

    def factors_quantized(self) -> bool:
        return isinstance(self.u, QuantizedMatrix)


@dataclass
class ResidualStats:
    rel_fro: float
    kurtosis: float
    layer_id: int
    expert_id: int
    projection_id: str
    degenerate: bool = False


def _residual_device(w, qm: QuantizedMatrix):
    torch = _lib.device_required()
    w = np.asarray(w, dtype=np.float64)
    if w.shape != (qm.rows, qm.cols):
        raise CompensatorError(f"shape mismatch: {w.shape} vs {(qm.rows, qm.cols)}")
    return torch.from_numpy(np.ascontiguousarray(w)).cuda() - dequantize_device(qm)


def residual(w: np.ndarray, qm: QuantizedMatrix) -> np.ndarray:
    """Quantization error W - deq(Q(W)) (ref/lowrank.py:64-69)."""
    return _residual_device(w, qm).cpu().numpy()


def _truncated_svd_device(e, r: int, seed: int = 0):
    torch = _lib.device_required()
    m, n = e.shape
    if r < 0 or r > min(m, n):
        raise CompensatorError(f"rank {r} outside [0, {min(m, n)}] for shape {tuple(e.shape)}")
    if r == 0:
        z = torch.zeros
        return (z((m, 0), dtype=torch.float64, device="cuda"), z(0, dtype=torch.float64, device="cuda"),
                z((0, n), dtype=torch.float64, device="cuda"))
    p = min(r + SVD_OVERSAMPLE, min(m, n))
    sketch = np.random.default_rng(seed).standard_normal((n, p))  # same draw as the reference
    q, _ = torch.linalg.qr(e @ torch.from_numpy(sketch).cuda())
    total = float((e * e).sum())
    if p != min(m, n) and total > 0.0:
        prev, stalls = -1.0, 0
        for it in range(SVD_MAX_ITERS):
            q, _ = torch.linalg.qr(e @ (e.T @ q))
            cap = float((torch.linalg.svdvals(q.T @ e)[:r] ** 2).sum())
            if it + 1 >= SVD_MIN_ITERS:
                if abs(cap - prev) <= SVD_STALL_REL * total:
                    stalls += 1
                    if stalls >= 2:
                        break
                else:
                    stalls = 0
            prev = cap
    ub, s, vt = torch.linalg.svd(q.T @ e, full_matrices=False)
    return q @ ub[:, :r], s[:r], vt[:r]


def truncated_svd(e: np.ndarray, r: int, seed: int = 0):
    """Rank-r SVD by randomized subspace iteration (ref/lowrank.py:72-115)."""
    torch = _lib.device_required()
    e = np.asarray(e, dtype=np.float64)
    if e.ndim != 2:
        raise CompensatorError(f"expected a 2-D matrix, got shape {e.shape}")
    if not np.all(np.isfinite(e)):
        raise CompensatorError("matrix contains non-finite values")
    u, s, vt = _truncated_svd_device(torch.from_numpy(np.ascontiguousarray(e)).cuda(), r, seed)
    return u.cpu().numpy(), s.cpu().numpy(), vt.cpu().numpy()


def default_factor_config(row_length: int, factor_bits: int = 3) -> QuantConfig:
    """ref/lowrank.py:118-120."""
    return QuantConfig(bits=factor_bits, group_size=min(64, max(1, row_length)))


def build_compensator(w: np.ndarray, qm: QuantizedMatrix, r: int, factor_bits: int = 3,
                      projection_id: str = "", quantize_factors: bool = True,
                      seed: int = 0) -> Compensator:
    """ref/lowrank.py:123-146."""
    if r == 0:
        return Compensator(rank=0, u=None, v=None, projection_id=projection_id,
                           factor_bits=factor_bits)
    e = _residual_device(w, qm)
    if not bool(e.isfinite().all()):
        raise CompensatorError("matrix contains non-finite values")
    u, s, vt = _truncated_svd_device(e, r, seed)
    root = s.sqrt()
    u_w = (u * root[None, :]).cpu().numpy()
    v_w = (root[:, None] * vt).cpu().numpy()
    if quantize_factors:
        u_q = quantize(u_w, default_factor_config(u_w.shape[1], factor_bits))
        v_q = quantize(v_w, default_factor_config(v_w.shape[1], factor_bits))
        return Compensator(rank=r, u=u_q, v=v_q, projection_id=projection_id,
                           factor_bits=factor_bits)
    return Compensator(rank=r, u=u_w, v=v_w, projection_id=projection_id, factor_bits=factor_bits)


def _factor_device(f):
    torch = _lib.device_required()
    if isinstance(f, QuantizedMatrix):
        return dequantize_device(f)
    return torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64)).cuda()


def apply_compensation(qm: QuantizedMatrix, comp: Compensator | None) -> np.ndarray:
    """deq(Q(W)) + U V, materialised (ref/lowrank.py:153-165)."""
    deq = dequantize_device(qm)
    if comp is None or comp.rank == 0:
        return deq.cpu().numpy()
    u, v = _factor_device(comp.u), _factor_device(comp.v)
    if tuple(u.shape) != (qm.rows, comp.rank) or tuple(v.shape) != (comp.rank, qm.cols):
        raise CompensatorError(
            f"factor shapes {tuple(u.shape)}/{tuple(v.shape)} incompatible with "
            f"({qm.rows}, {qm.cols}) at rank {comp.rank}")
    _lib.check(_lib.lib().lrc_add_lowrank_f64(_lib.ptr(u.contiguous()), _lib.ptr(v.contiguous()),
                                              qm.rows, qm.cols, comp.rank, _lib.ptr(deq),
                                              _lib.stream_ptr()),
               {_lib.LRC_ERR_INVALID: CompensatorError})
    return deq.cpu().numpy()


def compensator_size_bytes(m: int, n_cols: int, r: int, factor_bits: int = 3) -> int:
    """ref/lowrank.py:168-172."""
    if m < 0 or n_cols < 0 or r < 0 or factor_bits < 0:
        raise CompensatorError("sizes must be non-negative")
    return ((m + n_cols) * r * factor_bits + 7) // 8
