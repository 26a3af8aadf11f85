"""Groupwise asymmetric low-bit weight quantizer -- API of ref/quant.py, computed on the GPU.

Same names, argument meaning and errors as the reference module
(``/root/reference/pkg/src/moe_lrc/quant.py``); numpy arrays in, fresh numpy
arrays out, inputs never mutated.  The arithmetic runs in CUDA kernels of
``liblrc.so`` (``csrc/codes.cu``):

* ``quantize``     -> ``lrc_quantize_f64``  (ref/quant.py:146-213; fp64, bit-exact
  for ``hqq_iters == 0``; HQQ rounds follow numpy's pairwise summation order)
* ``dequantize``   -> ``lrc_dequantize_f64`` (ref/quant.py:216-224; bit-exact)
* ``pack_codes``   -> ``lrc_pack_codes``     (ref/quant.py:243-249; bit-exact)
* ``unpack_codes`` -> ``lrc_unpack_codes``   (ref/quant.py:252-262; bit-exact)

``packed_size_bytes`` / ``round_half_away`` are host-side integer/shape helpers.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

SUPPORTED_BITS = (2, 3, 4)
HQQ_BETA = 10.0
HQQ_KAPPA = 1.01


class QuantizationError(ValueError):
    """Raised for invalid quantization inputs or configs (ref/quant.py:26)."""


_EXC = {_lib.LRC_ERR_INVALID: QuantizationError}


@dataclass(frozen=True)
class QuantConfig:
    """ref/quant.py:30-56."""

    bits: int = 2
    group_size: int = 64
    hqq_iters: int = 20
    hqq_shrink_p: float = 0.7

    def __post_init__(self) -> None:
        if self.bits not in SUPPORTED_BITS:
            raise QuantizationError(f"bits must be one of {SUPPORTED_BITS}, got {self.bits}")
        if self.group_size < 1:
            raise QuantizationError(f"group_size must be >= 1, got {self.group_size}")
        if self.hqq_iters < 0:
            raise QuantizationError(f"hqq_iters must be >= 0, got {self.hqq_iters}")
        if not (0.0 < self.hqq_shrink_p <= 1.0):
            raise QuantizationError(f"hqq_shrink_p must be in (0, 1], got {self.hqq_shrink_p}")


@dataclass
class QuantizedMatrix:
    """Codes (uint8, (rows, cols)) + per-group f64 scales / zero points
    (rows, ceil(cols/group_size)); ref/quant.py:59-102."""

    rows: int
    cols: int
    bits: int
    group_size: int
    codes: np.ndarray
    scales: np.ndarray
    zero_points: np.ndarray

    @property
    def groups_per_row(self) -> int:
        return -(-self.cols // self.group_size)

    @property
    def num_groups(self) -> int:
        return self.rows * self.groups_per_row

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)

    def validate(self) -> None:
        if self.bits not in SUPPORTED_BITS:
            raise QuantizationError(f"unsupported bit width {self.bits}")
        if self.codes.shape != (self.rows, self.cols):
            raise QuantizationError(f"codes shape {self.codes.shape} != ({self.rows}, {self.cols})")
        if self.scales.shape != (self.rows, self.groups_per_row):
            raise QuantizationError(
                f"scales shape {self.scales.shape} != ({self.rows}, {self.groups_per_row})")
        if self.zero_points.shape != self.scales.shape:
            raise QuantizationError("zero_points shape differs from scales")
        if self.codes.size and int(self.codes.max()) >= (1 << self.bits):
            raise QuantizationError(f"code out of range for {self.bits} bits")


def round_half_away(x: np.ndarray) -> np.ndarray:
    """Round to nearest, halves away from zero (host helper, ref/quant.py:105-107)."""
    return np.copysign(np.floor(np.abs(x) + 0.5), x)


def _to_dev(a, dtype):
    torch = _lib.device_required()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()


def quantize(w: np.ndarray, cfg: QuantConfig) -> QuantizedMatrix:
    """Quantize a 2-D matrix groupwise on the GPU (ref/quant.py:146-185)."""
    w = np.asarray(w, dtype=np.float64)
    if w.ndim != 2 or w.size == 0:
        raise QuantizationError(f"expected a non-empty 2-D matrix, got shape {w.shape}")
    if not np.all(np.isfinite(w)):
        raise QuantizationError("matrix contains non-finite values")
    torch = _lib.device_required()
    lib = _lib.lib()
    rows, cols = w.shape
    gpr = -(-cols // cfg.group_size)
    wd = _to_dev(w, np.float64)
    codes = torch.empty((rows, cols), dtype=torch.uint8, device="cuda")
    scales = torch.empty((rows, gpr), dtype=torch.float64, device="cuda")
    zeros = torch.empty((rows, gpr), dtype=torch.float64, device="cuda")
    _lib.check(lib.lrc_quantize_f64(_lib.ptr(wd), rows, cols, cfg.bits, cfg.group_size,
                                    cfg.hqq_iters, float(cfg.hqq_shrink_p), _lib.ptr(codes),
                                    _lib.ptr(scales), _lib.ptr(zeros), _lib.stream_ptr()), _EXC)
    return QuantizedMatrix(rows=rows, cols=cols, bits=cfg.bits, group_size=cfg.group_size,
                           codes=codes.cpu().numpy(), scales=scales.cpu().numpy(),
                           zero_points=zeros.cpu().numpy())


def dequantize_device(qm: QuantizedMatrix):
    """Device tensor (f64) of code*scale + zero; ref/quant.py:216-224."""
    qm.validate()
    torch = _lib.device_required()
    out = torch.empty((qm.rows, qm.cols), dtype=torch.float64, device="cuda")
    c, s, z = (_to_dev(qm.codes, np.uint8), _to_dev(qm.scales, np.float64),
               _to_dev(qm.zero_points, np.float64))
    _lib.check(_lib.lib().lrc_dequantize_f64(_lib.ptr(c), _lib.ptr(s), _lib.ptr(z), qm.rows,
                                             qm.cols, qm.group_size, _lib.ptr(out),
                                             _lib.stream_ptr()), _EXC)
    return out


def dequantize(qm: QuantizedMatrix) -> np.ndarray:
    """Reconstruct the real-valued matrix (bit-exact with ref/quant.py:216-224)."""
    return dequantize_device(qm).cpu().numpy()


def packed_size_bytes(rows: int, cols: int, bits: int, include_metadata: bool = False,
                      group_size: int = 64) -> int:
    """ref/quant.py:227-240 (codes bit-packed; +4 B/group with metadata)."""
    if rows <= 0 or cols <= 0 or bits <= 0 or group_size <= 0:
        raise QuantizationError("rows, cols, bits and group_size must be positive")
    total = (rows * cols * bits + 7) // 8
    if include_metadata:
        total += rows * (-(-cols // group_size)) * 4
    return total


def pack_codes_device(codes_dev, bits: int):
    torch = _lib.device_required()
    n = int(codes_dev.numel())
    out = torch.empty(((n * bits + 7) // 8,), dtype=torch.uint8, device="cuda")
    if n:
        _lib.check(_lib.lib().lrc_pack_codes(_lib.ptr(codes_dev), n, bits, _lib.ptr(out),
                                             _lib.stream_ptr()), _EXC)
    return out


def pack_codes(codes: np.ndarray, bits: int) -> bytes:
    """LSB-first bitstream on the GPU (ref/quant.py:243-249)."""
    flat = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1)
    if flat.size == 0:
        return b""
    return pack_codes_device(_to_dev(flat, np.uint8), bits).cpu().numpy().tobytes()


def unpack_codes(buf: bytes, count: int, bits: int) -> np.ndarray:
    """Inverse of pack_codes on the GPU (ref/quant.py:252-262)."""
    if count == 0:
        return np.zeros(0, dtype=np.uint8)
    expected = (count * bits + 7) // 8
    if len(buf) < expected:
        raise QuantizationError(f"packed buffer too short: {len(buf)} < {expected}")
    torch = _lib.device_required()
    src = _to_dev(np.frombuffer(bytes(buf[:expected]), dtype=np.uint8), np.uint8)
    out = torch.empty((count,), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().lrc_unpack_codes(_lib.ptr(src), count, bits, _lib.ptr(out),
                                           _lib.stream_ptr()), _EXC)
    return out.cpu().numpy()
