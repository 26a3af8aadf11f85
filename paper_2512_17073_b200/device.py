"""Device-resident MoE layer: artifact upload + batched forward through the C-ABI.

``LRCMoELayer`` is the batched device API behind ``moe.forward``: it owns the
HBM copies of one layer's quantized experts (reference bitstream + fp16
scale/zero, plus the T2 tiled layout for 2-bit/group-64 weights) and runs
``lrc_layer_forward`` on torch tensors:

    layer = LRCMoELayer.from_artifacts(gate, artifacts, layer_id, num_experts, num_shared)
    y, idx, w = layer.forward(x_bf16, top_k=2, top_n=1)    # x (B, d) bf16 on cuda

HBM layout per expert: w1|w3 interleaved tiles
(``up_tiles``), w2 tiles (``down_tiles``), LR factors U/V as packed 3-bit
bitstreams with fp16 metadata.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .quant import QuantizedMatrix, pack_codes_device

PROJ = ("w1", "w3", "w2")


class _Keep:
    """Holds device tensors referenced by raw pointers in C descriptors."""

    def __init__(self):
        self.items = []

    def add(self, t):
        self.items.append(t)
        return t


def _qm_to_device(qm: QuantizedMatrix, keep: _Keep) -> _lib.LrcQmat:
    torch = _lib.device_required()
    codes = torch.from_numpy(np.ascontiguousarray(qm.codes, dtype=np.uint8)).cuda()
    packed = keep.add(pack_codes_device(codes, qm.bits))
    # scale/zero rounded to fp16 on the host (numpy rounding; the parity oracle
    # applies the identical rounding)
    s = keep.add(torch.from_numpy(_fp16_meta(qm.scales, "scale").view(np.uint16)).cuda())
    z = keep.add(torch.from_numpy(_fp16_meta(qm.zero_points, "zero point").view(np.uint16)).cuda())
    m = _lib.LrcQmat()
    m.packed, m.scales, m.zeros, m.dense = packed.data_ptr(), s.data_ptr(), z.data_ptr(), None
    m.rows, m.cols, m.bits, m.group_size = qm.rows, qm.cols, qm.bits, qm.group_size
    return m


def _fp16_meta(a, what: str):
    """Group scale / zero metadata as fp16 (the kernels' format).  The
    reference keeps them in f8 (ref/quant.py); a value that overflows fp16, or
    a nonzero scale that flushes to 0, would silently corrupt the output, so
    both raise ArtifactError.  (fp16 subnormals, |v| < 6.1e-5, keep an absolute
    error below 3e-8: accepted.)"""
    a64 = np.asarray(a, dtype=np.float64)
    with np.errstate(over="ignore"):
        h = a64.astype(np.float16)
    bad = ~np.isfinite(h) & np.isfinite(a64)
    if what == "scale":
        bad |= (a64 != 0) & (h == 0)
    bad |= ~np.isfinite(a64)
    if bad.any():
        from .artifact import ArtifactError

        v = float(a64.ravel()[np.flatnonzero(bad.ravel())[0]])
        raise ArtifactError(f"{what} value {v!r} does not fit the fp16 metadata the device kernels use")
    return np.ascontiguousarray(h)


def _packed_to_device(packed: bytes, rows, cols, bits, group_size, scales, zeros,
                      keep: _Keep) -> _lib.LrcQmat:
    """Reference on-disk form (ref/artifact.py:103-108) straight to HBM."""
    torch = _lib.device_required()
    p = keep.add(torch.frombuffer(bytearray(packed), dtype=torch.uint8).cuda())
    s = keep.add(torch.from_numpy(_fp16_meta(scales, "scale").view(np.uint16)).cuda())
    z = keep.add(torch.from_numpy(_fp16_meta(zeros, "zero point").view(np.uint16)).cuda())
    m = _lib.LrcQmat()
    m.packed, m.scales, m.zeros, m.dense = p.data_ptr(), s.data_ptr(), z.data_ptr(), None
    m.rows, m.cols, m.bits, m.group_size = rows, cols, bits, group_size
    return m


def _factor_to_device(f, keep: _Keep) -> _lib.LrcQmat:
    if hasattr(f, "codes"):  # QuantizedMatrix (or any duck-typed equivalent)
        return _qm_to_device(f, keep)
    torch = _lib.device_required()
    a = np.ascontiguousarray(f, dtype=np.float32)
    d = keep.add(torch.from_numpy(a).cuda())
    m = _lib.LrcQmat()
    m.packed = m.scales = m.zeros = None
    m.dense = d.data_ptr()
    m.rows, m.cols, m.bits, m.group_size = a.shape[0], a.shape[1], 32, 1
    return m


def _zero_qmat(rows, cols, keep: _Keep) -> _lib.LrcQmat:
    """All-zero 2-bit placeholder (experts absent from the artifact store)."""
    qm = QuantizedMatrix(rows, cols, 2, 64, np.zeros((rows, cols), np.uint8),
                         np.zeros((rows, -(-cols // 64))), np.zeros((rows, -(-cols // 64))))
    return _qm_to_device(qm, keep)


def build_tiles(mats, keep: _Keep):
    """T2 tiled layout of 1 or 2 same-shape 2-bit/gs64 matrices (LrcQmat)."""
    torch = _lib.device_required()
    lib = _lib.lib()
    ni = len(mats)
    nbytes = lib.lrc_tiles_bytes(mats[0].rows, mats[0].cols, ni)
    t = keep.add(torch.empty((nbytes,), dtype=torch.uint8, device="cuda"))
    arr = (_lib.LrcQmat * ni)(*mats)
    _lib.check(lib.lrc_build_tiles(arr, ni, _lib.ptr(t), _lib.stream_ptr()))
    return t


def build_down_tiles(w2: _lib.LrcQmat, keep: _Keep):
    """W2 tiles for the down kernel: the two row halves [0, H/2) and [H/2, H)
    interleaved as the kernel's two matrices (two accumulator chains)."""
    half = w2.rows // 2
    groups = -(-w2.cols // w2.group_size)
    views = []
    for r0 in (0, half):
        v = _lib.LrcQmat()
        ctypes.memmove(ctypes.byref(v), ctypes.byref(w2), ctypes.sizeof(_lib.LrcQmat))
        v.rows = half
        v.packed = w2.packed + (r0 * w2.cols * w2.bits) // 8
        v.scales = w2.scales + r0 * groups * 2
        v.zeros = w2.zeros + r0 * groups * 2
        views.append(v)
    return build_tiles(views, keep)


def build_lr_tiles(ex: _lib.LrcExpert, hidden: int, ffn: int, keep: _Keep) -> bool:
    """Low-rank factor tiles riding with the weight tiles (csrc/fast.cu); False if the
    factors cannot be tiled (raw fp32 factors -> generic kernels)."""
    torch = _lib.device_required()
    lib = _lib.lib()
    up, down = ctypes.c_int64(), ctypes.c_int64()
    if lib.lrc_lr_tiles_bytes(ctypes.byref(ex), hidden, ffn, ctypes.byref(up), ctypes.byref(down)) != 0:
        return False
    tu = keep.add(torch.empty((max(up.value, 16),), dtype=torch.uint8, device="cuda"))
    td = keep.add(torch.empty((max(down.value, 16),), dtype=torch.uint8, device="cuda"))
    _lib.check(lib.lrc_build_lr_tiles(ctypes.byref(ex), hidden, ffn, _lib.ptr(tu), _lib.ptr(td),
                                      _lib.stream_ptr()))
    ex.up_lr_tiles = tu.data_ptr() if up.value else None
    ex.down_lr_tiles = td.data_ptr() if down.value else None
    return True


def tiles_eligible(*mats: _lib.LrcQmat) -> bool:
    """2-bit gs64 codes; W2 (rows = hidden) must split into 16-row-tiled halves."""
    return all(m.bits == 2 and m.group_size == 64 and m.packed for m in mats) and mats[-1].rows % 32 == 0


class LRCMoELayer:
    """One MoE layer resident in HBM, forward through liblrc (no CPU path)."""

    def __init__(self, gate: np.ndarray, experts: list, hidden: int, ffn: int, num_experts: int,
                 num_shared: int, keep: _Keep, max_tokens: int = 64, top_k: int = 2,
                 missing: frozenset = frozenset()):
        torch = _lib.device_required()
        self.hidden, self.ffn = hidden, ffn
        self.num_experts, self.num_shared = num_experts, num_shared
        self.missing = missing
        self._keep = keep
        self._experts = experts
        self.gate_t = keep.add(torch.from_numpy(np.ascontiguousarray(np.asarray(gate, np.float64).T)).cuda())
        self.max_tokens, self.top_k = max_tokens, top_k
        self._handle = None
        self._prefill_min = None  # None: the library default (LRC_PREFILL_MIN or 128)
        self._tcd_max = None      # None: the library default (LRC_TCD_MAX or 8)
        self._pager = None        # lrc_layer_set_pager arguments (re-applied on re-create)
        self._pager_cache = None  # (cache handle, layer key) for lrc_layer_set_pager_cache
        self._create()

    def _create(self):
        lib = _lib.lib()
        if self._handle is not None:
            lib.lrc_layer_destroy(self._handle)
        arr = (_lib.LrcExpert * len(self._experts))(*self._experts)
        h = ctypes.c_void_p()
        _lib.check(lib.lrc_layer_create(_lib.ptr(self.gate_t), self.hidden, self.ffn,
                                        self.num_experts, self.num_shared, arr,
                                        self.max_tokens, max(self.top_k, 1), ctypes.byref(h)))
        self._handle = h
        if self._prefill_min is not None:
            _lib.check(lib.lrc_layer_set_prefill_min(h, int(self._prefill_min)))
        if self._tcd_max is not None:
            _lib.check(lib.lrc_layer_set_tcd_max(h, int(self._tcd_max)))
        if self._pager is not None:
            _lib.check(lib.lrc_layer_set_pager(h, *self._pager))
            if self._pager_cache is not None:
                _lib.check(lib.lrc_layer_set_pager_cache(h, *self._pager_cache))

    def set_pager(self, host_blocks, offsets, block_bytes: int, slots_ptr: int, n_slots: int,
                  slot_bytes: int):
        """GPU-driven expert paging (lrc_layer_set_pager); kept across workspace re-creates."""
        self._pager = (host_blocks, offsets, int(block_bytes), ctypes.c_void_p(slots_ptr), int(n_slots),
                       int(slot_bytes))
        _lib.check(_lib.lib().lrc_layer_set_pager(self._handle, *self._pager))


    def set_pager_cache(self, cache_handle, layer_key: int):
        """Budgeted LRU over the pager's slots shared across layers
        (lrc_layer_set_pager_cache); kept across workspace re-creates."""
        self._pager_cache = (ctypes.c_void_p(cache_handle), int(layer_key))
        _lib.check(_lib.lib().lrc_layer_set_pager_cache(self._handle, *self._pager_cache))
    def set_tcd_max(self, max_tokens: int):
        """Batches of <= max_tokens (<= 8) run the tensor-core decode engine when
        eligible; 0 disables it."""
        self._tcd_max = int(max_tokens)
        _lib.check(_lib.lib().lrc_layer_set_tcd_max(self._handle, self._tcd_max))

    @property
    def tcd_eligible(self) -> bool:
        return bool(_lib.lib().lrc_layer_tcd_eligible(self._handle))

    def set_prefill_min(self, min_tokens: int):
        """Batches of >= min_tokens run the tcgen05 grouped-GEMM prefill path
        (when eligible); <= 0 disables it."""
        self._prefill_min = int(min_tokens)
        _lib.check(_lib.lib().lrc_layer_set_prefill_min(self._handle, self._prefill_min))

    @property
    def prefill_eligible(self) -> bool:
        return bool(_lib.lib().lrc_layer_prefill_eligible(self._handle))

    def __del__(self):
        try:
            if self._handle is not None and _lib._lib is not None:
                _lib._lib.lrc_layer_destroy(self._handle)
        except Exception:
            pass

    @property
    def tiled(self) -> bool:
        return all(e.up_tiles and e.down_tiles for e in self._experts)

    def ensure_capacity(self, B: int, top_k: int):
        if B > self.max_tokens or top_k > self.top_k:
            self.max_tokens = max(B, self.max_tokens)
            self.top_k = max(top_k, self.top_k)
            self._create()

    def forward(self, x, top_k: int, top_n: int = 0, renormalize: bool = False,
                compensate_shared: bool = True, y=None, topk_idx=None, topk_w=None,
                generic: bool = False):
        """x: (B, hidden) bf16 cuda tensor -> y (B, hidden) f32, topk idx/w (B, top_k)."""
        torch = _lib.device_required()
        B = int(x.shape[0])
        self.ensure_capacity(B, top_k)
        if y is None:
            y = torch.empty((B, self.hidden), dtype=torch.float32, device="cuda")
        if topk_idx is None:
            topk_idx = torch.empty((B, max(top_k, 1)), dtype=torch.int32, device="cuda")
        if topk_w is None:
            topk_w = torch.empty((B, max(top_k, 1)), dtype=torch.float32, device="cuda")
        fn = self.lib_forward_generic if generic else self.lib_forward
        _lib.check(fn(self._handle, _lib.ptr(x), B, top_k, top_n, int(bool(renormalize)),
                      int(bool(compensate_shared)), _lib.ptr(y), _lib.ptr(topk_idx),
                      _lib.ptr(topk_w), _lib.stream_ptr()))
        return y, topk_idx, topk_w

    def forward_pairs(self, x, expert, weight, comp, y=None, validate: bool = True):
        """Given routing (expert-parallel receive side): row b of x (bf16 cuda)
        goes to expert[b] (int32) with weight[b] (f32); the low-rank term iff
        comp[b] (uint8).  Returns y (B, hidden) f32 = weight * E(x) per row.
        ``validate`` checks the ids on the host (one synchronisation); callers
        that build the ids themselves (the EP layer) pass False."""
        torch = _lib.device_required()
        B = int(x.shape[0])
        if y is None:
            y = torch.empty((B, self.hidden), dtype=torch.float32, device="cuda")
        if B == 0:
            return y
        self.ensure_capacity(B, 1)
        ne = self.num_experts + self.num_shared
        ex = expert.to(device="cuda", dtype=torch.int32).contiguous()
        if validate and (int(ex.min()) < 0 or int(ex.max()) >= ne):
            raise ValueError(f"forward_pairs: expert ids must be in [0, {ne})")
        w = weight.to(device="cuda", dtype=torch.float32).contiguous()
        c = comp.to(device="cuda", dtype=torch.uint8).contiguous()
        _lib.check(_lib.lib().lrc_layer_forward_pairs(self._handle, _lib.ptr(x.contiguous()), B,
                                                      _lib.ptr(ex), _lib.ptr(w), _lib.ptr(c),
                                                      _lib.ptr(y), _lib.stream_ptr()))
        return y

    def forward_host(self, x_host, y_host, top_k: int, top_n: int = 0, renormalize: bool = False,
                     compensate_shared: bool = True):
        """End-to-end call with HOST buffers (pinned torch CPU tensors): H2D of x,
        the layer forward and D2H of y, stream-ordered (caller synchronises)."""
        B = int(x_host.shape[0])
        self.ensure_capacity(B, top_k)
        _lib.check(_lib.lib().lrc_layer_forward_host(
            self._handle, _lib.ptr(x_host), B, top_k, top_n, int(bool(renormalize)),
            int(bool(compensate_shared)), _lib.ptr(y_host), _lib.stream_ptr()))
        return y_host

    def set_profiling(self, on: bool):
        _lib.check(_lib.lib().lrc_layer_set_profiling(self._handle, int(bool(on))))

    def phase_ms(self):
        """{route, lr_down, up, down} ms of the last forward (profiling on)."""
        ms = (ctypes.c_float * 4)()
        _lib.check(_lib.lib().lrc_layer_phase_ms(self._handle, ms))
        return list(ms)

    @property
    def lib_forward(self):
        return _lib.lib().lrc_layer_forward

    @property
    def lib_forward_generic(self):
        return _lib.lib().lrc_layer_forward_generic

    def last_launches(self) -> int:
        return int(_lib.lib().lrc_layer_last_launches(self._handle))

    # ------------------------------------------------------------ builders --
    @classmethod
    def from_records(cls, gate, records, hidden, ffn, num_experts, num_shared, max_tokens=64,
                     top_k=2, tiles=True):
        """records: list (num_experts + num_shared) of {proj: rec} with rec.qm / rec.comp,
        or None for an expert absent from the store."""
        keep = _Keep()
        experts, missing = [], set()
        absent = None  # one shared all-zero placeholder for every absent expert
        for eid, rec in enumerate(records):
            ex = _lib.LrcExpert()
            if rec is None:
                missing.add(eid)
                if absent is None:
                    absent = _lib.LrcExpert()
                    absent.w1 = _zero_qmat(ffn, hidden, keep)
                    absent.w3 = absent.w1
                    absent.w2 = _zero_qmat(hidden, ffn, keep)
                    if tiles and tiles_eligible(absent.w1, absent.w3, absent.w2):
                        absent.up_tiles = build_tiles([absent.w1, absent.w3], keep).data_ptr()
                        absent.down_tiles = build_down_tiles(absent.w2, keep).data_ptr()
                experts.append(absent)
                continue
            else:
                for p in PROJ:
                    setattr(ex, p, _qm_to_device(rec[p].qm, keep))
                rank = 0
                for p, (un, vn) in zip(PROJ, (("u1", "v1"), ("u3", "v3"), ("u2", "v2"))):
                    comp = rec[p].comp
                    if comp is not None and comp.rank > 0:
                        setattr(ex, un, _factor_to_device(comp.u, keep))
                        setattr(ex, vn, _factor_to_device(comp.v, keep))
                        rank = max(rank, comp.rank)
                ex.rank = rank
            if tiles and tiles_eligible(ex.w1, ex.w3, ex.w2):
                ex.up_tiles = build_tiles([ex.w1, ex.w3], keep).data_ptr()
                ex.down_tiles = build_down_tiles(ex.w2, keep).data_ptr()
                if ex.rank:
                    build_lr_tiles(ex, hidden, ffn, keep)
            experts.append(ex)
        return cls(gate, experts, hidden, ffn, num_experts, num_shared, keep, max_tokens, top_k,
                   frozenset(missing))

    @classmethod
    def from_artifacts(cls, gate, artifacts, layer_id, num_experts, num_shared, hidden, ffn,
                       **kw):
        """Pull every expert of ``layer_id`` through the reference's artifact
        protocol ``artifacts.get(layer, expert, proj)`` (ref/moe.py:196-214)."""
        records = []
        for eid in range(num_experts + num_shared):
            rec = {}
            try:
                for p in PROJ:
                    r = artifacts.get(layer_id, eid, p)
                    if r is None:
                        raise KeyError(p)
                    rec[p] = r
            except (KeyError, AttributeError):
                rec = None
            records.append(rec)
        return cls.from_records(gate, records, hidden, ffn, num_experts, num_shared, **kw)
