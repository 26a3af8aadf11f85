"""Offload engine (SURVEY config C3, north-star item 4): quantized experts and
low-rank factors live in pinned host memory; an LRU cache of GPU expert slots
holds the ones in use; misses are fetched on demand with cudaMemcpyAsync on a
side stream.

Per layer step (decode, B <= 8 tokens):

1. route on the GPU (``lrc_route``, the same fp64 router as the layer) and read
   the (B, k) expert ids back -- the only host synchronisation;
2. for each selected expert not resident: pick the least-recently-used slot
   not needed by this step, wait for its last use on the compute stream, and
   copy the expert's bytes host -> slot on the copy stream;
3. point the layer's expert descriptors at the slots (``lrc_layer_set_expert``)
   and run the layer forward on the compute stream after the copies' events;
All copies of a step are issued before the stream-ordered descriptor updates, so
the host link runs back to back.  Temporal locality of routing across tokens is
served by the LRU itself (a speculative next-layer prefetch was measured to
regress -- it reorders the LRU onto slots still in use -- and was removed).

What an expert costs on the host link is exactly what the tiled decode path
reads: the w1|w3 and w2 T2 tiles (codes + fp16 metadata, the reference's
``packed_size_bytes(include_metadata=True)``), the low-rank tiles, and the V1/V3
factors of the speculative V.x -- SURVEY 8(d)'s C3 bytes per token.  Fields the
tiled path never reads (reference-layout w1/w3/w2 codes, U factors, V2) point
at shared all-zero placeholders of the right shapes.
"""
from __future__ import annotations

import collections
import ctypes

from . import _lib
from .device import LRCMoELayer, _Keep, _zero_qmat, build_down_tiles, build_tiles

NAMES = ("up", "down", "up_lr", "down_lr", "v1p", "v1s", "v1z", "v3p", "v3s", "v3z")


class HostExpert:
    """Pinned host bytes of one expert + the descriptor fields (shapes, rank)."""

    def __init__(self, bufs: dict, proto: _lib.LrcExpert):
        self.bufs = bufs
        self.proto = proto

    @property
    def nbytes(self) -> int:
        return sum(int(t.numel()) for t in self.bufs.values())


def _lr_tiles(ex, hidden, ffn):
    torch = _lib.device_required()
    lib = _lib.lib()
    up, down = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(lib.lrc_lr_tiles_bytes(ctypes.byref(ex), hidden, ffn, ctypes.byref(up), ctypes.byref(down)))
    tu = torch.empty((max(up.value, 16),), dtype=torch.uint8, device="cuda")
    td = torch.empty((max(down.value, 16),), dtype=torch.uint8, device="cuda")
    _lib.check(lib.lrc_build_lr_tiles(ctypes.byref(ex), hidden, ffn, _lib.ptr(tu), _lib.ptr(td),
                                      _lib.stream_ptr()))
    return tu[:up.value], td[:down.value]


def host_experts_from_synth(sl) -> list:
    """Pinned host copies of every expert of a (device-resident) SynthLayer."""
    torch = _lib.device_required()
    out = []
    for e, ex in enumerate(sl.layer._experts):
        keep = _Keep()
        dev = {"up": build_tiles([ex.w1, ex.w3], keep), "down": build_down_tiles(ex.w2, keep)}
        if ex.rank:
            dev["up_lr"], dev["down_lr"] = _lr_tiles(ex, sl.hidden, sl.ffn)
            for v in ("v1", "v3"):
                p, s, z = sl.raw[e][v][:3]
                dev[v + "p"], dev[v + "s"], dev[v + "z"] = p, s, z
        bufs = {}
        for n in NAMES:
            t = dev.get(n)
            if t is None:
                bufs[n] = torch.empty((0,), dtype=torch.uint8).pin_memory()
            else:
                bufs[n] = t.contiguous().view(torch.uint8).reshape(-1).cpu().pin_memory()
        proto = _lib.LrcExpert()
        ctypes.memmove(ctypes.byref(proto), ctypes.byref(ex), ctypes.sizeof(_lib.LrcExpert))
        out.append(HostExpert(bufs, proto))
    torch.cuda.synchronize()
    return out


class OffloadEngine:
    """Layers whose experts are fetched on demand into ``n_slots`` GPU slots."""

    def __init__(self, gates, experts, hidden: int, ffn: int, top_k: int, top_n: int,
                 n_slots: int, max_tokens: int = 8):
        torch = _lib.device_required()
        self.hidden, self.ffn, self.k, self.n = hidden, ffn, top_k, top_n
        self.E = len(experts[0])
        self.host = experts  # [layer][expert] -> HostExpert
        size = {n: max(int(he.bufs[n].numel()) for lay in experts for he in lay) for n in NAMES}
        self.slots = [{n: torch.empty((max(size[n], 16),), dtype=torch.uint8, device="cuda") for n in NAMES}
                      for _ in range(n_slots)]
        self.slot_key = [None] * n_slots
        self.slot_used = [None] * n_slots   # compute-stream event of the slot's last use
        self.slot_ready = [None] * n_slots  # copy-stream event of the slot's last fill
        self.lru = collections.OrderedDict()  # (layer, expert) -> slot, oldest first
        self.copy_stream = torch.cuda.Stream()
        self.keep = _Keep()
        self.stats = {"hits": 0, "misses": 0, "bytes": 0}
        # routing read-back: pinned buffer + event polled by the host (a blocking
        # pageable .cpu() sync showed 10-600 ms host stalls on the B200 boxes)
        self._idx_host = torch.empty((max_tokens * max(top_k, 1),), dtype=torch.int32).pin_memory()
        self._idx_ev = torch.cuda.Event()
        # shared placeholders for the descriptor fields the tiled path never reads
        self._zw13 = _zero_qmat(ffn, hidden, self.keep)
        self._zw2 = _zero_qmat(hidden, ffn, self.keep)
        self._zfac = {}
        self.layers = []
        for l, gate in enumerate(gates):
            descs = [self._desc(l, e, 0) for e in range(self.E)]
            dl = LRCMoELayer(gate, descs, hidden, ffn, self.E, 0, self.keep, max_tokens=max_tokens, top_k=top_k)
            # the descriptors' reference-layout weights are zero placeholders: only
            # the tiled decode kernels (which read the slot tiles) may run
            dl.set_prefill_min(0)
            dl.set_tcd_max(0)
            self.layers.append(dl)

    # ----------------------------------------------------------- helpers --
    def _zero_factor(self, m: _lib.LrcQmat) -> _lib.LrcQmat:
        key = (m.rows, m.cols, m.bits, m.group_size)
        if key not in self._zfac:
            torch = _lib.device_required()
            nbytes = (m.rows * m.cols * m.bits + 7) // 8
            g = -(-m.cols // m.group_size) * m.rows
            p = self.keep.add(torch.zeros((max(nbytes, 16),), dtype=torch.uint8, device="cuda"))
            s = self.keep.add(torch.zeros((max(g, 8),), dtype=torch.int16, device="cuda"))
            z = _lib.LrcQmat()
            z.packed, z.scales, z.zeros = p.data_ptr(), s.data_ptr(), s.data_ptr()
            z.rows, z.cols, z.bits, z.group_size = m.rows, m.cols, m.bits, m.group_size
            self._zfac[key] = z
        return self._zfac[key]

    def _desc(self, layer: int, expert: int, slot: int) -> _lib.LrcExpert:
        he = self.host[layer][expert]
        buf = self.slots[slot]
        d = _lib.LrcExpert()
        d.w1, d.w3, d.w2 = self._zw13, self._zw13, self._zw2
        d.rank = he.proto.rank
        if he.proto.rank:
            for f in ("u1", "u3", "u2", "v2"):
                setattr(d, f, self._zero_factor(getattr(he.proto, f)))
            for v in ("v1", "v3"):
                q = _lib.LrcQmat()
                src = getattr(he.proto, v)
                q.rows, q.cols, q.bits, q.group_size = src.rows, src.cols, src.bits, src.group_size
                q.packed = buf[v + "p"].data_ptr()
                q.scales = buf[v + "s"].data_ptr()
                q.zeros = buf[v + "z"].data_ptr()
                setattr(d, v, q)
            d.up_lr_tiles = buf["up_lr"].data_ptr()
            d.down_lr_tiles = buf["down_lr"].data_ptr()
        d.up_tiles = buf["up"].data_ptr()
        d.down_tiles = buf["down"].data_ptr()
        return d

    def _fetch(self, key, busy: set):
        """Slot holding ``key``; issues the host->device copy on a miss."""
        torch = _lib.device_required()
        if key in self.lru:
            self.lru.move_to_end(key)
            self.stats["hits"] += 1
            return self.lru[key]
        free = [s for s in range(len(self.slots)) if self.slot_key[s] is None]
        if free:
            slot = free[0]
        else:
            victims = [k for k in self.lru if k not in busy]
            if not victims:
                raise RuntimeError("offload: more experts in flight than GPU slots")
            slot = self.lru.pop(victims[0])
            self.slot_key[slot] = None
        he = self.host[key[0]][key[1]]
        with torch.cuda.stream(self.copy_stream):
            if self.slot_used[slot] is not None:
                self.copy_stream.wait_event(self.slot_used[slot])
            for n in NAMES:
                src = he.bufs[n]
                if src.numel():
                    self.slots[slot][n][:src.numel()].copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        self.slot_ready[slot] = ev
        self.slot_key[slot] = key
        self.lru[key] = slot
        self.stats["misses"] += 1
        self.stats["bytes"] += he.nbytes
        return slot

    # -------------------------------------------------------------- step --
    def route(self, layer: int, x):
        torch = _lib.device_required()
        dl = self.layers[layer]
        B = int(x.shape[0])
        idx = torch.empty((B, self.k), dtype=torch.int32, device="cuda")
        w = torch.empty((B, self.k), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().lrc_route(_lib.ptr(dl.gate_t), _lib.ptr(x.contiguous()), _lib.DTYPE_BF16, B,
                                        self.hidden, self.E, self.k, self.n, 0, ctypes.c_void_p(0),
                                        _lib.ptr(idx), _lib.ptr(w), _lib.stream_ptr()))
        return idx

    def forward_layer(self, layer: int, x):
        """x (B, hidden) bf16 cuda -> y (B, hidden) f32 of layer ``layer``."""
        torch = _lib.device_required()
        idx = self.route(layer, x).reshape(-1)
        host = self._idx_host[:idx.numel()]
        host.copy_(idx, non_blocking=True)
        self._idx_ev.record(torch.cuda.current_stream())
        while not self._idx_ev.query():  # poll (no blocking driver wait)
            pass
        need = sorted(set(host.tolist()))
        if need and (need[0] < 0 or need[-1] >= self.E):
            raise ValueError("offload: the router selected no valid expert (non-finite input?)")
        keys = {(layer, e) for e in need}
        dl = self.layers[layer]
        # issue every copy of the step before the (blocking) descriptor updates,
        # so the host link stays busy back to back
        slots = {e: self._fetch((layer, e), keys) for e in need}
        for e in need:
            d = self._desc(layer, e, slots[e])
            _lib.check(_lib.lib().lrc_layer_set_expert_async(dl._handle, e, ctypes.byref(d),
                                                             _lib.stream_ptr()))
            dl._experts[e] = d  # a workspace re-create keeps the current slots
            torch.cuda.current_stream().wait_event(self.slot_ready[slots[e]])
        y, _, _ = dl.forward(x, self.k, self.n)
        done = torch.cuda.Event()
        done.record(torch.cuda.current_stream())
        for e in need:
            self.slot_used[self.lru[(layer, e)]] = done
        return y

    def forward(self, x, normalize: bool = False):
        """x through every layer (decode chain: y of layer l, rounded to bf16,
        is the input of layer l+1; ``normalize`` rescales each y to unit RMS as
        a stand-in for the model's RMSNorm between MoE layers)."""
        torch = _lib.device_required()
        for l in range(len(self.layers)):
            y = self.forward_layer(l, x)
            if normalize:
                y = y * torch.rsqrt(y.pow(2).mean(dim=-1, keepdim=True) + 1e-6)
            x = y.to(torch.bfloat16)
        return x


class GpuPagerEngine(OffloadEngine):
    """Offload with GPU-driven paging (``lrc_layer_set_pager``): every expert is
    one block of device-mapped pinned host memory (sections in ``NAMES`` order
    at fixed offsets); each layer forward copies its active experts into slots
    inside the stream (SM loads over the host link) and repoints their
    descriptors -- no host round trip per layer, so a token's whole layer chain
    is asynchronous and graph-capturable.  Default: no cross-token cache, slot
    a holds the a-th active expert of the current step (the C3 "cache budget
    0" case).  ``cache_slots`` > 0: a budgeted LRU over that many slots shared
    by all layers, decided on the device (``lrc_pager_cache``; hits move
    nothing) -- the reference cost model's cache_policy="lru".
    """

    def __init__(self, gates, experts, hidden: int, ffn: int, top_k: int, top_n: int, max_tokens: int = 1,
                 cache_slots: int = 0):
        torch = _lib.device_required()
        self.hidden, self.ffn, self.k, self.n = hidden, ffn, top_k, top_n
        self.E = len(experts[0])
        self.host = experts
        self.keep = _Keep()
        n_slots = min(self.E, max_tokens * max(top_k, 1))
        self.cache = None
        if cache_slots:
            if cache_slots < n_slots:
                raise ValueError(f"cache_slots must hold one step's experts (>= {n_slots})")
            n_slots = int(cache_slots)
            h = ctypes.c_void_p()
            _lib.check(_lib.lib().lrc_pager_cache_create(n_slots, ctypes.byref(h)))
            self.cache = h
        size = {n: max(int(he.bufs[n].numel()) for lay in experts for he in lay) for n in NAMES}
        self.offsets, o = {}, 0
        for n in NAMES:
            self.offsets[n] = o if size[n] else -1
            o += (size[n] + 255) // 256 * 256
        self.block_bytes = max(o, 256)
        self.slot_mem = self.keep.add(torch.zeros((n_slots, self.block_bytes), dtype=torch.uint8, device="cuda"))
        self.slots = [{n: self.slot_mem[s, max(self.offsets[n], 0):max(self.offsets[n], 0) + max(size[n], 1)]
                       for n in NAMES} for s in range(n_slots)]
        # one pinned block per (layer, expert); UVA: the host pointer is device-visible
        self.blocks = []
        for lay in experts:
            row = []
            for he in lay:
                blk = torch.zeros((self.block_bytes,), dtype=torch.uint8).pin_memory()
                for n in NAMES:
                    t = he.bufs[n]
                    if t.numel():
                        blk[self.offsets[n]:self.offsets[n] + t.numel()].copy_(t)
                row.append(blk)
            self.blocks.append(row)
        self.stats = {"bytes": 0, "steps": 0}
        self._trace = None
        self._zw13 = _zero_qmat(ffn, hidden, self.keep)
        self._zw2 = _zero_qmat(hidden, ffn, self.keep)
        self._zfac = {}
        offs = (ctypes.c_int64 * 10)(*[self.offsets[n] for n in NAMES])
        self.layers = []
        for l, gate in enumerate(gates):
            descs = [self._desc(l, e, 0) for e in range(self.E)]
            dl = LRCMoELayer(gate, descs, hidden, ffn, self.E, 0, self.keep, max_tokens=max_tokens, top_k=top_k)
            dl.set_prefill_min(0)
            dl.set_tcd_max(0)
            ptrs = (ctypes.c_void_p * self.E)(*[b.data_ptr() for b in self.blocks[l]])
            dl.set_pager(ptrs, offs, self.block_bytes, self.slot_mem.data_ptr(), n_slots, self.block_bytes)
            if self.cache is not None:
                dl.set_pager_cache(self.cache.value, l)
            self.layers.append(dl)

    def forward_layer(self, layer: int, x):
        y, idx, w = self.layers[layer].forward(x, self.k, self.n)
        self.stats["steps"] += 1
        if self._trace is not None:  # device copies only; read back by routing_trace()
            self._trace.append((layer, idx.clone(), w.clone()))
        return y

    def cache_stats(self):
        """Cumulative (hits, misses) of the budgeted cache (None without one)."""
        if self.cache is None:
            return None
        hm = (ctypes.c_int64 * 2)()
        _lib.check(_lib.lib().lrc_pager_cache_stats(self.cache, hm))
        return int(hm[0]), int(hm[1])

    def __del__(self):
        if getattr(self, "cache", None) is not None:
            try:
                _lib.lib().lrc_pager_cache_destroy(self.cache)
            except Exception:
                pass
            self.cache = None

    def start_trace(self):
        """Record the routing of every following layer step."""
        self._trace = []

    def routing_trace(self):
        """The recorded steps as a ``moe.RoutingTrace`` (token = decode step;
        one record per (token, layer) for the first row of each batch)."""
        from .moe import RoutingTrace, TraceRecord

        recs = []
        steps = self._trace or []
        nl = len(self.layers)
        for i, (layer, idx, w) in enumerate(steps):
            sel = [int(v) for v in idx[0].cpu().tolist()]
            ww = w[0].double().cpu().numpy()
            recs.append(TraceRecord(i // nl, layer, ww, sel, sel[: self.n]))
        self._trace = None
        return RoutingTrace(records=recs)

    def bytes_per_step(self, distinct_experts: int) -> int:
        """Host-link bytes of one layer step that selects ``distinct_experts``."""
        return distinct_experts * self.block_bytes


__all__ = ["HostExpert", "OffloadEngine", "GpuPagerEngine", "host_experts_from_synth", "NAMES"]
