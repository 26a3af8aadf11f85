"""Expert-parallel MoE layer (north-star item 5).

Experts are sharded across the ranks of a ``torch.distributed`` group: routed
expert e lives on rank ``e * G // E``; shared experts are replicated and run on
the token's own rank.  One step for a rank's local batch x (B, d):

1. route locally (fp64 gate, stable top-k, top-n flags: ref/moe.py:165-193);
2. dispatch: every (token, selected expert) pair is sent to the expert's owner
   in fixed-capacity blocks (no host synchronisation, graph-capturable) -- one
   all-to-all of the token rows and one of the packed (expert, weight,
   compensated) metadata;
3. the owner runs ``lrc_layer_forward_pairs`` on what it received: one launch
   sequence over its local experts, U.(V.x) applied for the flagged pairs;
4. combine: the weighted rows go back with the reverse all-to-all and are summed
   per token (ref/moe.py:237-258), plus the local shared experts.

Collectives are NCCL over NVLink/NVSwitch on the GPU path and gloo in the CPU
tests (``route_fn`` / ``compute_fn`` let the tests inject the oracle; the
defaults are the CUDA library and fail loudly without it).
"""
from __future__ import annotations

import ctypes

from . import _lib


def owner_of(expert, num_experts: int, world: int):
    """Rank owning routed expert ``expert`` (tensor or int): floor(e * G / E)."""
    return (expert * world) // num_experts


class ExpertParallelLayer:
    """One MoE layer sharded over ``group``; see the module docstring."""

    def __init__(self, group, num_experts: int, num_shared: int, top_k: int, top_n: int,
                 route_fn, compute_fn, compensate_shared: bool = True, comm_device=None,
                 max_tokens: int = 64):
        import torch.distributed as dist

        self.comm_device = comm_device  # None: collectives on x's device (NCCL); "cpu" for gloo
        self.max_tokens = int(max_tokens)  # per rank and step; the same on every rank
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if num_experts < self.world:
            raise ValueError("expert parallelism needs at least one routed expert per rank")
        self.E, self.S, self.k, self.n = num_experts, num_shared, top_k, top_n
        self.route_fn, self.compute_fn = route_fn, compute_fn
        self.compensate_shared = compensate_shared

    def local_experts(self):
        return [e for e in range(self.E) if owner_of(e, self.E, self.world) == self.rank]

    # ---------------------------------------------------------------- step --
    def first_expert(self, r: int) -> int:
        """Lowest routed expert id owned by rank r: ceil(r E / G)."""
        return -(-r * self.E // self.world)

    def forward(self, x):
        """x (B, d) on this rank's device -> y (B, d) float32 (sum over the
        token's experts, as ref/moe.py:forward in mode "compensated").

        No host synchronisation and static shapes (graph-capturable): every
        rank sends a fixed-capacity block of C = max_tokens k rows to every
        rank (the worst case, so nothing is ever dropped; max_tokens is the
        same on every rank, the local batches B <= max_tokens may differ).  A (token, expert) pair's slot
        in its owner's block is its rank among the pairs with the same owner
        (a one-hot cumulative sum); unused slots carry a zero row for the
        receiver's first expert with weight 0, which adds nothing (and only
        keeps an expert busy on a rank that would otherwise idle)."""
        import torch
        import torch.distributed as dist

        B, d = int(x.shape[0]), int(x.shape[1])
        dev = x.device
        W = self.world
        idx, w = self.route_fn(x)                      # (B, k) int, (B, k) float
        k = int(idx.shape[1])
        if B > self.max_tokens:
            raise ValueError(f"EP forward: {B} tokens above max_tokens={self.max_tokens}")
        C = self.max_tokens * k
        if x.is_cuda and x.dtype == torch.bfloat16 and self.comm_device is None:
            return self._forward_cuda(x, idx, w, B, d, k, C)
        idx = idx.to(dev, torch.int64)
        w = w.to(dev, torch.float32)
        token = torch.arange(B, device=dev).repeat_interleave(k)
        expert = idx.reshape(-1)
        weight = w.reshape(-1)
        comp = (torch.arange(k, device=dev) < self.n).repeat(B).to(torch.int32)
        dest = owner_of(expert, self.E, W)
        ranks = torch.arange(W, device=dev)
        onehot = (dest[:, None] == ranks[None, :]).to(torch.int32)  # (no one_hot: it validates on the host)
        pos = (onehot.cumsum(0) * onehot).sum(1) - 1
        slot = dest * C + pos
        first = (-(-ranks * self.E // W)).to(torch.int32)  # ceil(r E / G), computed on the device
        meta = torch.zeros((W * C, 3), dtype=torch.int32, device=dev)
        meta[:, 0] = first.repeat_interleave(C)
        meta[slot, 0] = expert.to(torch.int32)
        meta[slot, 1] = weight.view(torch.int32)
        meta[slot, 2] = comp
        src = torch.full((W * C,), B, dtype=torch.int64, device=dev)  # dummy slots -> row B
        src[slot] = token
        x_send = torch.zeros((W * C, d), dtype=x.dtype, device=dev)
        x_send[slot] = x[token]
        cdev = self.comm_device or dev
        x_recv = torch.empty((W * C, d), dtype=x.dtype, device=cdev)
        meta_recv = torch.empty((W * C, 3), dtype=torch.int32, device=cdev)
        dist.all_to_all_single(x_recv, x_send.to(cdev), group=self.group)
        dist.all_to_all_single(meta_recv, meta.to(cdev), group=self.group)
        x_recv, meta_recv = x_recv.to(dev), meta_recv.to(dev)
        y_rows = self.compute_fn(x_recv, meta_recv[:, 0].contiguous(),
                                 meta_recv[:, 1].contiguous().view(torch.float32),
                                 meta_recv[:, 2].contiguous().to(torch.uint8))
        y_rows = y_rows.to(torch.float32).contiguous()
        y_back = torch.empty((W * C, d), dtype=torch.float32, device=cdev)
        dist.all_to_all_single(y_back, y_rows.to(cdev), group=self.group)
        y = torch.zeros((B + 1, d), dtype=torch.float32, device=dev)
        y.index_add_(0, src, y_back.to(dev))
        y = y[:B]
        if self.S:  # shared experts: replicated, computed on the token's own rank
            xs = x.repeat(self.S, 1)
            ex = torch.arange(self.E, self.E + self.S, device=dev).repeat_interleave(B).to(torch.int32)
            ws = torch.ones(B * self.S, dtype=torch.float32, device=dev)
            cs = torch.full((B * self.S,), int(self.compensate_shared), dtype=torch.uint8, device=dev)
            ys = self.compute_fn(xs, ex, ws, cs).to(torch.float32)
            y = y + ys.reshape(self.S, B, d).sum(0)
        return y


def _shared_rows(self, x, y, B, d):
    import torch

    dev = x.device
    xs = x.repeat(self.S, 1)
    ex = torch.arange(self.E, self.E + self.S, device=dev).repeat_interleave(B).to(torch.int32)
    ws = torch.ones(B * self.S, dtype=torch.float32, device=dev)
    cs = torch.full((B * self.S,), int(self.compensate_shared), dtype=torch.uint8, device=dev)
    ys = self.compute_fn(xs, ex, ws, cs).to(torch.float32)
    return y + ys.reshape(self.S, B, d).sum(0)


def _forward_cuda(self, x, idx, w, B, d, k, C):
    """The same exchange with the dispatch and the combine as one CUDA kernel
    each (lrc_ep_dispatch / lrc_ep_combine): route, dispatch, 2 all-to-alls,
    the owner's forward_pairs, 1 all-to-all back, combine."""
    import torch
    import torch.distributed as dist

    W = self.world
    lib = _lib.lib()
    idx = idx.to(torch.int32).contiguous()
    w = w.to(torch.float32).contiguous()
    x = x.contiguous()
    x_send = torch.empty((W * C, d), dtype=torch.bfloat16, device=x.device)
    meta = torch.empty((W * C, 3), dtype=torch.int32, device=x.device)
    slot_of = torch.empty((B * k,), dtype=torch.int32, device=x.device)
    _lib.check(lib.lrc_ep_dispatch(_lib.ptr(idx), _lib.ptr(w), _lib.ptr(x), B, k, self.n, self.E, W, C, d,
                                   _lib.ptr(x_send), _lib.ptr(meta), _lib.ptr(slot_of), _lib.stream_ptr()))
    x_recv = torch.empty_like(x_send)
    meta_recv = torch.empty_like(meta)
    dist.all_to_all_single(x_recv, x_send, group=self.group)
    dist.all_to_all_single(meta_recv, meta, group=self.group)
    y_rows = self.compute_fn(x_recv, meta_recv[:, 0].contiguous(),
                             meta_recv[:, 1].contiguous().view(torch.float32),
                             meta_recv[:, 2].contiguous().to(torch.uint8))
    y_back = torch.empty_like(y_rows)
    dist.all_to_all_single(y_back, y_rows.contiguous(), group=self.group)
    y = torch.empty((B, d), dtype=torch.float32, device=x.device)
    _lib.check(lib.lrc_ep_combine(_lib.ptr(y_back), _lib.ptr(slot_of), B, k, d, _lib.ptr(y), _lib.stream_ptr()))
    if self.S:
        y = _shared_rows(self, x, y, B, d)
    return y


ExpertParallelLayer._forward_cuda = _forward_cuda


def cuda_route_fn(dl, top_k: int, top_n: int, renormalize: bool = False):
    """Routing of a rank's local tokens on the GPU (lrc_route, bit-exact fp64)."""
    torch = _lib.device_required()

    def route(x):
        B = int(x.shape[0])
        idx = torch.empty((B, top_k), dtype=torch.int32, device="cuda")
        w = torch.empty((B, top_k), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().lrc_route(_lib.ptr(dl.gate_t), _lib.ptr(x.contiguous()), _lib.DTYPE_BF16, B,
                                        dl.hidden, dl.num_experts, top_k, top_n, int(bool(renormalize)),
                                        ctypes.c_void_p(0), _lib.ptr(idx), _lib.ptr(w), _lib.stream_ptr()))
        return idx, w

    return route


def from_device_layer(group, dl, top_k: int, top_n: int, renormalize: bool = False,
                      compensate_shared: bool = True, comm_device=None,
                      max_tokens: int = 64) -> ExpertParallelLayer:
    """EP layer over a rank-local ``LRCMoELayer`` that holds (at least) the
    experts this rank owns plus the shared experts (absent experts may be
    None records: they share one placeholder)."""
    return ExpertParallelLayer(group, dl.num_experts, dl.num_shared, top_k, top_n,
                               cuda_route_fn(dl, top_k, top_n, renormalize),
                               lambda xr, e, w, c: dl.forward_pairs(xr, e, w, c, validate=False),
                               compensate_shared, comm_device, max_tokens)


def owned_records(records, num_experts: int, world: int, rank: int):
    """Records list with the experts of other ranks replaced by None (shared
    experts, at index >= num_experts, are kept on every rank)."""
    return [r if (i >= num_experts or owner_of(i, num_experts, world) == rank) else None
            for i, r in enumerate(records)]


__all__ = ["ExpertParallelLayer", "owner_of", "from_device_layer", "owned_records", "cuda_route_fn"]
