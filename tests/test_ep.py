"""Expert-parallel layer.

CPU: world_size 2 over gloo -- the dispatch / combine logic of
``ep.ExpertParallelLayer`` with the oracle injected as the router and the
per-row expert compute, checked against the oracle's single-rank forward.
GPU: ``lrc_layer_forward_pairs`` (the owner-side compute) reproduces the
routed layer forward, and the EP layer over a 1-rank NCCL group matches it.
"""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import lrc as O
from paper_2512_17073_b200 import ep

HID, FFN, E, S, K, N = 64, 96, 4, 1, 2, 1


def _model():
    layers = O.gen_model(3, HID, FFN, 1, E, num_shared=S, router_skew=1.4)
    store = O.compress(layers, bits=2, group_size=64, hqq_iters=0, rank=4, factor_bits=3, seed=0)
    return layers[0], store


def _oracle_fns(layer, store):
    cache = {}

    def route(x):
        idx, w = [], []
        for row in x.double().numpy():
            wts, sel, _ = O.route(row, layer.gate, K, N)
            idx.append(sel)
            w.append(wts[sel])
        return torch.tensor(idx), torch.tensor(np.array(w), dtype=torch.float32)

    def compute(xr, e, w, c):
        out = np.zeros((xr.shape[0], HID))
        for i in range(xr.shape[0]):
            key = (int(e[i]), bool(c[i]))
            if key not in cache:
                cache[key] = O.resolve(store, 0, key[0], key[1])
            out[i] = float(w[i]) * O.expert_forward(*cache[key], xr[i].double().numpy())
        return torch.from_numpy(out).float()

    return route, compute


def _worker(rank, world, port, result_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layer, store = _model()
        route, compute = _oracle_fns(layer, store)
        # each rank routes its own tokens; compute only ever sees this rank's experts
        def guarded(xr, e, w, c):
            for ei in e.tolist():
                assert ei >= E or ep.owner_of(ei, E, world) == rank, "row dispatched to a non-owner"
            return compute(xr, e, w, c)

        layer_ep = ep.ExpertParallelLayer(dist.group.WORLD, E, S, K, N, route, guarded, max_tokens=8)
        x = torch.from_numpy(O.to_bf16(O.gen_tokens(10 + rank, HID, 5 + rank))).double()
        y = layer_ep.forward(x).double().numpy()
        worst = 0.0
        for b in range(x.shape[0]):
            ref = O.forward(x[b].numpy(), layer.gate, None, K, N, "compensated", store, 0,
                            shared=[None] * S)
            worst = max(worst, float(np.linalg.norm(y[b] - ref) / np.linalg.norm(ref)))
        with open(f"{result_path}.{rank}", "w") as f:
            f.write(repr(worst))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_owner_partition():
    for world in (1, 2, 4, 8):
        owners = [ep.owner_of(e, 8, world) for e in range(8)]
        assert owners == sorted(owners) and set(owners) == set(range(world))
    recs = list(range(E + S))
    kept = ep.owned_records(recs, E, 2, 1)
    assert kept == [None, None, 2, 3, 4]


def test_ep_gloo_world2(tmp_path):
    import torch.multiprocessing as mp

    res = str(tmp_path / "worst")
    mp.spawn(_worker, args=(2, _free_port(), res), nprocs=2, join=True)
    for r in range(2):
        worst = float(open(f"{res}.{r}").read())
        assert worst < 1e-5, f"rank {r}: EP output differs from the oracle ({worst:.2e})"


@pytest.mark.gpu
def test_forward_pairs_matches_layer_forward():
    from paper_2512_17073_b200.synth import SynthLayer

    sl = SynthLayer(512, 1024, 8, top_k=2, rank=16, seed=5, max_tokens=64)
    B = 6
    x = torch.randn((B, 512), device="cuda").to(torch.bfloat16)
    y_ref, idx, w = sl.layer.forward(x, 2, 1)
    # the same routing as explicit (token, expert) pairs, top-1 compensated
    rows = x.repeat_interleave(2, dim=0)
    comp = torch.tensor([1, 0] * B, dtype=torch.uint8, device="cuda")
    yp = sl.layer.forward_pairs(rows, idx.reshape(-1), w.reshape(-1), comp)
    y = yp.reshape(B, 2, -1).sum(1)
    err = (y - y_ref).norm() / y_ref.norm()
    assert err < 1e-5, float(err)


@pytest.mark.gpu
def test_ep_single_rank_nccl():
    import torch.distributed as dist
    from paper_2512_17073_b200.synth import SynthLayer

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        sl = SynthLayer(512, 1024, 8, top_k=2, rank=16, seed=6, max_tokens=64)
        layer_ep = ep.from_device_layer(dist.group.WORLD, sl.layer, 2, 1, max_tokens=8)
        x = torch.randn((5, 512), device="cuda").to(torch.bfloat16)
        y = layer_ep.forward(x)
        y_ref, _, _ = sl.layer.forward(x, 2, 1)
        err = (y - y_ref).norm() / y_ref.norm()
        assert err < 1e-5, float(err)
    finally:
        dist.destroy_process_group()


def _gpu_worker(rank, world, port, result_path):
    """One rank of a world-2 EP layer on the SAME GPU: the CUDA router and
    ``forward_pairs`` compute, the all-to-alls over gloo on host copies."""
    import torch.distributed as dist
    from paper_2512_17073_b200 import _lib
    from paper_2512_17073_b200.synth import SynthLayer

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _lib.load()
        sl = SynthLayer(512, 1024, 8, top_k=2, num_shared=1, rank=16, seed=8, max_tokens=64)
        dl = sl.layer
        layer_ep = ep.from_device_layer(dist.group.WORLD, dl, 2, 1, comm_device="cpu", max_tokens=8)
        owned = set(layer_ep.local_experts())

        def guarded(xr, e, w, c):  # every row this rank computes belongs to one of its experts
            bad = [int(v) for v in e.cpu().tolist() if v < 8 and int(v) not in owned]
            assert not bad, f"rows of experts {bad} dispatched to rank {rank}"
            return dl.forward_pairs(xr, e, w, c, validate=False)

        layer_ep.compute_fn = guarded
        g = torch.Generator(device="cuda").manual_seed(100 + rank)
        x = torch.randn((5 + rank, 512), device="cuda", generator=g).to(torch.bfloat16)
        y = layer_ep.forward(x)
        y_ref, _, _ = dl.forward(x, 2, 1)
        err = float((y - y_ref).norm() / y_ref.norm())
        with open(f"{result_path}.{rank}", "w") as f:
            f.write(repr(err))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_ep_world2_cuda_compute(tmp_path):
    """World-size-2 EP with the CUDA owner-side compute (forward_pairs) and the
    CUDA router on both ranks vs the single-GPU routed layer forward."""
    import torch.multiprocessing as mp

    res = str(tmp_path / "err")
    mp.spawn(_gpu_worker, args=(2, _free_port(), res), nprocs=2, join=True)
    for r in range(2):
        err = float(open(f"{res}.{r}").read())
        assert err < 1e-5, f"rank {r}: EP output differs from the layer forward ({err:.2e})"
