"""A few decode tokens of a 4-layer C3-shaped chain through the GPU pager, for
ncu host-link counters on pager_kernel (profiles/r2_offload_ncu.md):

    ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,... -k regex:pager_kernel python tools/offload_ncu.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_17073_b200 import _lib, offload  # noqa: E402
from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402


def main():
    _lib.load()
    gates, host = [], []
    for l in range(4):
        sl = SynthLayer(4096, 14336, 8, top_k=2, bits=2, rank=32, seed=900 + l, max_tokens=8)
        gates.append(sl.gate)
        host.append(offload.host_experts_from_synth(sl))
        del sl
        torch.cuda.empty_cache()
    eng = offload.GpuPagerEngine(gates, host, 4096, 14336, top_k=2, top_n=1, max_tokens=1)
    x = torch.randn((1, 4096), device="cuda").to(torch.bfloat16)
    for _ in range(3):
        x = eng.forward(x, normalize=True)
    torch.cuda.synchronize()
    print("block bytes", eng.block_bytes, flush=True)


if __name__ == "__main__":
    main()
