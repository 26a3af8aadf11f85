"""C4 prefill timing: one Mixtral-shaped layer (d=4096, ffn=14336, 8 experts
top-2, INT2 + r32) over B tokens through lrc_layer_forward, top_n sweep, on the
tcgen05 path (and optionally the mma.sync decode path for comparison).

  python tools/prefill_bench.py [--B 16384] [--iters 5] [--decode-too]
Prints one JSON line per (path, top_n): ms per layer, TFLOP/s (SURVEY 8(d)
flop formula), fraction of MEASURED_PEAKS bf16.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_17073_b200.synth import SynthLayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=16384)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--rank", type=int, default=32)
    ap.add_argument("--decode-too", action="store_true")
    ap.add_argument("--phases", action="store_true")
    ap.add_argument("--n", type=int, nargs="*", default=[0, 1, 2], help="top_n values to run")
    args = ap.parse_args()
    d, ffn, E, k, r = 4096, 14336, 8, 2, args.rank
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    peak = float(peaks.get("bf16_tflops", 1644.4))
    sl = SynthLayer(d, ffn, E, top_k=k, rank=r, seed=0, max_tokens=args.B)
    x = torch.randn((args.B, d), device="cuda").to(torch.bfloat16)
    y = torch.empty((args.B, d), device="cuda", dtype=torch.float32)
    paths = [("tcgen05", 1)] + ([("mma.sync", 0)] if args.decode_too else [])
    for name, pmin in paths:
        sl.layer.set_prefill_min(pmin)
        for n in args.n:
            for _ in range(2):
                sl.layer.forward(x, top_k=k, top_n=n, y=y)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            for _ in range(args.iters):
                sl.layer.forward(x, top_k=k, top_n=n, y=y)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1]) / args.iters
            flops = args.B * (k * 2 * 3 * d * ffn + n * 3 * 2 * r * (d + ffn) + 2 * d * E)
            tf = flops / ms / 1e9
            rec = {"path": name, "B": args.B, "top_n": n, "ms": round(ms, 3), "tflops": round(tf, 1),
                   "frac_bf16_peak": round(tf / peak, 3), "launches": sl.layer.last_launches()}
            if args.phases:
                sl.layer.set_profiling(True)
                sl.layer.forward(x, top_k=k, top_n=n, y=y)
                torch.cuda.synchronize()
                rec["phase_ms"] = [round(v, 3) for v in sl.layer.phase_ms()]
                sl.layer.set_profiling(False)
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
