"""Write the toy compressed model with the REAL reference's ``save_artifact``
(build container only; needs /root/reference).

    python tests/golden/make_artifact.py

The toy model is the one of make_golden.py (seed 7, hidden 64, ffn 128, 2
layers, 8 routed + 1 shared expert, INT2 gs64 HQQ-20, rank-16 INT3 factors,
compress seed 3), so the records this artifact holds are exactly the
``toy_*`` arrays pinned in golden.npz.  Output: tests/golden/artifact_toy/
(manifest.json + blobs/), read by tests/test_artifact.py through
paper_2512_17073_b200.artifact (no reference import at test time).
"""
from __future__ import annotations

import math
import os
import shutil
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from moe_lrc import moe, quant
    from moe_lrc.artifact import load_artifact, save_artifact
    from moe_lrc.pipeline import compress_model, uniform_allocation
    from moe_lrc.ranks import kurtosis_profile

    m = moe.gen_synthetic_model(seed=7, hidden=64, ffn=128, num_layers=2, num_experts=8, top_k=2,
                                num_shared=1, tail_dofs=(4.0, math.inf), router_skew=1.4)
    prof = kurtosis_profile(m)
    cm = compress_model(m, quant.QuantConfig(bits=2, group_size=64, hqq_iters=20),
                        uniform_allocation(prof, 16), prof, seed=3)
    out = os.path.join(HERE, "artifact_toy")
    shutil.rmtree(out, ignore_errors=True)
    save_artifact(cm, out)
    back = load_artifact(out)  # the reference's own round trip
    assert sorted(back.records) == sorted(cm.records)
    print("wrote", out, len(cm.records), "records")


if __name__ == "__main__":
    main()
