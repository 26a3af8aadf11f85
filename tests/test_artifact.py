"""Reference artifact format loader.

tests/golden/artifact_toy/ was written by the REAL reference's save_artifact
(tests/golden/make_artifact.py); its records are the toy_* arrays pinned in
golden.npz.  CPU: sections are sliced without unpacking, checksums, version
and missing-blob errors behave as ref/artifact.py:229-262.  GPU: a layer loaded
straight from the artifact (packed codes to HBM) matches the oracle forward.
"""
import json
import math
import os
import shutil

import numpy as np
import pytest

from oracle import lrc
from paper_2512_17073_b200 import artifact

HERE = os.path.dirname(os.path.abspath(__file__))
ART = os.path.join(HERE, "golden", "artifact_toy")
G = np.load(os.path.join(HERE, "golden", "golden.npz"))


def test_manifest_and_records_bit_exact():
    man = artifact.read_manifest(ART)
    assert (man.hidden, man.ffn, man.num_experts, man.num_shared) == (64, 128, 8, 1)
    assert len(man.records) == 2 * 9 * 3
    for (l, e, p) in man.records:
        rec = artifact.read_record(man, l, e, p)
        base = f"toy_l{l}_e{e}_{p}"
        codes = lrc.unpack_codes(rec.qm.packed, rec.qm.rows * rec.qm.cols, rec.qm.bits)
        assert np.array_equal(codes.reshape(rec.qm.rows, rec.qm.cols), G[base + "_codes"])
        assert np.array_equal(rec.qm.scales, G[base + "_scales"])
        assert np.array_equal(rec.qm.zeros, G[base + "_zeros"])
        assert rec.comp_rank == 16
        for f in ("u", "v"):
            pm = getattr(rec, f)
            c = lrc.unpack_codes(pm.packed, pm.rows * pm.cols, pm.bits).reshape(pm.rows, pm.cols)
            assert np.array_equal(c, G[f"{base}_{f}_codes"])
            assert np.array_equal(pm.scales, G[f"{base}_{f}_scales"])


def _copy(tmp_path):
    dst = tmp_path / "art"
    shutil.copytree(ART, dst)
    return dst


def test_checksum_error_names_record(tmp_path):
    dst = _copy(tmp_path)
    blob = dst / "blobs" / "l001_e003_w2.bin"
    data = bytearray(blob.read_bytes())
    data[5] ^= 0xFF
    blob.write_bytes(bytes(data))
    man = artifact.read_manifest(dst)
    artifact.read_record(man, 0, 0, "w1")  # untouched records still load
    with pytest.raises(artifact.ArtifactChecksumError, match="layer 1, expert 3, projection w2"):
        artifact.read_record(man, 1, 3, "w2")


def test_version_kind_and_missing_blob(tmp_path):
    dst = _copy(tmp_path)
    mp = dst / "manifest.json"
    man = json.loads(mp.read_text())
    man["format_version"] = 2
    mp.write_text(json.dumps(man))
    with pytest.raises(artifact.ArtifactVersionError):
        artifact.read_manifest(dst)
    man["format_version"] = 1
    man["kind"] = "synthetic-moe"
    mp.write_text(json.dumps(man))
    with pytest.raises(artifact.ArtifactError, match="not a compressed artifact"):
        artifact.read_manifest(dst)
    man["kind"] = "compressed-moe"
    mp.write_text(json.dumps(man))
    (dst / "blobs" / "l000_e002_w3.bin").unlink()
    m = artifact.read_manifest(dst)
    with pytest.raises(artifact.ArtifactError, match="missing blob"):
        artifact.read_record(m, 0, 2, "w3")
    assert issubclass(artifact.ArtifactError, ValueError)
    with pytest.raises(artifact.ArtifactError):
        artifact.read_manifest(tmp_path / "nowhere")


@pytest.mark.gpu
def test_load_layer_forward_vs_oracle():
    import torch

    layers = lrc.gen_model(7, 64, 128, 2, 8, num_shared=1, tail_dofs=(4.0, math.inf), router_skew=1.4)
    man = artifact.read_manifest(ART)
    # oracle store from the same artifact (fp16-rounded metadata, as on device)
    st = lrc.Store()
    for (l, e, p) in man.records:
        rec = artifact.read_record(man, l, e, p)

        def qm(pm):
            c = lrc.unpack_codes(pm.packed, pm.rows * pm.cols, pm.bits).reshape(pm.rows, pm.cols)
            return lrc.QM(pm.rows, pm.cols, pm.bits, pm.group_size, c, pm.scales.copy(), pm.zeros.copy())

        st.records[(l, e, p)] = lrc.Rec(qm(rec.qm), lrc.Comp(rec.comp_rank, qm(rec.u), qm(rec.v), p))
    st16 = lrc.round_store_meta(st)
    xs = lrc.to_bf16(G["toy_x"])
    for l in range(2):
        dl = artifact.load_layer(man, l, layers[l].gate, max_tokens=16, top_k=2)
        assert dl.tiled
        y, _, _ = dl.forward(torch.from_numpy(xs).cuda().to(torch.bfloat16), 2, 1)
        y = y.double().cpu().numpy()
        for t in range(len(xs)):
            yo = lrc.forward(xs[t], layers[l].gate, None, 2, 1, "compensated", st16, l, shared=layers[l].shared)
            err = np.linalg.norm(y[t] - yo) / np.linalg.norm(yo)
            assert err <= 1e-2, (l, t, err)
    with pytest.raises(artifact.ArtifactError, match="gate shape"):
        artifact.load_layer(man, 0, np.zeros((64, 7)))
