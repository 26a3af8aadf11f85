"""Reference artifact format -> HBM / pinned host, without unpacking.

The reference persists a compressed model as ``manifest.json`` plus one blob per
(layer, expert, projection) (ref/artifact.py:132-197): each blob concatenates
the LSB-first packed codes (ref/quant.py:243-249), little-endian f8 scales and
zero points, and, for a compensated projection, the same three sections for
the U and V factors; the manifest carries the section offsets and a CRC32 per
blob.  ``ref/artifact.py:load_artifact`` unpacks every code into a uint8 matrix
(~2 s per Mixtral projection).  Here the packed bytes go to HBM as they are --
they are exactly the storage format of the CUDA kernels (``lrc_qmat``) -- and
the metadata is rounded to fp16, the kernels' metadata format.

Errors mirror the reference: ``ArtifactError`` (ValueError),
``ArtifactVersionError`` and ``ArtifactChecksumError`` naming the record
(ref/artifact.py:27-36, 229-262).
"""
from __future__ import annotations

import json
import zlib
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from .device import (LRCMoELayer, _Keep, _packed_to_device, build_down_tiles, build_lr_tiles,
                     build_tiles, tiles_eligible)

FORMAT_VERSION = 1  # ref/artifact.py:24
PROJ = ("w1", "w3", "w2")


class ArtifactError(ValueError):
    """Malformed or inconsistent artifact files."""


class ArtifactVersionError(ArtifactError):
    """The file was written by an unsupported format version."""


class ArtifactChecksumError(ArtifactError):
    """A blob failed its CRC32 check."""


@dataclass
class Manifest:
    root: Path
    header: dict
    records: dict = field(default_factory=dict)  # (layer, expert, proj) -> manifest record

    @property
    def hidden(self) -> int:
        return int(self.header["hidden"])

    @property
    def ffn(self) -> int:
        return int(self.header["ffn"])

    @property
    def num_experts(self) -> int:
        return int(self.header["num_experts"])

    @property
    def num_shared(self) -> int:
        return int(self.header["num_shared"])


def read_manifest(path) -> Manifest:
    """Parse and check ``manifest.json`` (ref/artifact.py:229-244)."""
    root = Path(path)
    mp = root / "manifest.json"
    if not mp.exists():
        raise ArtifactError(f"no manifest.json under {root}")
    man = json.loads(mp.read_text())
    if man.get("format_version") != FORMAT_VERSION:
        raise ArtifactVersionError(
            f"{mp}: format_version {man.get('format_version')} not supported (expected {FORMAT_VERSION})")
    if man.get("kind") != "compressed-moe":
        raise ArtifactError(f"{mp}: not a compressed artifact")
    out = Manifest(root, man["header"])
    for rec in man["records"]:
        key = (int(rec["layer"]), int(rec["expert"]), str(rec["projection"]))
        if key in out.records:
            raise ArtifactError(f"duplicate record {key}")
        out.records[key] = rec
    h = out.header
    expected = int(h["num_layers"]) * (int(h["num_experts"]) + int(h["num_shared"])) * len(PROJ)
    if len(out.records) != expected:
        raise ArtifactError(f"expected {expected} projection records, found {len(out.records)}")
    return out


@dataclass
class PackedMatrix:
    """One quantized matrix as stored: packed codes + f8 metadata."""

    rows: int
    cols: int
    bits: int
    group_size: int
    packed: bytes
    scales: np.ndarray  # (rows, groups) float64
    zeros: np.ndarray


@dataclass
class PackedRecord:
    qm: PackedMatrix
    comp_rank: int = 0
    u: PackedMatrix | None = None
    v: PackedMatrix | None = None


def read_record(man: Manifest, layer: int, expert: int, projection: str) -> PackedRecord:
    """Blob of one projection, CRC-checked, sections sliced without unpacking."""
    key = (layer, expert, projection)
    rec = man.records.get(key)
    if rec is None:
        raise ArtifactError(f"no record for layer {layer}, expert {expert}, projection {projection}")
    path = man.root / rec["blob"]
    if not path.exists():
        raise ArtifactError(f"missing blob for record {key}: {path}")
    blob = path.read_bytes()
    if zlib.crc32(blob) != int(rec["crc32"]):
        raise ArtifactChecksumError(
            f"checksum mismatch for layer {layer}, expert {expert}, projection {projection}")
    sections = rec["sections"]

    def matrix(meta: dict, prefix: str) -> PackedMatrix:
        rows, cols = int(meta["rows"]), int(meta["cols"])
        bits, gs = int(meta["bits"]), int(meta["group_size"])
        gpr = -(-cols // gs)

        def sect(name):
            off, n = sections[prefix + name]
            return blob[off:off + n]

        codes = sect("codes")
        if len(codes) != (rows * cols * bits + 7) // 8:
            raise ArtifactError(f"record {key}: {prefix}codes holds {len(codes)} bytes")
        sc = np.frombuffer(sect("scales"), dtype="<f8").reshape(rows, gpr)
        zp = np.frombuffer(sect("zero_points"), dtype="<f8").reshape(rows, gpr)
        return PackedMatrix(rows, cols, bits, gs, codes, sc, zp)

    out = PackedRecord(matrix(rec["qm"], "qm."))
    if rec.get("comp") is not None and int(rec["comp"]["rank"]) > 0:
        out.comp_rank = int(rec["comp"]["rank"])
        out.u = matrix(rec["comp"]["u"], "u.")
        out.v = matrix(rec["comp"]["v"], "v.")
    return out


def _to_device(pm: PackedMatrix, keep: _Keep) -> _lib.LrcQmat:
    return _packed_to_device(pm.packed, pm.rows, pm.cols, pm.bits, pm.group_size, pm.scales, pm.zeros, keep)


def expert_descriptor(man: Manifest, layer: int, expert: int, keep: _Keep, tiles: bool = True) -> _lib.LrcExpert:
    """An ``lrc_expert`` for one expert: codes straight to HBM, fp16 metadata,
    plus the streamed T2 / low-rank tiles when the shapes allow them."""
    ex = _lib.LrcExpert()
    rank = 0
    for proj, (un, vn) in zip(PROJ, (("u1", "v1"), ("u3", "v3"), ("u2", "v2"))):
        rec = read_record(man, layer, expert, proj)
        setattr(ex, proj, _to_device(rec.qm, keep))
        if rec.comp_rank:
            setattr(ex, un, _to_device(rec.u, keep))
            setattr(ex, vn, _to_device(rec.v, keep))
            rank = max(rank, rec.comp_rank)
    ex.rank = rank
    if tiles and tiles_eligible(ex.w1, ex.w3, ex.w2):
        ex.up_tiles = build_tiles([ex.w1, ex.w3], keep).data_ptr()
        ex.down_tiles = build_down_tiles(ex.w2, keep).data_ptr()
        if rank:
            build_lr_tiles(ex, man.hidden, man.ffn, keep)
    return ex


def load_layer(path_or_manifest, layer: int, gate: np.ndarray, max_tokens: int = 64, top_k: int = 2,
               tiles: bool = True) -> LRCMoELayer:
    """One MoE layer of a reference artifact, resident in HBM.  ``gate`` is the
    layer's router (hidden, num_experts) -- the artifact stores experts only."""
    man = path_or_manifest if isinstance(path_or_manifest, Manifest) else read_manifest(path_or_manifest)
    gate = np.asarray(gate, dtype=np.float64)
    if gate.shape != (man.hidden, man.num_experts):
        raise ArtifactError(f"gate shape {gate.shape} does not match the artifact "
                            f"({man.hidden}, {man.num_experts})")
    keep = _Keep()
    experts = [expert_descriptor(man, layer, e, keep, tiles) for e in range(man.num_experts + man.num_shared)]
    return LRCMoELayer(gate, experts, man.hidden, man.ffn, man.num_experts, man.num_shared, keep,
                       max_tokens=max_tokens, top_k=top_k)


__all__ = ["ArtifactError", "ArtifactVersionError", "ArtifactChecksumError", "Manifest", "PackedMatrix",
           "PackedRecord", "read_manifest", "read_record", "expert_descriptor", "load_layer",
           "FORMAT_VERSION"]
