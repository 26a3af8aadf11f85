"""CPU-side tests: the C-ABI library loads and exports every declared symbol,
host logic (configs, byte accounting, generators, traces) matches the reference."""

import hashlib
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def header_functions():
    src = open(os.path.join(ROOT, "include", "lrc.h")).read()
    return sorted(set(re.findall(r"^\s*(?:lrc_status|int64_t|int|void|const char\*)\s+(lrc_\w+)\(",
                                 src, re.M)))


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2512_17073_b200 import _lib

    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.EXPORTED, n
    assert lib.lrc_abi_version() == 1
    # struct layout agrees with the header (ctypes mirrors the C ABI)
    assert ctypes.sizeof(_lib.LrcQmat) == 48
    assert ctypes.sizeof(_lib.LrcExpert) == 3 * 48 + 8 + 6 * 48 + 32


def test_library_is_sm100a():
    import subprocess

    from paper_2512_17073_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_byte_accounting_c1():
    """Acceptance c1 (ref tests/test_acceptance.py:40-54) + SURVEY 8(d) roofline bytes."""
    from paper_2512_17073_b200 import lowrank, quant

    assert 3 * quant.packed_size_bytes(4096, 14336, 2) == 44_040_192
    r16 = 3 * lowrank.compensator_size_bytes(4096, 14336, 16)
    assert r16 == 331_776 and round(r16 / 2**20, 3) == 0.316
    r128 = 3 * lowrank.compensator_size_bytes(4096, 14336, 128)
    assert r128 == 2_654_208 and round(r128 / 2**20, 2) == 2.53
    assert 3 * quant.packed_size_bytes(4096, 14336, 2, include_metadata=True) == 55_050_240
    assert 3 * quant.packed_size_bytes(4096, 14336, 3, include_metadata=True) == 77_070_336
    assert quant.packed_size_bytes(4, 128, 2, include_metadata=True) == (4 * 128 * 2 + 7) // 8 + 32
    with pytest.raises(quant.QuantizationError):
        quant.packed_size_bytes(0, 4, 2)
    with pytest.raises(lowrank.CompensatorError):
        lowrank.compensator_size_bytes(-1, 4, 2)


def test_roofline_bytes_formula():
    import bench

    b = bench.layer_bytes(hidden=4096, ffn=14336, bits=2, rank=32, d_sel=2, d_comp=1, B=1, E=8)
    assert abs(b / 1e6 - 111.09) < 0.01  # C2 INT2 B=1 = 111.09 MB
    assert bench.comp_bytes(4096, 14336, 32) == 839_680
    f = bench.layer_flops(4096, 14336, 2, 1, 32, 8)
    assert abs(f / 1e6 - 708.2) < 0.5  # 708.2 MFLOP per token


def test_configs_validate():
    from paper_2512_17073_b200 import moe, quant

    with pytest.raises(quant.QuantizationError):
        quant.QuantConfig(bits=5)
    with pytest.raises(quant.QuantizationError):
        quant.QuantConfig(bits=2, group_size=0)
    with pytest.raises(quant.QuantizationError):
        quant.QuantConfig(hqq_shrink_p=0.0)
    with pytest.raises(moe.MoEError):
        moe.ForwardConfig(top_k=1, top_n=2)
    with pytest.raises(moe.MoEError):
        moe.ForwardConfig(top_k=-1)
    assert issubclass(moe.MissingArtifactError, KeyError)
    assert issubclass(quant.QuantizationError, ValueError)


def test_generator_bit_exact_with_reference():
    from paper_2512_17073_b200 import moe

    m = moe.gen_synthetic_model(seed=7, hidden=64, ffn=128, num_layers=2, num_experts=8,
                                top_k=2, num_shared=1, tail_dofs=(4.0, math.inf), router_skew=1.4)
    assert [sha(m.layers[0].gate), sha(m.layers[1].experts[3].w2),
            sha(m.layers[1].shared_experts[0].w1)] == list(G["toy_sha"])
    with pytest.raises(moe.MoEError):
        moe.gen_synthetic_model(seed=0, hidden=4, ffn=4, num_layers=1, num_experts=2,
                                tail_dofs=(2.0,))
    np.testing.assert_array_equal(moe.gen_tokens(11, 64, 6), G["toy_x"])


def test_trace_jsonl_round_trip(tmp_path):
    from paper_2512_17073_b200 import moe

    recs = [moe.TraceRecord(t, l, np.random.default_rng(t).random(4), [1, 2], [1])
            for t in range(3) for l in range(2)]
    tr = moe.RoutingTrace(recs)
    tr.to_jsonl(tmp_path / "t.jsonl")
    back = moe.RoutingTrace.from_jsonl(tmp_path / "t.jsonl")
    assert len(back.records) == 6 and back.num_tokens() == 3 and back.num_layers() == 2
    for a, b in zip(recs, back.records):
        np.testing.assert_array_equal(a.scores, b.scores)
        assert a.selected == b.selected
    with pytest.raises(moe.MoEError):
        moe.routing_stats(moe.RoutingTrace([]))


def test_no_cpu_fallback_without_device():
    """The product refuses to compute without CUDA instead of silently using the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_2512_17073_b200 import quant

    with pytest.raises(RuntimeError):
        quant.dequantize(quant.QuantizedMatrix(1, 4, 2, 64, np.zeros((1, 4), np.uint8),
                                               np.ones((1, 1)), np.zeros((1, 1))))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2512_17073_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith(".py") and f != "synth.py":
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_fp16_metadata_range_check():
    """Artifact metadata that does not fit the kernels' fp16 format raises
    (overflow -> inf, nonzero scales flushing to 0)."""
    from paper_2512_17073_b200.artifact import ArtifactError
    from paper_2512_17073_b200.device import _fp16_meta

    assert _fp16_meta([0.01, 0.0, 1e-6], "scale").dtype == np.float16
    assert _fp16_meta([1e-9, -3.0], "zero point")[0] == 0.0  # tiny zero points: < 3e-8 absolute error
    for bad in ([7e4], [1e-9], [float("nan")]):
        with pytest.raises(ArtifactError):
            _fp16_meta(bad, "scale")
    with pytest.raises(ArtifactError):
        _fp16_meta([-1e5], "zero point")


def test_tiled_core_digit_arithmetic():
    """The integer arithmetic of the tiled decode core (csrc/tiled.cu), restated
    in numpy: per (token, 64-column group) X = rint(x 2^S) with S = 138 - E
    (E = exponent field of max|x|), digits d0 = X >> 7, d1 = X & 127 fit s8;
    the u8 x s8 sums of 2-bit codes (x1 row, x4 row) stay inside the exact
    window of the 1.5 * 2^23 magic float; and the group dot product is within
    2^-12 max|x| sum(c) of the exact one (each x moves by at most half a unit
    2^-S <= 2^-12 max|x|)."""
    rng = np.random.default_rng(3)
    magic = np.float32(12582912.0)
    for scale in (1e-30, 1e-3, 1.0, 7.5, 3e4):
        x = (rng.standard_normal((256, 64)) * scale).astype(np.float32)
        x[0] = 0.0
        x[1, :] = scale  # all equal: the rounding edge |X| = 2^12
        amax = np.abs(x).max(axis=1)
        E = (amax.view(np.uint32) >> 23) & 255
        S = np.minimum(138 - E.astype(np.int64), 126)
        X = np.rint(x.astype(np.float64) * np.exp2(S)[:, None]).astype(np.int64)
        assert np.abs(X).max() <= 4096
        d0, d1 = X >> 7, X & 127
        assert d0.min() >= -128 and d0.max() <= 127 and d1.min() >= 0 and d1.max() <= 127
        assert np.array_equal(128 * d0 + d1, X)
        c = rng.integers(0, 4, size=(256, 64))
        for mult in (1, 4):  # row gid codes x1, row gid+8 codes x4
            v = 128 * (mult * c * d0).sum(axis=1) + (mult * c * d1).sum(axis=1)
            assert np.abs(v).max() < 2 ** 22
            f = (np.full(256, magic).view(np.int32) + v.astype(np.int32)).view(np.float32)
            inv = np.exp2(-S).astype(np.float32) / mult
            t = (f.astype(np.float64) * inv - magic.astype(np.float64) * inv)
            exact = (c * X).sum(axis=1) * np.exp2(-S)
            assert np.array_equal(t, exact)  # the magic float holds the dot product exactly
            err = np.abs(exact - (c * x.astype(np.float64)).sum(axis=1))
            bound = 0.5 * np.exp2(-S) * c.sum(axis=1)
            assert np.all(err <= bound + 1e-300)
            live = amax > 0  # an all-zero group is exact (X = 0)
            assert np.all(err[~live] == 0)
            assert np.all(bound[live] <= np.exp2(-12) * amax[live] * c.sum(axis=1)[live])
