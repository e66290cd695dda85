"""Host-side logic of the product package (no GPU): config validation, the
numpy codebook restatement against the reference's tables, the rotation table
identity used by the encode kernel, and kvpack header validation."""

import os
import struct
import zlib

import numpy as np
import pytest

from conftest import GOLDEN, load_codec_fixture

import paper_2605_27646_b200 as m
from paper_2605_27646_b200 import codebook as cb


def test_config_validation_and_bits():
    cfg = m.CodecConfig(codebook_size=96, radius_bits=4)
    assert cfg.index_count == 2304 and cfg.index_bits == 12
    assert m.CodecConfig(16, 4).index_bits == 9
    assert m.CodecConfig(64, 4).index_bits == 11
    assert m.CodecConfig(256, 4).index_bits == 13
    for bad in (dict(codebook_size=0, radius_bits=4), dict(codebook_size=24, radius_bits=9),
                dict(codebook_size=24, radius_bits=4, seed=-1),
                dict(codebook_size=24, radius_bits=4, outlier_multiplier=0.0),
                dict(codebook_size=24, radius_bits=4, median_pooling="global")):
        with pytest.raises(m.InvalidArgument):
            m.CodecConfig(**bad)


def test_shape_properties():
    s = m.TensorShape(2, 4, 16, 126)
    assert s.chunks_per_vector == 32 and s.padded_dim == 128
    assert s.n_chunks == 2 * 4 * 16 * 32
    with pytest.raises(m.InvalidArgument):
        m.TensorShape(0, 1, 1, 4)
    with pytest.raises(m.InvalidArgument):
        m.TensorShape(1, 1, -1, 4)
    assert m.TensorShape(1, 1, 0, 4).elements == 0


def test_attention_config():
    with pytest.raises(m.InvalidArgument):
        m.AttentionConfig(1, 3, 2, 8, 8, 16)
    with pytest.raises(m.InvalidArgument):
        m.AttentionConfig(1, 2, 2, 16, 8, 16)
    cfg = m.AttentionConfig(1, 8, 2, 8, 8, 64)
    assert cfg.group_size == 4 and cfg.logit_scale == pytest.approx(0.125)


def test_codebooks_bitwise_equal_reference():
    z = np.load(os.path.join(GOLDEN, "codebooks.npz"))
    for key in z.files:
        seed, layer, head, role, size = key.split("_")
        bank = m.CodebookBank(int(seed), int(size))
        assert np.array_equal(bank.joint(int(layer), int(head), role).codewords, z[key]), key


def test_codebook_nesting_and_validation():
    small = cb.build_secondary(7, 0, 0, "K", 96)
    large = cb.build_secondary(7, 0, 0, "K", 192)
    assert np.array_equal(small.entries, large.entries[:96])
    with pytest.raises(m.InvalidArgument):
        cb.build_secondary(0, 0, 0, "Q", 8)
    with pytest.raises(m.InvalidArgument):
        cb.build_secondary(0, -1, 0, "K", 8)


def test_rotation_table_identity():
    """The encode kernel's float2 FMA chains compute u (x) conj(s) and the
    closed-form coset score equals the max over the 24 joint codewords."""
    sec = cb.build_secondary(0, 1, 2, "V", 32).entries
    rot = cb.rotation_table(sec).astype(np.float64)
    rs = np.random.default_rng(0)
    u = rs.standard_normal((50, 4))
    u /= np.linalg.norm(u, axis=1)[:, None]
    a, b, c, d = u.T
    for s in range(32):
        t = rot[s]
        wx = (a[:, None] * t[0:2] + b[:, None] * t[2:4] + c[:, None] * t[4:6] + d[:, None] * t[6:8])
        yz = (a[:, None] * t[8:10] + b[:, None] * t[10:12] + c[:, None] * t[12:14]
              + d[:, None] * t[14:16])
        v = np.concatenate([wx, yz], axis=1)
        conj = sec[s] * np.array([1, -1, -1, -1])
        expect = cb.hamilton(u, conj)
        assert np.allclose(v, expect, atol=1e-6)
        joint = cb.hamilton(cb.primary_entries(), sec[s][None, :])
        best = (u @ joint.T).max(axis=1)
        av = np.abs(v)
        closed = np.maximum(av.max(axis=1), av.sum(axis=1) / 2)
        assert np.allclose(best, closed, atol=1e-6)


def test_kvpack_header_validation_before_upload():
    """Corruptions detectable from the header raise CorruptData / UnsupportedVersion
    without a device (the CRC itself is checked on the GPU: test_gpu_parity)."""
    meta, g = load_codec_fixture("frozen")
    blob = g["blob"].tobytes()
    with pytest.raises(m.CorruptData):
        m.from_bytes(blob[:100])
    bad = bytearray(blob)
    bad[0] ^= 1
    with pytest.raises(m.CorruptData):
        m.from_bytes(bytes(bad))
    bad = bytearray(blob)
    struct.pack_into("<H", bad, 4, 2)
    bad[-4:] = struct.pack("<I", zlib.crc32(bytes(bad[:-4])) & 0xFFFFFFFF)
    with pytest.raises(m.UnsupportedVersion):
        m.from_bytes(bytes(bad))


def test_raw_tensor_round_trip_and_validation(tmp_path):
    """KVRW raw files (kvpack.py:309-347): host-side format, same checks."""
    import numpy as np

    x = np.arange(2 * 3 * 4 * 8, dtype=np.float32).reshape(2, 3, 4, 8) / 7.0
    p = tmp_path / "x.raw"
    n = m.write_raw(x, p)
    assert n == struct.calcsize("<4sBIIII") + x.nbytes
    np.testing.assert_array_equal(m.read_raw(p), x)
    m.write_raw(x, p, dtype="f16")
    np.testing.assert_array_equal(m.read_raw(p), x.astype(np.float16))
    with pytest.raises(m.InvalidArgument):
        m.write_raw(x, p, dtype="f64")
    with pytest.raises(m.InvalidArgument):
        m.write_raw(x[0], p)
    blob = bytearray(p.read_bytes())
    blob[0] ^= 1
    p.write_bytes(bytes(blob))
    with pytest.raises(m.CorruptData):
        m.read_raw(p)
    p.write_bytes(bytes(blob[:10]))
    with pytest.raises(m.CorruptData):
        m.read_raw(p)


def test_cli_parser_matches_reference_options():
    from paper_2605_27646_b200 import cli

    a = cli.build_parser().parse_args(["quantize", "i", "o", "--S", "64", "--br", "4", "--outlier-c",
                                       "3", "--per-head-median", "--role", "V", "--layer", "5",
                                       "--head", "2"])
    assert (a.S, a.br, a.outlier_c, a.per_head_median, a.role, a.layer, a.head) == (
        64, 4, 3.0, True, "V", 5, 2)
    a = cli.build_parser().parse_args(["dequantize", "i", "o", "--dtype", "f16"])
    assert a.dtype == "f16"
    with pytest.raises(SystemExit):
        cli.build_parser().parse_args(["quantize", "i", "o"])
