"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python oracle/build.py          # installs the reference into oracle/_ref
    python tests/golden/make_golden.py

The reference package (hqmq, built unmodified from /root/reference/pkg) is
imported from oracle/_ref; every fixture records inputs and the reference's
outputs, so the GPU box (which has no /root/reference) can check both the
oracle restatement and the CUDA path against them.  Fixtures are small
(<= a few hundred KB each).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import hqmq  # noqa: E402  (the reference)
from hqmq.attention import AttentionConfig, fused_attend, reference_attend  # noqa: E402
from hqmq.codebook import CodebookBank, SecondaryCodebook, build_joint, build_secondary  # noqa: E402
from hqmq.codec import CodecConfig, TensorShape, decode_tensor, encode_tensor  # noqa: E402
from hqmq.hurwitz import build_primary_codebook  # noqa: E402
from hqmq.kernels import COMPILED_AVAILABLE, nearest_scan  # noqa: E402
from hqmq.kvpack import to_bytes  # noqa: E402
from hqmq.quat import haar_quaternions  # noqa: E402
from hqmq.rng import RandomStream  # noqa: E402
from hqmq.synth import GAUSSIAN, OUTLIER_HEAVY, gen_chunks  # noqa: E402

assert COMPILED_AVAILABLE, "the reference must be built with its compiled scan"
assert os.path.realpath(hqmq.__file__).startswith(os.path.join(ROOT, "oracle", "_ref"))


def save_codec_case(name, data, cast, cfg: CodecConfig, layer=0, role="K", head_base=0):
    """cast: dtype the GPU path receives ('f16', 'bf16', 'f32', 'f64').  `data`
    holds the exact float64 values of that dtype (what the reference encodes)."""
    packed = encode_tensor(data, cfg, layer=layer, role=role, head_base=head_base)
    bank = CodebookBank(seed=cfg.seed, size=cfg.codebook_size)
    blob = to_bytes(packed)
    dec = decode_tensor(packed, bank)
    meta = dict(
        name=name, cast=cast, codebook_size=cfg.codebook_size, radius_bits=cfg.radius_bits,
        seed=cfg.seed, outlier_multiplier=cfg.outlier_multiplier,
        median_pooling=cfg.median_pooling, layer=layer, role=role, head_base=head_base,
        digest=hashlib.sha256(blob).hexdigest(), nbytes=len(blob),
    )
    np.savez_compressed(
        os.path.join(HERE, f"codec_{name}.npz"),
        data=data, scales=packed.scales, indices=packed.indices, quanta=packed.quanta,
        flags=packed.flags, payloads=packed.payloads, decoded=dec,
        blob=np.frombuffer(blob, dtype=np.uint8), meta=json.dumps(meta),
    )
    return meta


def bf16_values(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to bf16 (RNE) and return them as exact float64."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def main():
    metas = []
    # 1. the reference's own frozen-digest fixture (test_kvpack.py:31-46,162-167)
    data = RandomStream(0x5EA1).gaussian(1 * 2 * 16 * 32).reshape(1, 2, 16, 32)
    data[0, 0, 3, 0:4] *= 60.0
    m = save_codec_case("frozen", data, "f64",
                        CodecConfig(codebook_size=48, radius_bits=4, seed=7, outlier_multiplier=3.0))
    assert m["digest"] == "12b2dfad207652800819a0ab439f8ef44c1c5ce33eff0f70979bc4e8b2cc1039"
    metas.append(m)
    # 2. C1 slice: Mistral-shaped Gaussian KV, fp16, S=16, b_r=4, C=3
    x = gen_chunks(GAUSSIAN, TensorShape(1, 8, 64, 128), seed=0).astype(np.float16).astype(np.float64)
    metas.append(save_codec_case("c1_slice", x, "f16",
                                 CodecConfig(codebook_size=16, radius_bits=4, outlier_multiplier=3.0)))
    # 3. S=64 without extraction, layer/role/head_base keying
    x = gen_chunks(GAUSSIAN, TensorShape(1, 4, 32, 128), seed=11).astype(np.float16).astype(np.float64)
    metas.append(save_codec_case("s64_v_l5_hb2", x, "f16",
                                 CodecConfig(codebook_size=64, radius_bits=4), layer=5, role="V",
                                 head_base=2))
    # 4. S=256 (the 70B config)
    x = gen_chunks(GAUSSIAN, TensorShape(1, 2, 16, 128), seed=3).astype(np.float16).astype(np.float64)
    metas.append(save_codec_case("s256", x, "f16", CodecConfig(codebook_size=256, radius_bits=4),
                                 layer=79, role="K"))
    # 5. Qwen-style outlier-heavy, S=64, b_r=6, Med3x
    x = gen_chunks(OUTLIER_HEAVY, TensorShape(1, 4, 64, 128), seed=5).astype(np.float16).astype(np.float64)
    metas.append(save_codec_case("outlier_heavy", x, "f16",
                                 CodecConfig(codebook_size=64, radius_bits=6, outlier_multiplier=3.0),
                                 layer=2))
    # 6. per-head pooling, odd shapes, fp64 input
    x = RandomStream(0xDA7A).gaussian(2 * 3 * 10 * 12).reshape(2, 3, 10, 12)
    x[:, 1] *= 10.0
    metas.append(save_codec_case("per_head_d12", x, "f64",
                                 CodecConfig(codebook_size=24, radius_bits=3, outlier_multiplier=3.0,
                                             median_pooling="per_head", seed=123)))
    # 7. padding (head_dim 126), fp32 input
    x = RandomStream(0x126).gaussian(1 * 2 * 8 * 126).reshape(1, 2, 8, 126).astype(np.float32).astype(np.float64)
    metas.append(save_codec_case("pad126_f32", x, "f32",
                                 CodecConfig(codebook_size=48, radius_bits=5, outlier_multiplier=3.0)))
    # 8. bf16 input, multiplier 2.5
    x = bf16_values(RandomStream(0xBF16).gaussian(1 * 2 * 16 * 64).reshape(1, 2, 16, 64))
    metas.append(save_codec_case("bf16", x, "bf16",
                                 CodecConfig(codebook_size=32, radius_bits=8, outlier_multiplier=2.5)))
    # 9. zeros: all-zero token, zero chunks, sigma sentinel
    x = RandomStream(0x2E80).gaussian(1 * 1 * 4 * 8).reshape(1, 1, 4, 8)
    x[0, 0, 1] = 0.0
    x[0, 0, 2, 4:8] = 0.0
    metas.append(save_codec_case("zeros", x, "f64", CodecConfig(codebook_size=24, radius_bits=3)))
    # 10. cell-exact inputs (codec roundtrip to 1e-9, test_codec.py:127-145)
    cfg = CodecConfig(codebook_size=24, radius_bits=4)
    joint = CodebookBank(seed=0, size=24).joint(0, 0, "K")
    top, sigma = 15, 2.0
    picks = RandomStream(0x9E7).raw(32)
    rows = []
    for i in range(32):
        cw = joint.codewords[int(picks[i]) % joint.codewords.shape[0]]
        level = int(picks[i] >> np.uint64(32)) % top + 1
        rows.append(cw * (sigma * level / top))
    x = np.stack(rows).reshape(1, 1, 8, 16)
    x[0, 0, :, 0:4] = joint.codewords[0] * sigma
    metas.append(save_codec_case("cell_exact", x, "f64", cfg))

    # codebook tables (pin the numpy restatement)
    tabs = {}
    for (seed, layer, head, role, size) in [(0, 0, 0, "K", 24), (7, 3, 1, "V", 48),
                                            (0, 79, 7, "V", 256), (123, 0, 2, "K", 5)]:
        tabs[f"{seed}_{layer}_{head}_{role}_{size}"] = build_joint(
            build_primary_codebook(), build_secondary(seed, layer, head, role, size)).codewords
    np.savez_compressed(os.path.join(HERE, "codebooks.npz"), **tabs)

    # nearest-scan known answers: bare 24-cell tie (test_codebook.py:91-103),
    # random directions, exact hits
    prim = build_primary_codebook()
    ident = SecondaryCodebook(entries=np.array([[1.0, 0.0, 0.0, 0.0]]), seed=0, layer=0, head=0, role="K")
    cell = build_joint(prim, ident).codewords
    xh = 1.0 / np.sqrt(2.0)
    tie_dirs = np.array([[xh, xh, 0.0, 0.0], [0.5, 0.5, 0.5, 0.5], [xh, 0.0, -xh, 0.0],
                         [0.0, 0.0, 0.0, 1.0]])
    j96 = build_joint(prim, build_secondary(0, 0, 0, "K", 96)).codewords
    rnd = haar_quaternions(RandomStream(0xC0DE), 3000)
    hits = j96[[0, 1, 13 * 96 + 42, 2303]]
    it, ct = nearest_scan(tie_dirs, cell)
    ir, cr = nearest_scan(rnd, j96)
    ih, ch = nearest_scan(hits, j96)
    np.savez_compressed(os.path.join(HERE, "scan.npz"), cell=cell, tie_dirs=tie_dirs, tie_idx=it,
                        tie_cos=ct, j96=j96, rnd=rnd, rnd_idx=ir, rnd_cos=cr, hits=hits,
                        hit_idx=ih, hit_cos=ch)

    # attention: decode-time GQA (T_q = 1) and a causal prefill block
    for name, (b, hq, hkv, tq, tkv, d, key) in {
        "decode_gqa": (2, 8, 2, 1, 96, 32, 0xA7A),
        "prefill_causal": (1, 4, 1, 16, 16, 16, 0xA77),
    }.items():
        cfg = AttentionConfig(b, hq, hkv, tq, tkv, d)
        st = RandomStream(key)
        q = st.gaussian(b * hq * tq * d).reshape(b, hq, tq, d)
        k = st.gaussian(b * hkv * tkv * d).reshape(b, hkv, tkv, d)
        v = st.gaussian(b * hkv * tkv * d).reshape(b, hkv, tkv, d)
        codec = CodecConfig(codebook_size=24, radius_bits=4)
        bank = CodebookBank(seed=0, size=24)
        pk = encode_tensor(k, codec, role="K", bank=bank)
        pv = encode_tensor(v, codec, role="V", bank=bank)
        dense = reference_attend(q, decode_tensor(pk, bank), decode_tensor(pv, bank), cfg)
        fused = fused_attend(q, pk, pv, bank, cfg, tile=32)
        np.savez_compressed(os.path.join(HERE, f"attn_{name}.npz"), q=q, k=k, v=v, dense=dense,
                            fused=fused, dims=np.array([b, hq, hkv, tq, tkv, d]))
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as f:
        json.dump(metas, f, indent=1)
    print(f"wrote {len(metas)} codec fixtures")


if __name__ == "__main__":
    main()
