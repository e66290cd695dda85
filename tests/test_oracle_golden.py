"""The oracle restatement (oracle/) against the reference's own outputs.

CPU-only.  Pins the checker before it is trusted: every golden fixture was
produced by the unmodified reference (tests/golden/make_golden.py), including
the reference's frozen SHA-256 digest (test_kvpack.py:28).
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, adversarial_fixtures, codec_fixtures, load_adversarial, load_codec_fixture

FROZEN = "12b2dfad207652800819a0ab439f8ef44c1c5ce33eff0f70979bc4e8b2cc1039"


@pytest.mark.parametrize("name", codec_fixtures())
def test_oracle_encode_matches_reference(oracle, name):
    meta, g = load_codec_fixture(name)
    enc = oracle.encode(g["data"], meta["codebook_size"], meta["radius_bits"], seed=meta["seed"],
                        multiplier=meta["outlier_multiplier"], pooling=meta["median_pooling"],
                        layer=meta["layer"], role=meta["role"], head_base=meta["head_base"])
    for f in ("scales", "indices", "quanta", "flags", "payloads"):
        assert np.array_equal(getattr(enc, f), g[f]), f
    blob = oracle.to_bytes(enc)
    assert blob == g["blob"].tobytes()
    assert hashlib.sha256(blob).hexdigest() == meta["digest"]
    assert np.array_equal(oracle.decode(enc), g["decoded"])


def test_frozen_digest(oracle):
    meta, g = load_codec_fixture("frozen")
    assert meta["digest"] == FROZEN
    data = oracle.Stream(0x5EA1).gaussian(1 * 2 * 16 * 32).reshape(1, 2, 16, 32)
    data[0, 0, 3, 0:4] *= 60.0
    enc = oracle.encode(data, 48, 4, seed=7, multiplier=3.0)
    assert oracle.digest(enc) == FROZEN


def test_codebooks_match_reference(oracle):
    z = np.load(os.path.join(GOLDEN, "codebooks.npz"))
    for key in z.files:
        seed, layer, head, role, size = key.split("_")
        cw = oracle.joint(int(seed), int(layer), int(head), role, int(size))
        assert np.array_equal(cw, z[key]), key


def test_scan_known_answers(oracle):
    z = np.load(os.path.join(GOLDEN, "scan.npz"))
    for dirs, cw, idx, cos in (("tie_dirs", "cell", "tie_idx", "tie_cos"),
                               ("rnd", "j96", "rnd_idx", "rnd_cos"),
                               ("hits", "j96", "hit_idx", "hit_cos")):
        i, c = oracle.nearest_scan(z[dirs], z[cw])
        assert np.array_equal(i, z[idx])
        assert np.array_equal(c, z[cos])
        i2, c2 = oracle.nearest_scan_numpy(z[dirs], z[cw])
        assert np.array_equal(i2, z[idx])
        assert np.array_equal(c2, z[cos])
    # the bare 24-cell tie resolves to flat index 0 (test_codebook.py:91-103)
    assert z["tie_idx"][0] == 0


def test_scan_threads_invariant(oracle):
    z = np.load(os.path.join(GOLDEN, "scan.npz"))
    a = oracle.nearest_scan(z["rnd"], z["j96"], threads=1)
    b = oracle.nearest_scan(z["rnd"], z["j96"], threads=4)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("name", ["decode_gqa", "prefill_causal"])
def test_oracle_attention_matches_reference(oracle, name):
    z = np.load(os.path.join(GOLDEN, f"attn_{name}.npz"))
    b, hq, hkv, tq, tkv, d = (int(v) for v in z["dims"])
    pk = oracle.encode(z["k"], 24, 4, role="K")
    pv = oracle.encode(z["v"], 24, 4, role="V")
    out = oracle.reference_attend(z["q"], oracle.decode(pk), oracle.decode(pv), hq // hkv)
    assert np.array_equal(out, z["dense"])
    assert np.max(np.abs(z["fused"] - z["dense"])) <= 1e-10


def test_lower_median_and_threshold(oracle):
    # outliers.py:50-55 lower median; codec.py:215 strict threshold
    assert oracle.lower_median(np.array([3.0, 1.0, 2.0, 4.0])) == 2.0
    assert oracle.lower_median(np.array([5.0, 1.0, 3.0])) == 3.0
    norms = np.array([1.0, 1.0, 3.0, 3.0000001]).reshape(1, 1, 1, 4)
    flags = oracle.outlier_flags(norms, 3.0, "batch")
    assert flags.ravel().tolist() == [False, False, False, True]


def test_synth_generators(oracle):
    # the oracle's synth restatement feeds the CPU baseline (synth.py:73-111)
    x = oracle.gen_outlier_heavy((1, 2, 64, 128), seed=5)
    ch = oracle.chunked(x)
    n = np.sqrt((ch * ch).sum(-1)).ravel()
    med = oracle.lower_median(n)
    assert abs(n.max() / med - 150.0) < 1e-6
    g = oracle.gen_gaussian((1, 1, 4, 8), seed=0)
    assert g.shape == (1, 1, 4, 8)


@pytest.mark.parametrize("name", adversarial_fixtures())
def test_oracle_adversarial_matches_reference(oracle, name):
    """Boundary chunks (tests/golden/make_adversarial.py): top-2 score gaps
    down to 1e-10 (fp16) and exact ties (fp64) resolve like the reference."""
    meta, g = load_adversarial(name)
    assert meta["n_gap_below_1e5"] > meta["n_chunks"] // 2  # really on the boundaries
    enc = oracle.encode(g["data"], meta["codebook_size"], meta["radius_bits"], seed=meta["seed"],
                        layer=meta["layer"], role=meta["role"])
    for f in ("scales", "indices", "quanta"):
        assert np.array_equal(getattr(enc, f), g[f]), f
    assert hashlib.sha256(oracle.to_bytes(enc)).hexdigest() == meta["digest"]


def test_oracle_covering_matches_reference(oracle):
    """The oracle's covering estimate (packing.py:59-83) reproduces the
    reference's golden values bit for bit (small cases; the GPU test runs all)."""
    import json

    cases = json.load(open(os.path.join(GOLDEN, "covering.json")))
    for c in cases:
        if c["S"] > 16:
            continue
        if c["S"] == 0:
            cw = oracle.hamilton(oracle.primary_2t()[:, None, :],
                                 np.array([[[1.0, 0.0, 0.0, 0.0]]])).reshape(-1, 4)
        else:
            cw = oracle.joint(c["seed"], c["layer"], c["head"], c["role"], c["S"])
        rho, mean = oracle.estimate_covering(cw, c["n_probes"], c["probe_seed"])
        assert rho == float.fromhex(c["rho_hat"]) and mean == float.fromhex(c["mean_angle"])
