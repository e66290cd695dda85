"""Med3x (C = 3 outlier extraction) on the serving path, against the oracle:

* frozen thresholds: encode_tensor(..., outlier_thresholds=) flags r > the
  given threshold (the reference's strict test, codec.py:208-219) and is
  bit-exact against the oracle's encode with the same thresholds; the
  thresholds an encode used (QuantizedTensor.outlier_thresholds) equal the
  oracle's C * lower_median (outliers.py:50-55);
* decode attention over a Med3x cache on the tensor-core kernel
  (attention_mma_kernel<Med3x>), within the reference's fp32 bound 1e-3
  (test_attention.py:97-102; relative to |out| where it exceeds 1: outlier
  payload rows are large) of the oracle's dense fp64 attention
  (attention.py:80-101) over the oracle's decode;
* PagedKVCache with Med3x: the prefill is the reference's encode of that call,
  later appends use its frozen thresholds (the deviation from a
  one-shot encode), attend() against the oracle; appends are token-local.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def hq():
    import paper_2605_27646_b200 as m

    return m


def heavy(shape, gen, dev):
    """synth.py:91-109-style outlier-heavy fp16 data: 2% of chunks scaled by
    exp(ln 25 + 0.6 N)."""
    B, H, T, D = shape
    x = torch.randn((B, H, T, D // 4, 4), generator=gen, device=dev)
    mark = torch.rand((B, H, T, D // 4, 1), generator=gen, device=dev) < 0.02
    mult = torch.exp(np.log(25.0) + 0.6 * torch.randn((B, H, T, D // 4, 1), generator=gen,
                                                      device=dev))
    return torch.where(mark, x * mult, x).reshape(shape).half()


def np64(x):
    return x.double().cpu().numpy()


def oracle_norms(oracle, x64):
    ch = oracle.chunked(x64)
    return np.sqrt((ch * ch).sum(axis=4))


@pytest.mark.parametrize("S,br,pool", [(64, 6, "batch"), (16, 4, "per_head"), (256, 4, "batch")])
def test_frozen_threshold_encode_vs_oracle(cuda, oracle, S, br, pool):
    m = hq()
    gen = torch.Generator(device=cuda).manual_seed(S + br)
    cfg = m.CodecConfig(S, br, seed=5, outlier_multiplier=3.0, median_pooling=pool)
    bank = m.CodebookBank(5, S)
    x = heavy((2, 3, 96, 128), gen, cuda)
    qt = m.encode_tensor(x, cfg, layer=3, role="V", bank=bank)
    thr_ref = oracle.outlier_thresholds(oracle_norms(oracle, np64(x)), 3.0, pool)
    np.testing.assert_array_equal(qt.outlier_thresholds.cpu().numpy(), thr_ref)
    # new tokens flagged against the frozen thresholds
    y = heavy((2, 3, 40, 128), gen, cuda)
    y[0, 1, 7, 0:4] = 0.0  # an all-zero chunk: r = 0 is never flagged
    qy = m.encode_tensor(y, cfg, layer=3, role="V", bank=bank,
                         outlier_thresholds=qt.outlier_thresholds)
    ref = oracle.encode(np64(y), S, br, seed=5, multiplier=3.0, pooling=pool, layer=3,
                        role="V", thresholds=thr_ref)
    assert ref.flags.any()
    assert m.to_bytes(qy) == oracle.to_bytes(ref)
    np.testing.assert_array_equal(m.decode_tensor(qy, bank, dtype=torch.float64).cpu().numpy(),
                                  oracle.decode(ref))
    np.testing.assert_array_equal(qy.outlier_thresholds.cpu().numpy(), thr_ref)
    # token-local: a token slice encodes to the slice of the whole
    qa = m.encode_tensor(y[:, :, 11:29], cfg, layer=3, role="V", bank=bank,
                         outlier_thresholds=torch.as_tensor(thr_ref))
    assert torch.equal(qa.flags, qy.flags[:, :, 11:29])
    assert torch.equal(qa.indices, qy.indices[:, :, 11:29])
    assert torch.equal(qa.quanta, qy.quanta[:, :, 11:29])


def test_frozen_threshold_errors(cuda):
    m = hq()
    x = torch.randn((1, 2, 8, 128), device=cuda).half()
    with pytest.raises(m.InvalidArgument):
        m.encode_tensor(x, m.CodecConfig(16, 4), outlier_thresholds=1.0)
    with pytest.raises(m.InvalidArgument):  # per-head pooling needs one threshold per head
        m.encode_tensor(x, m.CodecConfig(16, 4, outlier_multiplier=3.0, median_pooling="per_head"),
                        outlier_thresholds=[1.0, 2.0, 3.0])
    with pytest.raises(m.InvalidArgument):
        m.PagedKVCache(m.CodecConfig(16, 4), 1, 1, 128, outlier_thresholds=1.0)
    with pytest.raises(m.InvalidArgument):  # four S=256 tables exceed shared memory
        m.PagedKVCache(m.CodecConfig(256, 4, outlier_multiplier=3.0), 1, 1, 128)


@pytest.mark.parametrize("S,br,B,HQ,HKV,TQ,T,causal,C", [
    (64, 6, 2, 8, 2, 1, 2048, True, 3.0),     # the C3 codec config, GQA 4
    (64, 6, 1, 7, 1, 1, 4104, False, 3.0),    # GQA 7 (Qwen), T % 128 != 0
    (16, 4, 2, 8, 2, 2, 1032, True, 3.0),     # C1 codec config, T_q = 2 (causal offsets)
    (256, 4, 1, 8, 1, 1, 520, True, 3.0),     # S = 256 (13-bit codes)
    (64, 4, 1, 8, 2, 1, 1024, True, 1.2),     # ~25% outliers: tiles past the staged payload rows
])
def test_med3x_attention_tensor_core_vs_oracle(cuda, oracle, S, br, B, HQ, HKV, TQ, T, causal, C):
    m = hq()
    gen = torch.Generator(device=cuda).manual_seed(T + S)
    cfg = m.CodecConfig(S, br, outlier_multiplier=C)
    bank = m.CodebookBank(0, S)
    k = heavy((B, HKV, T, 128), gen, cuda)
    v = heavy((B, HKV, T, 128), gen, cuda)
    pk = m.encode_tensor(k, cfg, role="K", bank=bank, layer=4)
    pv = m.encode_tensor(v, cfg, role="V", bank=bank, layer=4)
    assert pk.n_payload > 0 and pv.n_payload > 0
    rk = oracle.encode(np64(k), S, br, multiplier=C, layer=4, role="K")
    rv = oracle.encode(np64(v), S, br, multiplier=C, layer=4, role="V")
    assert m.to_bytes(pk) == oracle.to_bytes(rk) and m.to_bytes(pv) == oracle.to_bytes(rv)
    q = torch.randn((B, HQ, TQ, 128), generator=gen, device=cuda)
    acfg = m.AttentionConfig(B, HQ, HKV, TQ, T, 128, causal=causal)
    # S = 256 Med3x needs more shared memory than a CTA has (four 48 KB tables):
    # the fp32 CUDA-core kernel serves it
    want = "attention_mma_kernel<Med3x>" if S <= 64 else "attention_split_kernel"
    assert m.attention_kernel(q, pk, pv, bank, acfg) == want
    dense = oracle.reference_attend(np64(q), oracle.decode(rk), oracle.decode(rv), HQ // HKV,
                                    causal=causal)
    bound = np.maximum(1.0, np.abs(dense))
    for splits in (0, 1, 3):
        out = m.fused_attend(q, pk, pv, bank, acfg, num_splits=splits)
        err = (np.abs(np64(out) - dense) / bound).max()
        assert err <= 1e-3, (splits, err)
    # the fp32 CUDA-core path agrees too (and the outliers matter: dropping them
    # would move the output far beyond the bound)
    precise = m.fused_attend(q, pk, pv, bank, acfg, precise=True)
    assert (np.abs(np64(precise) - dense) / bound).max() <= 2e-5


def _paged_reference(oracle, calls, thr, S, br, layer, B, HKV):
    """Oracle K/V per sequence from the cache's append calls: the first call of
    each role is encoded with its own median, later ones with its thresholds."""
    seqs_k = [np.zeros((HKV, 0, 128)) for _ in range(B)]
    seqs_v = [np.zeros((HKV, 0, 128)) for _ in range(B)]
    for seqs, k64, v64 in calls:
        for role, x64, store in (("K", k64, seqs_k), ("V", v64, seqs_v)):
            first = thr[role] is None
            enc = oracle.encode(x64, S, br, multiplier=3.0, layer=layer, role=role,
                                thresholds=None if first else thr[role])
            if first:
                thr[role] = oracle.outlier_thresholds(
                    np.sqrt((oracle.chunked(x64) ** 2).sum(axis=4)), 3.0, "batch")
            dec = oracle.decode(enc)
            for i, b in enumerate(seqs):
                store[b] = np.concatenate([store[b], dec[i]], axis=1)
    return seqs_k, seqs_v


def test_paged_med3x_vs_oracle(cuda, oracle):
    m = hq()
    S, br, B, HKV, g, layer = 64, 6, 3, 2, 4, 6
    gen = torch.Generator(device=cuda).manual_seed(77)
    cfg = m.CodecConfig(S, br, outlier_multiplier=3.0)
    bank = m.CodebookBank(0, S)
    cache = m.PagedKVCache(cfg, B, HKV, max_tokens=800, layer=layer, bank=bank,
                           page_order_seed=3)
    steps = [([0, 1, 2], 130), ([1], 77), ([0, 1, 2], 1), ([0, 2], 129), ([2], 1)]
    calls, thr = [], {"K": None, "V": None}
    for seqs, n in steps:
        k = heavy((len(seqs), HKV, n, 128), gen, cuda)
        v = heavy((len(seqs), HKV, n, 128), gen, cuda)
        cache.append(k, v, seqs=seqs)
        calls.append((seqs, np64(k), np64(v)))
        thr = {"K": None, "V": None}
        ks, vs = _paged_reference(oracle, calls, thr, S, br, layer, B, HKV)
        for role in ("K", "V"):
            np.testing.assert_array_equal(cache.thresholds[role].cpu().numpy(), thr[role])
        q = torch.randn((B, HKV * g, 1, 128), generator=gen, device=cuda)
        dense = np.concatenate([oracle.reference_attend(np64(q[b:b + 1]), ks[b][None], vs[b][None],
                                                        g, causal=True) for b in range(B)])
        bound = np.maximum(1.0, np.abs(dense))
        for splits in (0, 2):
            out = cache.attend(q, num_splits=splits)
            err = (np.abs(np64(out) - dense) / bound).max()
            # 2e-3 as the no-Med3x paged test: short rows (1 key after the
            # prefill of sequence 1's ...) are dominated by fp16 P / V rounding
            assert err <= 2e-3, (seqs, n, splits, err)
    assert cache.lengths == [260, 208, 261]
    assert cache.n_payload["K"] > 0 and cache.n_payload["V"] > 0


def _slot_payloads(cache, role):
    """{slot: fp16 payload rows of that token, in chunk order} of a Med3x cache."""
    flags = cache.pages[role]["flags"].view(-1).cpu().numpy().view(np.uint32)
    payoff = cache.pages[role]["payoff"].view(-1).cpu().numpy().view(np.uint32)
    pool = cache.payloads[role][: cache.n_payload[role]].cpu().numpy()
    out = {}
    for slot in np.nonzero(flags)[0]:
        n = bin(int(flags[slot])).count("1")
        out[int(slot)] = pool[payoff[slot]: payoff[slot] + n]
    return out


def test_paged_med3x_appends_token_local(cuda):
    """With frozen thresholds, appending tokens in pieces leaves exactly the
    page contents of appending them at once, and every token's payload rows
    (the pool's row order follows the append calls)."""
    m = hq()
    cfg = m.CodecConfig(64, 4, outlier_multiplier=3.0)
    bank = m.CodebookBank(0, 64)
    gen = torch.Generator(device=cuda).manual_seed(9)
    pre_k, pre_v = heavy((2, 2, 64, 128), gen, cuda), heavy((2, 2, 64, 128), gen, cuda)
    yk, yv = heavy((2, 2, 50, 128), gen, cuda), heavy((2, 2, 50, 128), gen, cuda)
    a = m.PagedKVCache(cfg, 2, 2, max_tokens=256, bank=bank)
    b = m.PagedKVCache(cfg, 2, 2, max_tokens=256, bank=bank)
    for c in (a, b):
        c.append(pre_k, pre_v)
    a.append(yk, yv)
    for lo, hi in ((0, 20), (20, 21), (21, 50)):
        b.append(yk[:, :, lo:hi], yv[:, :, lo:hi])
    assert torch.equal(a.block_table, b.block_table)
    for role in ("K", "V"):
        for name in ("index", "radius", "scales", "flags"):
            assert torch.equal(a.pages[role][name], b.pages[role][name]), (role, name)
        n = a.n_payload[role]
        assert n == b.n_payload[role] and n > 0
        pa, pb = _slot_payloads(a, role), _slot_payloads(b, role)
        assert pa.keys() == pb.keys() and len(pa) > 0
        for slot in pa:
            np.testing.assert_array_equal(pa[slot], pb[slot])


@pytest.mark.parametrize("dtype,D,pool", [(torch.float32, 96, "batch"), (torch.bfloat16, 64, "per_head")])
def test_frozen_threshold_general_path(cuda, oracle, dtype, D, pool):
    """Frozen thresholds on the general encode path (not fp16 / head_dim 128:
    the tile kernel): thresholds_out equals the oracle's C * median, and a
    frozen-threshold encode is bit-exact against the oracle."""
    m = hq()
    gen = torch.Generator(device=cuda).manual_seed(D)
    cfg = m.CodecConfig(24, 5, seed=3, outlier_multiplier=2.5, median_pooling=pool)
    bank = m.CodebookBank(3, 24)
    x = heavy((2, 3, 40, D), gen, cuda).to(dtype)
    qt = m.encode_tensor(x, cfg, layer=2, role="K", bank=bank)
    thr_ref = oracle.outlier_thresholds(oracle_norms(oracle, np64(x)), 2.5, pool)
    np.testing.assert_array_equal(qt.outlier_thresholds.cpu().numpy(), thr_ref)
    y = heavy((2, 3, 17, D), gen, cuda).to(dtype)
    qy = m.encode_tensor(y, cfg, layer=2, role="K", bank=bank, outlier_thresholds=thr_ref)
    ref = oracle.encode(np64(y), 24, 5, seed=3, multiplier=2.5, pooling=pool, layer=2, role="K",
                        thresholds=thr_ref)
    assert m.to_bytes(qy) == oracle.to_bytes(ref)
