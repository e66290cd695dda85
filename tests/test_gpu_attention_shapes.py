"""Decode attention at the BASELINE config shapes, against the oracle
(VERDICT r01 parity items 1(b) and 1(c)).

* C4: Llama-3-8B decode step, B = 32, H_q = 32, H_kv = 8, T_q = 1, d = 128,
  S = 64, b_r = 4, at 32k keys (and 128k), the serving path (fp32 out,
  tensor cores) within the reference's fp32 bound 1e-3
  (test_attention.py:97-102) and the fp64 path within 1e-10
  (test_attention.py:83-87);
* C3: Qwen2.5-7B shape (H_q = 28, H_kv = 4, GQA 7) over an outlier-heavy cache
  encoded with Med3x (S = 64, b_r = 6, C = 3) at 32k keys.

The comparison is the oracle's dense fp64 attention (oracle.reference_attend,
attention.py:80-101) over the fp64 decode of sampled batch rows (the fp64
decode is bit-exact against the oracle's, test_gpu_parity.py), so the kernel is
never compared with itself.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def decoded_rows(m, packed, bank, rows, chunk=4096):
    """fp64 decode of batch rows `rows`, token chunk by token chunk."""
    T = packed.shape.tokens
    parts = []
    for t0 in range(0, T, chunk):
        t1 = min(T, t0 + chunk)
        d = m.decode_token_range(packed, bank, t0, t1, dtype=torch.float64)
        parts.append(d[rows].cpu().numpy())
        del d
    return np.concatenate(parts, axis=2)


def check_rows(m, oracle, q, out, pk, pv, bank, rows, group, tol, rel=False):
    kd = decoded_rows(m, pk, bank, rows)
    vd = decoded_rows(m, pv, bank, rows)
    qr = q[rows].double().cpu().numpy()
    dense = oracle.reference_attend(qr, kd, vd, group, causal=True)
    got = out[rows].double().cpu().numpy()
    err = np.abs(got - dense)
    if rel:
        err = err / np.maximum(1.0, np.abs(dense))
    assert err.max() <= tol, err.max()
    return err.max()


@pytest.mark.parametrize("T,rows", [(32768, [0, 13, 31]), (131072, [5, 30])])
def test_c4_decode_attention_full_shape(cuda, oracle, T, rows):
    import paper_2605_27646_b200 as m

    B, HQ, HKV, D = 32, 32, 8, 128
    g = torch.Generator(device=cuda).manual_seed(T)
    cfg = m.CodecConfig(64, 4)
    bank = m.CodebookBank(0, 64)
    k = torch.randn((B, HKV, T, D), generator=g, device=cuda, dtype=torch.float16)
    pk = m.encode_tensor(k, cfg, role="K", bank=bank, layer=7)
    del k
    v = torch.randn((B, HKV, T, D), generator=g, device=cuda, dtype=torch.float16)
    pv = m.encode_tensor(v, cfg, role="V", bank=bank, layer=7)
    del v
    q = torch.randn((B, HQ, 1, D), generator=g, device=cuda)
    acfg = m.AttentionConfig(B, HQ, HKV, 1, T, D)
    fast = m.fused_attend(q, pk, pv, bank, acfg)
    assert fast.dtype == torch.float32
    check_rows(m, oracle, q, fast, pk, pv, bank, rows, HQ // HKV, 1e-3)
    if T == 32768:
        exact = m.fused_attend(q.double(), pk, pv, bank, acfg)
        assert exact.dtype == torch.float64
        check_rows(m, oracle, q, exact, pk, pv, bank, rows, HQ // HKV, 1e-10)


def test_c3_med3x_decode_attention(cuda, oracle):
    import paper_2605_27646_b200 as m

    B, HQ, HKV, T, D = 4, 28, 4, 32768, 128
    g = torch.Generator(device=cuda).manual_seed(3)
    cfg = m.CodecConfig(64, 6, outlier_multiplier=3.0)
    bank = m.CodebookBank(0, 64)

    def heavy():
        x = torch.randn((B, HKV, T, D // 4, 4), generator=g, device=cuda)
        mark = torch.rand((B, HKV, T, D // 4, 1), generator=g, device=cuda) < 0.02
        mult = torch.exp(np.log(25.0) + 0.6 * torch.randn((B, HKV, T, D // 4, 1), generator=g,
                                                          device=cuda))
        return torch.where(mark, x * mult, x).reshape(B, HKV, T, D).half()

    pk = m.encode_tensor(heavy(), cfg, role="K", bank=bank, layer=2)
    pv = m.encode_tensor(heavy(), cfg, role="V", bank=bank, layer=2)
    assert pk.n_payload > 0.01 * pk.shape.n_chunks and pv.n_payload > 0
    q = torch.randn((B, HQ, 1, D), generator=g, device=cuda)
    acfg = m.AttentionConfig(B, HQ, HKV, 1, T, D)
    rows = [0, 3]
    fast = m.fused_attend(q, pk, pv, bank, acfg)
    # outlier payload rows can exceed 1 in magnitude: bound relative to |out| > 1
    check_rows(m, oracle, q, fast, pk, pv, bank, rows, HQ // HKV, 1e-3, rel=True)
    exact = m.fused_attend(q.double(), pk, pv, bank, acfg)
    check_rows(m, oracle, q, exact, pk, pv, bank, rows, HQ // HKV, 1e-10)


@pytest.mark.parametrize("B,HQ,HKV,TQ,T,causal", [
    (16, 32, 8, 2, 32768, True),    # T_q = 2 (speculative decode): 8 rows, causal offsets
    (8, 64, 8, 1, 65536, True),     # GQA 8
    (32, 8, 8, 1, 16392, False),    # no GQA, T % 16 != 0 (partial last block), non-causal
])
def test_pair_kernel_shapes(cuda, oracle, B, HQ, HKV, TQ, T, causal):
    """Shapes above the K/V CTA-pair kernel's size threshold (>= 4M cached
    keys) with the row / block edge cases it must mask."""
    import paper_2605_27646_b200 as m

    D = 128
    g = torch.Generator(device=cuda).manual_seed(B * T + HQ)
    cfg = m.CodecConfig(64, 4)
    bank = m.CodebookBank(0, 64)
    k = torch.randn((B, HKV, T, D), generator=g, device=cuda, dtype=torch.float16)
    pk = m.encode_tensor(k, cfg, role="K", bank=bank, layer=3)
    del k
    v = torch.randn((B, HKV, T, D), generator=g, device=cuda, dtype=torch.float16)
    pv = m.encode_tensor(v, cfg, role="V", bank=bank, layer=3)
    del v
    q = torch.randn((B, HQ, TQ, D), generator=g, device=cuda)
    acfg = m.AttentionConfig(B, HQ, HKV, TQ, T, D, causal=causal)
    out = m.fused_attend(q, pk, pv, bank, acfg)
    rows = [0, B - 1]
    kd = decoded_rows(m, pk, bank, rows)
    vd = decoded_rows(m, pv, bank, rows)
    dense = oracle.reference_attend(q[rows].double().cpu().numpy(), kd, vd, HQ // HKV, causal=causal)
    err = np.abs(out[rows].double().cpu().numpy() - dense).max()
    assert err <= 1e-3, err


def test_pair_kernel_paged_ragged(cuda, oracle):
    """The serving layout through the pair kernel: 128-token pages in random
    order, ragged sequence lengths (partial last pages, lengths not a multiple
    of 16), against the oracle per sequence."""
    import paper_2605_27646_b200 as m

    B, HQ, HKV, D = 24, 32, 8, 128
    g = torch.Generator(device=cuda).manual_seed(11)
    cfg = m.CodecConfig(64, 4)
    bank = m.CodebookBank(0, 64)
    lens = [int(x) for x in torch.randint(16000, 32768, (B,), generator=g, device=cuda).tolist()]
    lens[0], lens[1] = 32768, 20001
    cache = m.PagedKVCache(cfg, B, HKV, max_tokens=32768, bank=bank, page_order_seed=5, device=cuda)
    assert B * HKV * max(lens) >= 1 << 22  # the pair kernel's regime
    seqs_k, seqs_v = {}, {}
    for b, n in enumerate(lens):
        k = torch.randn((1, HKV, n, D), generator=g, device=cuda).half()
        v = torch.randn((1, HKV, n, D), generator=g, device=cuda).half()
        cache.append(k, v, seqs=[b])
        if b in (0, 1, B - 1):
            seqs_k[b], seqs_v[b] = k, v
    q = torch.randn((B, HQ, 1, D), generator=g, device=cuda)
    out = cache.attend(q)
    for b in seqs_k:
        pk = m.encode_tensor(seqs_k[b], cfg, role="K", bank=bank)
        pv = m.encode_tensor(seqs_v[b], cfg, role="V", bank=bank)
        kd = m.decode_tensor(pk, bank, dtype=torch.float64).cpu().numpy()
        vd = m.decode_tensor(pv, bank, dtype=torch.float64).cpu().numpy()
        dense = oracle.reference_attend(q[b:b + 1].double().cpu().numpy(), kd, vd, HQ // HKV, causal=True)
        err = np.abs(out[b:b + 1].double().cpu().numpy() - dense).max()
        assert err <= 1e-3, (b, err)
