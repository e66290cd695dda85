"""Paged decode-attention over an appendable HQMQ cache:
`PagedKVCache.append` + `attend` against the dense fp64 attention
(attention.py:80-101) over the decode of each sequence's tokens encoded in one
call.  Without Med3x the codec is token-local, so the paged codes must also be
bit-identical to a one-shot encode of the concatenated tokens."""

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def hq():
    import paper_2605_27646_b200 as m

    return m


def _dense(m, cfg, bank, q, ks, vs, g, layer=0):
    """Per-sequence reference: one-shot encode + fp64 decode (bit-exact against
    the oracle's decode, test_gpu_parity.py) + the ORACLE's dense fp64
    attention (oracle.reference_attend, attention.py:80-101)."""
    import hqmq_oracle as O

    outs = []
    for b, (k, v) in enumerate(zip(ks, vs)):
        pk = m.encode_tensor(k[None], cfg, role="K", bank=bank, layer=layer)
        pv = m.encode_tensor(v[None], cfg, role="V", bank=bank, layer=layer)
        kd = m.decode_tensor(pk, bank, dtype=torch.float64).cpu().numpy()
        vd = m.decode_tensor(pv, bank, dtype=torch.float64).cpu().numpy()
        outs.append(torch.from_numpy(O.reference_attend(q[b:b + 1].double().cpu().numpy(), kd, vd,
                                                        q.shape[1] // k.shape[0], causal=True)))
    return torch.cat(outs).to(q.device)


@pytest.mark.parametrize("S,br,g", [(64, 4, 4), (16, 4, 8), (256, 4, 1), (64, 6, 2)])
def test_paged_attention_ragged_appends(cuda, S, br, g):
    m = hq()
    B, HKV = 3, 2
    gen = torch.Generator(device=cuda).manual_seed(S * 10 + br)
    cfg = m.CodecConfig(S, br)
    bank = m.CodebookBank(0, S)
    cache = m.PagedKVCache(cfg, B, HKV, max_tokens=1000, layer=2, bank=bank, page_order_seed=S)
    full_k = [torch.empty((HKV, 0, 128), device=cuda, dtype=torch.float16) for _ in range(B)]
    full_v = [t.clone() for t in full_k]
    # ragged prompts, then decode-style appends of 1 token and a 2nd chunk
    steps = [({0: 300, 1: 5, 2: 129}), ({0: 1, 1: 1, 2: 1}), ({1: 250}), ({0: 128, 2: 1})]
    for step in steps:
        for b, n in step.items():
            k = torch.randn((1, HKV, n, 128), generator=gen, device=cuda).half()
            v = torch.randn((1, HKV, n, 128), generator=gen, device=cuda).half()
            cache.append(k, v, seqs=[b])
            full_k[b] = torch.cat([full_k[b], k[0]], dim=1)
            full_v[b] = torch.cat([full_v[b], v[0]], dim=1)
        q = torch.randn((B, HKV * g, 1, 128), generator=gen, device=cuda)
        dense = _dense(m, cfg, bank, q, full_k, full_v, g, layer=2)
        for splits in (0, 1, 3):
            out = cache.attend(q, num_splits=splits).double()
            # 2e-3: with a handful of keys (sequence 1 starts at 5) the fp16
            # rounding of P and V dominates, as in the prefill test
            assert (out - dense).abs().max().item() <= 2e-3, (step, splits)
    assert cache.lengths == [429, 256, 131]


def test_paged_codes_match_one_shot_encode(cuda):
    """Page contents are bit-identical to the one-shot encode's token rows."""
    m = hq()
    cfg = m.CodecConfig(64, 4)
    bank = m.CodebookBank(0, 64)
    gen = torch.Generator(device=cuda).manual_seed(5)
    cache = m.PagedKVCache(cfg, 1, 2, max_tokens=512, bank=bank)
    ks = [torch.randn((1, 2, n, 128), generator=gen, device=cuda).half() for n in (100, 60, 1)]
    for k in ks:
        cache.append(k, k)
    ref = m.encode_tensor(torch.cat(ks, dim=2), cfg, role="K", bank=bank)
    w, br = cfg.index_bits, cfg.radius_bits
    T = 161
    pool = cache.pages["K"]
    for h in range(2):
        for t in range(T):
            pid = int(cache.block_table[0, h, t // 128]) * 128 + t % 128
            row = h * T + t
            assert torch.equal(pool["index"].view(-1, w)[pid], ref.index_words[row * w:(row + 1) * w])
            assert torch.equal(pool["radius"].view(-1, br)[pid],
                               ref.radius_words[row * br:(row + 1) * br])
            assert torch.equal(pool["scales"].view(-1)[pid], ref.scales.reshape(-1)[row])


def test_paged_errors(cuda):
    m = hq()
    cache = m.PagedKVCache(m.CodecConfig(16, 4), 1, 1, 128, num_pages=1)
    x = torch.zeros((1, 1, 129, 128), device=cuda, dtype=torch.float16)
    with pytest.raises(m.InvalidArgument):
        cache.append(x, x)  # past max_tokens
    with pytest.raises(m.InvalidArgument):
        cache.attend(torch.zeros((1, 4, 1, 128), device=cuda))  # empty
