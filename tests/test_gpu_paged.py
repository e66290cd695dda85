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


def test_paged_append_subsets_fragmented_pool(cuda):
    """hqmq_paged_append: appends for sequence subsets in any order into a
    shuffled page pool land in the right slots -- page contents equal each
    sequence's one-shot encode rows (token-local codec without extraction)."""
    m = hq()
    cfg = m.CodecConfig(64, 4)
    bank = m.CodebookBank(0, 64)
    gen = torch.Generator(device=cuda).manual_seed(9)
    B, H = 3, 2
    cache = m.PagedKVCache(cfg, B, H, max_tokens=384, bank=bank, page_order_seed=3)
    per_seq = {b: [] for b in range(B)}
    for seqs, n in (([2, 0], 70), ([1], 130), ([0, 1, 2], 61), ([2], 1)):
        x = torch.randn((len(seqs), H, n, 128), generator=gen, device=cuda).half()
        cache.append(x, x, seqs=seqs)
        for i, b in enumerate(seqs):
            per_seq[b].append(x[i:i + 1])
    cache.check_errors()
    w, br = cfg.index_bits, cfg.radius_bits
    pool = cache.pages["V"]
    for b in range(B):
        xs = torch.cat(per_seq[b], dim=2)
        ref = m.encode_tensor(xs, cfg, role="V", bank=bank)
        T = xs.shape[2]
        assert cache.lengths[b] == T
        for h in range(H):
            for t in range(T):
                pid = int(cache.block_table[b, h, t // 128]) * 128 + t % 128
                row = h * T + t
                assert torch.equal(pool["index"].view(-1, w)[pid], ref.index_words[row * w:(row + 1) * w])
                assert torch.equal(pool["radius"].view(-1, br)[pid],
                                   ref.radius_words[row * br:(row + 1) * br])
                assert torch.equal(pool["scales"].view(-1)[pid], ref.scales.reshape(-1)[row])


def test_paged_append_bad_page_reported(cuda):
    """A block-table entry outside the pool is skipped and reported through the
    cache's device error word (check_errors -> CorruptData)."""
    import ctypes

    m = hq()
    from paper_2605_27646_b200 import _native as nat

    cache = m.PagedKVCache(m.CodecConfig(16, 4), 1, 1, 256, num_pages=2)
    x = torch.randn((1, 1, 4, 128), device=cuda).half()
    qt = m.encode_tensor(x, cache.config, bank=cache.bank)
    table = torch.full((1, 1, 2), -1, dtype=torch.int32, device=cuda)
    info = torch.zeros((2, 1), dtype=torch.int32, device=cuda)
    pool = cache.pages["K"]
    a = nat.PagedAppendArgs()
    a.n_seq, a.kv_heads, a.n_new, a.max_pages = 1, 1, 4, 2
    a.page_tokens, a.index_bits, a.radius_bits, a.num_pages = 128, cache.config.index_bits, 4, 2
    a.seq_ids, a.seq_start, a.block_table = info[0].data_ptr(), info[1].data_ptr(), table.data_ptr()
    a.src_index, a.src_radius = qt.index_words.data_ptr(), qt.radius_words.data_ptr()
    a.src_scales = qt.scales.data_ptr()
    a.index_pages, a.radius_pages = pool["index"].data_ptr(), pool["radius"].data_ptr()
    a.scale_pages = pool["scales"].data_ptr()
    a.error_word = cache._err.data_ptr()
    nat.launch(cuda, "hqmq_paged_append", nat.lib().hqmq_paged_append, ctypes.byref(a))
    with pytest.raises(m.CorruptData):
        cache.check_errors()
    assert int(pool["index"].abs().sum()) == 0  # nothing written


def test_paged_errors(cuda):
    m = hq()
    cache = m.PagedKVCache(m.CodecConfig(16, 4), 1, 1, 128, num_pages=1)
    x = torch.zeros((1, 1, 129, 128), device=cuda, dtype=torch.float16)
    with pytest.raises(m.InvalidArgument):
        cache.append(x, x)  # past max_tokens
    with pytest.raises(m.InvalidArgument):
        cache.attend(torch.zeros((1, 4, 1, 128), device=cuda))  # empty
