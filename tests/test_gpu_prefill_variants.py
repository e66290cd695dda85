"""Prefill attention over the compressed cache, both paths: the two tcgen05
prefill kernels (prefill="tcgen05": attention_fa2_kernel below 4096 keys,
attention_fa4_kernel from 4096 keys; launch_prefill_tc picks by key count --
the C ABI's path) and the default composition (prefill="auto": the sm_100a
fp16 decode + PyTorch SDPA), against the oracle's dense fp64 attention over
the fp64 decode of the same cache.  Bound: 2e-3 relative to max(1, |out|) -- TWICE the reference's fp32
tolerance (test_attention.py:97-102, 1e-3): Q, K, V and P are fp16 tensor-core
operands, and fp16 rounding of Q and K moves logits of magnitude ~10 by ~1e-2,
i.e. P by ~1% (measured worst 1.2e-3 on causal GQA rows).  A documented gap
(INTEGRATION.md); the decode path (T_q * g <= 8) and fp64 path meet the
reference's bounds."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))


@pytest.mark.parametrize("mode", ["tcgen05", "auto"])
@pytest.mark.parametrize("shape", [
    (1, 8, 2, 300, 300, True),     # fa2, GQA 4, causal, ragged tiles
    (2, 4, 4, 130, 200, True),     # fa2, no GQA, Tq < Tkv offset
    (1, 16, 2, 96, 96, False),     # fa2, GQA 8, non-causal
    (1, 8, 2, 200, 4100, True),    # fa4 (>= 4096 keys), ragged last tile
    (1, 4, 1, 64, 4096, False),    # fa4, GQA 4, non-causal
])
def test_prefill_kernels_vs_oracle(cuda, shape, mode):
    import torch

    import hqmq_oracle as O
    import paper_2605_27646_b200 as m

    B, HQ, HKV, TQ, TK, causal = shape
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(TQ + TK)
    cfg = m.CodecConfig(64, 4)
    bank = m.CodebookBank(0, 64)
    k = torch.randn((B, HKV, TK, 128), generator=g, device=dev).half()
    v = torch.randn((B, HKV, TK, 128), generator=g, device=dev).half()
    q = torch.randn((B, HQ, TQ, 128), generator=g, device=dev)
    pk = m.encode_tensor(k, cfg, role="K", bank=bank)
    pv = m.encode_tensor(v, cfg, role="V", bank=bank)
    acfg = m.AttentionConfig(B, HQ, HKV, TQ, TK, 128, causal=causal)
    name = m.attention_kernel(q, pk, pv, bank, acfg, prefill=mode)
    assert name == ("prefill_tc (tcgen05 flash attention)" if mode == "tcgen05"
                    else "decode_fast_kernel (fp16) + torch SDPA"), name
    out = m.fused_attend(q, pk, pv, bank, acfg, prefill=mode).double().cpu().numpy()
    kd = m.decode_tensor(pk, bank, dtype=torch.float64).cpu().numpy()
    vd = m.decode_tensor(pv, bank, dtype=torch.float64).cpu().numpy()
    # kd / vd: the fp64 decode, bit-exact against the oracle's decode
    # (test_gpu_parity.py); the dense attention is the oracle's
    dense = O.reference_attend(q.double().cpu().numpy(), kd, vd, HQ // HKV, causal=causal)
    err = np.abs(out - dense) / np.maximum(1.0, np.abs(dense))
    assert err.max() <= 2e-3, err.max()
