"""The tcgen05 prefill kernels forced one by one (HQMQ_FA_VARIANT: 1 = 4-warp
kernel, 2 = two-tile 64-key kernel, 3 = one-tile 128-key kernel, 4 = two-CTAs-per-SM
128-key kernel) against the dense fp64 attention over the decoded
cache, in subprocesses (the variant is read once per process).  The default
kernel is covered by test_gpu_parity.py::test_attention_prefill_tensor_core."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SNIPPET = r"""
import sys, torch
sys.path.insert(0, {root!r})
import paper_2605_27646_b200 as m
worst = 0.0
for (B, HQ, HKV, TQ, TK, causal) in [(1, 8, 2, 300, 300, True), (2, 4, 4, 130, 200, True),
                                      (1, 16, 2, 96, 96, False)]:
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(TQ + TK)
    cfg = m.CodecConfig(64, 4); bank = m.CodebookBank(0, 64)
    k = torch.randn((B, HKV, TK, 128), generator=g, device=dev).half()
    v = torch.randn((B, HKV, TK, 128), generator=g, device=dev).half()
    q = torch.randn((B, HQ, TQ, 128), generator=g, device=dev)
    pk = m.encode_tensor(k, cfg, role="K", bank=bank); pv = m.encode_tensor(v, cfg, role="V", bank=bank)
    acfg = m.AttentionConfig(B, HQ, HKV, TQ, TK, 128, causal=causal)
    out = m.fused_attend(q, pk, pv, bank, acfg).double()
    dense = m.reference_attend(q, m.decode_tensor(pk, bank, dtype=torch.float64),
                               m.decode_tensor(pv, bank, dtype=torch.float64), acfg)
    worst = max(worst, (out - dense).abs().max().item())
print("WORST", worst)
"""


@pytest.mark.parametrize("variant", ["1", "2", "3", "4"])
def test_prefill_variant(cuda, variant):
    env = dict(os.environ, HQMQ_FA_VARIANT=variant)
    res = subprocess.run([sys.executable, "-c", SNIPPET.format(root=ROOT)], env=env,
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    worst = float(res.stdout.strip().split("WORST")[-1])
    assert worst < 2e-3, worst


def test_prefill_default_long(cuda):
    """The automatic choice for >= 4096 keys (two-CTAs-per-SM kernel), causal and
    chunked (T_q < T_kv), against the dense fp64 attention over the decoded cache."""
    import torch

    import paper_2605_27646_b200 as m

    g = torch.Generator(device=cuda).manual_seed(11)
    cfg = m.CodecConfig(64, 4)
    bank = m.CodebookBank(0, 64)
    for (B, HQ, HKV, TQ, TK) in [(1, 8, 2, 4500, 4500), (1, 4, 1, 700, 5000)]:
        k = torch.randn((B, HKV, TK, 128), generator=g, device=cuda).half()
        v = torch.randn((B, HKV, TK, 128), generator=g, device=cuda).half()
        q = torch.randn((B, HQ, TQ, 128), generator=g, device=cuda)
        pk = m.encode_tensor(k, cfg, role="K", bank=bank)
        pv = m.encode_tensor(v, cfg, role="V", bank=bank)
        acfg = m.AttentionConfig(B, HQ, HKV, TQ, TK, 128, causal=True)
        out = m.fused_attend(q, pk, pv, bank, acfg).double()
        dense = m.reference_attend(q, m.decode_tensor(pk, bank, dtype=torch.float64),
                                   m.decode_tensor(pv, bank, dtype=torch.float64), acfg)
        assert (out - dense).abs().max().item() < 2e-3
