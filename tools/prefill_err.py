"""Prefill accuracy: our tcgen05 fused_attend vs decode(fp16) + torch SDPA (cuDNN),
both against the oracle's dense fp64 attention over the fp64 decode."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np, torch
import torch.nn.functional as F
import paper_2605_27646_b200 as m
import hqmq_oracle as O

dev = torch.device("cuda", 0)
for (B, HQ, HKV, TQ, TK, causal) in [(1, 8, 2, 300, 300, True), (2, 4, 4, 130, 200, True),
                                      (1, 16, 2, 96, 96, False), (1, 8, 2, 200, 4100, True),
                                      (1, 4, 1, 64, 4096, False), (1, 32, 8, 256, 256, True)]:
    g = torch.Generator(device=dev).manual_seed(TQ + TK)
    cfg = m.CodecConfig(64, 4)
    bank = m.CodebookBank(0, 64)
    k = torch.randn((B, HKV, TK, 128), generator=g, device=dev).half()
    v = torch.randn((B, HKV, TK, 128), generator=g, device=dev).half()
    q = torch.randn((B, HQ, TQ, 128), generator=g, device=dev)
    pk = m.encode_tensor(k, cfg, role="K", bank=bank)
    pv = m.encode_tensor(v, cfg, role="V", bank=bank)
    acfg = m.AttentionConfig(B, HQ, HKV, TQ, TK, 128, causal=causal)
    kd = m.decode_tensor(pk, bank, dtype=torch.float64)
    vd = m.decode_tensor(pv, bank, dtype=torch.float64)
    dense = O.reference_attend(q.double().cpu().numpy(), kd.cpu().numpy(), vd.cpu().numpy(),
                               HQ // HKV, causal=causal)
    bound = np.maximum(1.0, np.abs(dense))
    ours = m.fused_attend(q, pk, pv, bank, acfg).double().cpu().numpy()
    # SDPA's causal mask is top-left aligned; the reference's is bottom-right (T_q <= T_kv)
    mask = None
    if causal:
        i = torch.arange(TQ, device=dev)[:, None]
        j = torch.arange(TK, device=dev)[None, :]
        mask = j <= i + (TK - TQ)
    sd = F.scaled_dot_product_attention(q.half(), kd.half(), vd.half(), attn_mask=mask,
                                        enable_gqa=True).double().cpu().numpy()
    e_o = (np.abs(ours - dense) / bound).max()
    e_s = (np.abs(sd - dense) / bound).max()
    print(f"B={B} HQ={HQ} HKV={HKV} TQ={TQ} TK={TK} causal={causal}: {m.attention_kernel(q, pk, pv, bank, acfg)} "
          f"err {e_o:.2e} | decode fp16 + SDPA err {e_s:.2e}")
