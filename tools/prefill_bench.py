"""Prefill attention over the compressed cache (Tq = Tkv, causal) vs fp16 SDPA,
the paper's prefill workload: B=1, Hq=32, Hkv=8, T=2048, d=128."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import paper_2605_27646_b200 as hq  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


dev = torch.device("cuda", 0)
for B, T in ((1, 2048), (1, 8192), (4, 4096)):
    g = torch.Generator(device=dev).manual_seed(1)
    cfg = hq.CodecConfig(64, 4)
    bank = hq.CodebookBank(0, 64)
    k = torch.randn((B, 8, T, 128), generator=g, device=dev).half()
    v = torch.randn((B, 8, T, 128), generator=g, device=dev).half()
    q = torch.randn((B, 32, T, 128), generator=g, device=dev)
    pk = hq.encode_tensor(k, cfg, role="K", bank=bank)
    pv = hq.encode_tensor(v, cfg, role="V", bank=bank)
    acfg = hq.AttentionConfig(B, 32, 8, T, T, 128)
    t_hq = timeit(lambda: hq.fused_attend(q, pk, pv, bank, acfg))
    qh = q.half()
    t_sd = timeit(lambda: F.scaled_dot_product_attention(qh, k, v, is_causal=True, enable_gqa=True))
    kd = hq.decode_tensor(pk, bank, dtype=torch.float16)
    vd = hq.decode_tensor(pv, bank, dtype=torch.float16)
    t_dq = timeit(lambda: F.scaled_dot_product_attention(
        qh, hq.decode_tensor(pk, bank, dtype=torch.float16, out=kd, check=False),
        hq.decode_tensor(pv, bank, dtype=torch.float16, out=vd, check=False),
        is_causal=True, enable_gqa=True))
    print(f"B={B} T={T}: fused {t_hq:.3f} ms | decode-then-SDPA {t_dq:.3f} ms | fp16 SDPA {t_sd:.3f} ms")
