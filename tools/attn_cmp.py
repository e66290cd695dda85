import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2605_27646_b200 as hq
dev = torch.device("cuda", 0)
def run(B, HKV, T, reps=20):
    HQ, D = HKV * 4, 128
    g = torch.Generator(device=dev).manual_seed(4)
    cfg = hq.CodecConfig(64, 4); bank = hq.CodebookBank(0, 64)
    k = torch.randn((B, HKV, T, D), generator=g, device=dev, dtype=torch.float16)
    pk = hq.encode_tensor(k, cfg, role="K", bank=bank); del k
    v = torch.randn((B, HKV, T, D), generator=g, device=dev, dtype=torch.float16)
    pv = hq.encode_tensor(v, cfg, role="V", bank=bank); del v
    q = torch.randn((B, HQ, 1, D), generator=g, device=dev)
    acfg = hq.AttentionConfig(B, HQ, HKV, 1, T, D)
    out = torch.empty_like(q)
    for _ in range(3): hq.fused_attend(q, pk, pv, bank, acfg, out=out)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): hq.fused_attend(q, pk, pv, bank, acfg, out=out)
    b.record(); torch.cuda.synchronize()
    print(f"B={B} Hkv={HKV} T={T}: {a.elapsed_time(b)/reps:.4f} ms")
for args in [(32, 8, 32768), (32, 8, 131072), (1, 8, 32768), (4, 8, 8192), (8, 8, 4096), (64, 8, 2048)]:
    run(*args)
