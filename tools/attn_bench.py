import sys, os, torch, time
sys.path.insert(0, os.getcwd())
import paper_2605_27646_b200 as hq
dev = torch.device("cuda", 0)
B, HQ, HKV, T, D = 32, 32, 8, 32768, 128
g = torch.Generator(device=dev).manual_seed(4)
c = hq.CodecConfig(64, 4); bank = hq.CodebookBank(0, 64)
k = torch.randn((B, HKV, T, D), generator=g, device=dev, dtype=torch.float16)
pk = hq.encode_tensor(k, c, role="K", bank=bank); del k
v = torch.randn((B, HKV, T, D), generator=g, device=dev, dtype=torch.float16)
pv = hq.encode_tensor(v, c, role="V", bank=bank); del v
q = torch.randn((B, HQ, 1, D), generator=g, device=dev)
acfg = hq.AttentionConfig(B, HQ, HKV, 1, T, D)
out = torch.empty_like(q)
for splits in (0, 2, 4, 8, 16):
    for _ in range(3): hq.fused_attend(q, pk, pv, bank, acfg, out=out, num_splits=splits)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): hq.fused_attend(q, pk, pv, bank, acfg, out=out, num_splits=splits)
    b.record(); torch.cuda.synchronize()
    print("splits", splits, "ms", a.elapsed_time(b) / 10)
