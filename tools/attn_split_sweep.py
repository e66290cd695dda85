import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2605_27646_b200 as hq
dev = torch.device("cuda", 0)
B, HQ, HKV, D, T = 32, 32, 8, 128, 32768
g = torch.Generator(device=dev).manual_seed(4)
cfg = hq.CodecConfig(64, 4); bank = hq.CodebookBank(0, 64)
k = torch.randn((B, HKV, T, D), generator=g, device=dev, dtype=torch.float16)
pk = hq.encode_tensor(k, cfg, role="K", bank=bank)
v = torch.randn((B, HKV, T, D), generator=g, device=dev, dtype=torch.float16)
pv = hq.encode_tensor(v, cfg, role="V", bank=bank)
del k, v
q = torch.randn((B, HQ, 1, D), generator=g, device=dev)
acfg = hq.AttentionConfig(B, HQ, HKV, 1, T, D)
out = torch.empty_like(q)
def timeit(fn, reps=20):
    for _ in range(3): fn()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for s in [0, 1, 2, 3, 4, 5, 6, 8, 10, 12, 16]:
    print(s, round(timeit(lambda: hq.fused_attend(q, pk, pv, bank, acfg, out=out, num_splits=s)), 4))
