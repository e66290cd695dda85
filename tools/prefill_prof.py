import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2605_27646_b200 as hq
dev = torch.device("cuda", 0)
B, T = 1, 8192
g = torch.Generator(device=dev).manual_seed(1)
cfg = hq.CodecConfig(64, 4); bank = hq.CodebookBank(0, 64)
k = torch.randn((B, 8, T, 128), generator=g, device=dev).half()
v = torch.randn((B, 8, T, 128), generator=g, device=dev).half()
q = torch.randn((B, 32, T, 128), generator=g, device=dev)
pk = hq.encode_tensor(k, cfg, role="K", bank=bank); pv = hq.encode_tensor(v, cfg, role="V", bank=bank)
acfg = hq.AttentionConfig(B, 32, 8, T, T, 128)
for _ in range(2): hq.fused_attend(q, pk, pv, bank, acfg)
torch.cuda.synchronize()
