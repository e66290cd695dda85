"""Med3x decode timing on C3 units: 56 decodes (28 layers x K,V, (1,4,32768,128),
S=64, b_r=6, C=3) back to back on one stream."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27646_b200 as hq
from bench import WORKLOADS, make_input
dev = torch.device("cuda", 0)
wl = WORKLOADS["c3"]
cfg = hq.CodecConfig(64, 6, outlier_multiplier=3.0)
bank = hq.CodebookBank(0, 64)
qts = [hq.encode_tensor(make_input(torch, wl, l, r, dev), cfg, layer=l, role=r, bank=bank)
       for l in range(28) for r in ("K", "V")]
outs = [torch.empty((1, 4, 32768, 128), dtype=torch.float16, device=dev) for _ in range(2)]
for _ in range(2):
    for i, qt in enumerate(qts):
        hq.decode_tensor(qt, bank, dtype=torch.float16, out=outs[i % 2], check=False)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for i, qt in enumerate(qts):
        hq.decode_tensor(qt, bank, dtype=torch.float16, out=outs[i % 2], check=False)
    b.record(); torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b))
print(f"C3 decode step (56 units): {best:.3f} ms")
