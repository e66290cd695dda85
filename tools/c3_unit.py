"""One C3 unit (Qwen2.5-7B outlier-heavy, (1, 4, 32768, 128), S=64, b_r=6, C=3)
encoded `reps` times on one stream: device time per encode (CUDA events, back
to back) -- and, under ncu, the launch list of the encode's kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27646_b200 as hq
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import WORKLOADS, make_input

dev = torch.device("cuda", 0)
wl = WORKLOADS["c3"]
x = make_input(torch, wl, 3, "K", dev)
cfg = hq.CodecConfig(64, 6, outlier_multiplier=3.0)
bank = hq.CodebookBank(0, 64)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for _ in range(3):
    hq.encode_tensor(x, cfg, layer=3, role="K", bank=bank, sync=False)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    hq.encode_tensor(x, cfg, layer=3, role="K", bank=bank, sync=False)
b.record(); torch.cuda.synchronize()
print(f"C3 unit encode: {a.elapsed_time(b) / reps:.4f} ms (back to back, {reps} reps)")
