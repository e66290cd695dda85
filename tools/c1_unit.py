"""Time one C1 unit encode (1, 8, 4096, 128) fp16, S=16, Med3x, replayed as a CUDA graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_27646_b200 as hq  # noqa: E402

dev = torch.device("cuda", 0)
x = torch.randn((1, 8, 4096, 128), generator=torch.Generator(device=dev).manual_seed(0),
                device=dev).half()
cfg = hq.CodecConfig(16, 4, outlier_multiplier=3.0)
bank = hq.CodebookBank(0, 16)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    hq.encode_tensor(x, cfg, bank=bank, sync=False)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    hq.encode_tensor(x, cfg, bank=bank, sync=False)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    g.replay()
b.record()
torch.cuda.synchronize()
print(f"C1 unit encode (graph): {a.elapsed_time(b) / 50 * 1e3:.1f} us")
