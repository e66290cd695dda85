"""Host-side cost of the public API per (1, 8, 32768, 128) unit: time to
enqueue encode_tensor + decode_tensor (no synchronisation), vs GPU time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_27646_b200 as hq  # noqa: E402

dev = torch.device("cuda", 0)
x = torch.randn((1, 8, 32768, 128), device=dev).half()
cfg = hq.CodecConfig(64, 4)
bank = hq.CodebookBank(0, 64)
out = torch.empty_like(x)
for _ in range(3):
    qt = hq.encode_tensor(x, cfg, bank=bank, sync=False)
    hq.decode_tensor(qt, bank, dtype=torch.float16, out=out, check=False)
torch.cuda.synchronize()
n = 64
t0 = time.perf_counter()
for _ in range(n):
    qt = hq.encode_tensor(x, cfg, bank=bank, sync=False)
t1 = time.perf_counter()
for _ in range(n):
    hq.decode_tensor(qt, bank, dtype=torch.float16, out=out, check=False)
t2 = time.perf_counter()
torch.cuda.synchronize()
t3 = time.perf_counter()
print(f"host enqueue: encode {1e3 * (t1 - t0) / n:.3f} ms/unit, decode {1e3 * (t2 - t1) / n:.3f} "
      f"ms/unit; wall incl. GPU {1e3 * (t3 - t0) / n:.3f} ms/unit")
