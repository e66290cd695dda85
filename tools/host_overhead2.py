"""Host-side cost of the public API calls (no GPU work in the way): wall time
per call of decode_tensor / encode_tensor(sync=False) / fused_attend on tiny
inputs, averaged over many calls, and the device time of the same calls."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_27646_b200 as hq  # noqa: E402

dev = torch.device("cuda", 0)
cfg = hq.CodecConfig(64, 4)
bank = hq.CodebookBank(0, 64)
x = torch.randn((1, 8, 64, 128), device=dev).half()
qt = hq.encode_tensor(x, cfg, bank=bank)
out = torch.empty_like(x)


def wall(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6


print(f"decode_tensor(out=, check=False): {wall(lambda: hq.decode_tensor(qt, bank, out=out, check=False)):.1f} us/call")
print(f"decode_tensor(dtype=f16, check=False): {wall(lambda: hq.decode_tensor(qt, bank, dtype=torch.float16, check=False)):.1f} us/call")
print(f"encode_tensor(sync=False): {wall(lambda: hq.encode_tensor(x, cfg, bank=bank, sync=False), 500):.1f} us/call")
q = torch.randn((1, 32, 1, 128), device=dev)
pk = hq.encode_tensor(x, cfg, role="K", bank=bank)
pv = hq.encode_tensor(x, cfg, role="V", bank=bank)
acfg = hq.AttentionConfig(1, 32, 8, 1, 64, 128)
o = torch.empty_like(q)
print(f"fused_attend(out=): {wall(lambda: hq.fused_attend(q, pk, pv, bank, acfg, out=o)):.1f} us/call")
