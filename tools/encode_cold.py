"""Encode timing for one (1,8,32768,128) fp16 unit: the same input repeatedly
(L2-warm) vs rotating over 16 distinct inputs (L2-cold), per kernel variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_27646_b200 as hq  # noqa: E402

dev = torch.device("cuda", 0)
S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
xs = [torch.randn((1, 8, 32768, 128), device=dev).half() for _ in range(16)]
cfg = hq.CodecConfig(S, 4)
bank = hq.CodebookBank(0, S)


def run(inputs, reps=32):
    for i in range(3):
        hq.encode_tensor(inputs[i % len(inputs)], cfg, bank=bank, sync=False)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(reps):
        hq.encode_tensor(inputs[i % len(inputs)], cfg, bank=bank, sync=False)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


print(f"S={S} variant={os.environ.get('HQMQ_ENC_VARIANT', '0')}: warm {run(xs[:1]):.3f} ms, "
      f"cold {run(xs):.3f} ms per unit")
