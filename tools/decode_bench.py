"""Decode kernel timing for one (1, 8, 32768, 128) S=64 unit beside write-only
and copy references of the same output size (CUDA events, L2-cold by size)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_27646_b200 as hq  # noqa: E402


def timeit(fn, reps=50, warm=5):
    for _ in range(warm):
        fn()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


dev = torch.device("cuda", 0)
units = 16  # rotate over units so the packed inputs are L2-cold
xs = [torch.randn((1, 8, 32768, 128), device=dev).half() for _ in range(units)]
cfg = hq.CodecConfig(64, 4)
bank = hq.CodebookBank(0, 64)
qts = [hq.encode_tensor(x, cfg, bank=bank) for x in xs]
outs = [torch.empty_like(xs[0]) for _ in range(2)]
i = [0]


def dec(dtype=torch.float16):
    k = i[0] = i[0] + 1
    hq.decode_tensor(qts[k % units], bank, dtype=dtype, out=outs[k & 1] if dtype == torch.float16
                     else None, check=False)


t16 = timeit(dec)
packed = (qts[0].n_coded * 15 + 7) // 8 + 2 * 8 * 32768
fp16 = xs[0].numel() * 2
print(f"decode fp16: {t16:.2f} us  alg bytes {(packed + fp16) / 1e6:.1f} MB -> "
      f"{(packed + fp16) / t16 / 1e3:.0f} GB/s")
big = [torch.empty(64 * 1024 * 1024 // 2, dtype=torch.float16, device=dev) for _ in range(4)]
j = [0]


def fill():
    j[0] += 1
    big[j[0] % 4][: fp16 // 2].fill_(1.0)


tw = timeit(fill)
print(f"write-only fill of {fp16 / 1e6:.1f} MB: {tw:.2f} us -> {fp16 / tw / 1e3:.0f} GB/s")


def copy():
    j[0] += 1
    big[j[0] % 4][: fp16 // 2].copy_(big[(j[0] + 1) % 4][: fp16 // 2])


tc = timeit(copy)
print(f"copy {fp16 / 1e6:.1f} MB: {tc:.2f} us -> {2 * fp16 / tc / 1e3:.0f} GB/s (read+write)")
