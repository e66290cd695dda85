"""Small driver for ncu captures: one C2 unit (1, 8, 32768, 128) fp16, S=64,
encoded and decoded `--reps` times, plus one C4-shaped fused attention call.

    ncu --set full --clock-control none --import-source on -k regex:encode_tile \
        -s 1 -c 1 -o gpurun_out/prof_encode python tools/prof_unit.py
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_27646_b200 as hq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--S", type=int, default=64)
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--outlier", action="store_true")
    ap.add_argument("--attn-tokens", type=int, default=32768)
    ap.add_argument("--attn-batch", type=int, default=32)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((1, 8, args.tokens, 128), generator=g, device=dev).half()
    cfg = hq.CodecConfig(args.S, 4, outlier_multiplier=3.0 if args.outlier else None)
    bank = hq.CodebookBank(0, args.S)
    out = torch.empty_like(x)
    for _ in range(args.reps):
        qt = hq.encode_tensor(x, cfg, bank=bank, sync=False)
        hq.decode_tensor(qt, bank, dtype=torch.float16, out=out, check=False)
    torch.cuda.synchronize()
    if args.attn_batch:
        B, T = args.attn_batch, args.attn_tokens
        c = hq.CodecConfig(64, 4)
        b64 = hq.CodebookBank(0, 64)
        k = torch.randn((B, 8, T, 128), generator=g, device=dev).half()
        pk = hq.encode_tensor(k, c, role="K", bank=b64)
        v = torch.randn((B, 8, T, 128), generator=g, device=dev).half()
        pv = hq.encode_tensor(v, c, role="V", bank=b64)
        q = torch.randn((B, 32, 1, 128), generator=g, device=dev)
        acfg = hq.AttentionConfig(B, 32, 8, 1, T, 128)
        for _ in range(2):
            hq.fused_attend(q, pk, pv, b64, acfg)
        torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
