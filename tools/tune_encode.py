"""Time the encode of one (1, 8, 32768, 128) fp16 unit per kernel variant.

    python tools/tune_encode.py            # runs every HQMQ_ENC_VARIANT in a subprocess
"""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(S: int, outlier: bool, reps: int = 20):
    sys.path.insert(0, ROOT)
    import torch

    import paper_2605_27646_b200 as hq

    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((1, 8, 32768, 128), generator=g, device=dev).half()
    cfg = hq.CodecConfig(S, 4, outlier_multiplier=3.0 if outlier else None)
    bank = hq.CodebookBank(0, S)
    for _ in range(3):
        qt = hq.encode_tensor(x, cfg, bank=bank, sync=False)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        qt = hq.encode_tensor(x, cfg, bank=bank, sync=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    lane_ops = 20 * S * x.numel() / 4
    return {"S": S, "outlier": outlier, "ms": round(ms, 4),
            "gbs": round(x.numel() * 2 / ms / 1e6, 2),
            "tlane": round(lane_ops / ms / 1e9, 2), "fixup": qt.n_fixup}


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        res = [one(64, False), one(256, False), one(16, True), one(64, True)]
        print(json.dumps(res))
    else:
        for v in (sys.argv[1:] or ["0", "1", "2", "3"]):
            env = dict(os.environ, HQMQ_ENC_VARIANT=v)
            out = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True,
                                 text=True)
            print("variant", v, out.stdout.strip() or out.stderr[-500:], flush=True)
